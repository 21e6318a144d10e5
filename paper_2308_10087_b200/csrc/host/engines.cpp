// Trainers of the C++ API (engines.hpp:79-99) on the GPU engine.
//
// train_pipeline<float> keeps the reference's contract (engines_impl.hpp:515-537
// validation, :901-907 result assembly) and runs one gp_ctx per stage, one host
// thread per stage (the reference's Fabric::Mode::Concurrent shape,
// fabric.cpp:401-422). The chunk schedule (shuffle_chunk_order) is computed on
// the host and handed to every stage, so schedule order is bit-exact. Stage
// boundaries use gp_link_local (device-to-device copies ordered by CUDA events);
// the one-process-per-GPU NCCL path is driven directly through the C-ABI
// (bench.py).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <type_traits>

#include "gnnsim_b200.hpp"

namespace gnnsim {

namespace {

void check(gp_status s, gp_ctx* ctx, const char* what) {
    if (s == GP_OK) return;
    const std::string msg = std::string(what) + ": " + gp_last_error(ctx);
    switch (s) {
        case GP_EINVAL: throw std::invalid_argument(msg);
        case GP_ENUMERIC: throw NumericError(msg);
        case GP_EFABRIC: throw FabricError(msg);
        default: throw GpError(s, msg);
    }
}

// Epoch barrier that can be aborted when a stage thread fails.
class StageBarrier {
  public:
    explicit StageBarrier(uint32_t n) : n_(n) {}
    bool arrive_and_wait() {
        std::unique_lock<std::mutex> lk(mu_);
        if (aborted_) return false;
        const uint64_t gen = gen_;
        if (++waiting_ == n_) {
            waiting_ = 0;
            ++gen_;
            cv_.notify_all();
            return true;
        }
        cv_.wait(lk, [&] { return gen_ != gen || aborted_; });
        return !aborted_;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu_);
        aborted_ = true;
        cv_.notify_all();
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    uint32_t n_, waiting_ = 0;
    uint64_t gen_ = 0;
    bool aborted_ = false;
};

// GP_HOST_TIMING=1: wall time of each phase of a trainer call on stderr (e2e diagnosis).
struct PhaseTimer {
    bool on = false;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    PhaseTimer() {
        const char* e = std::getenv("GP_HOST_TIMING");
        on = e && std::string(e) == "1";
    }
    void mark(const char* what) {
        if (!on) return;
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gp host] %-20s %8.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
        t0 = t1;
    }
};

gp_layer_spec to_gp(const LayerSpec& s) {
    gp_layer_spec g{};
    g.kind = uint32_t(s.kind);
    g.in_dim = s.in_dim;
    g.out_dim = s.out_dim;
    g.relu = s.relu ? 1u : 0u;
    g.alpha = s.alpha;
    g.beta = s.beta;
    return g;
}

struct Ctxs {
    std::vector<gp_ctx*> v;
    void destroy() {
        for (auto* c : v) gp_destroy(c);
        v.clear();
    }
    ~Ctxs() { destroy(); }
};

void validate_run(const Dataset& ds, const ChunkPlan& plan, const StageAssignment& sa, uint32_t L) {
    const uint32_t S = sa.num_stages;
    if (plan.chunk_of.size() != ds.num_vertices())
        throw std::invalid_argument("train_hybrid: plan/partition do not cover the graph");
    if (plan.num_chunks == 0) throw std::invalid_argument("train_pipeline: empty chunk plan");
    if (sa.ranges.size() != S || S == 0 || sa.begin(0) != 0 || sa.end(S - 1) != L)
        throw std::invalid_argument("train_hybrid: stage ranges must cover all layers");
    for (uint32_t s = 0; s + 1 < S; ++s)
        if (sa.end(s) != sa.begin(s + 1) || sa.end(s) <= sa.begin(s))
            throw std::invalid_argument("train_hybrid: stage ranges must be consecutive");
    if (sa.end(S - 1) <= sa.begin(S - 1)) throw std::invalid_argument("train_hybrid: empty stage");
}

}  // namespace

namespace {

// The worker body of train_hybrid (engines_impl.hpp:515-909) for S stages x G
// graph partitions: worker (s, r) is one gp_ctx; `part` is null for G = 1.
// `worker_id[s*G + r]` is the fabric worker id (GroupMap::groups[s][r]) and
// node_of is indexed by it (link classes of the ledger).
TrainResult<float> run_hybrid_f32(const Dataset& ds, const Partition* part, const ChunkPlan& plan,
                                  const StageAssignment& sa, uint32_t G, const std::vector<uint32_t>& worker_id,
                                  std::vector<uint32_t> node_of, const TrainOptions<float>& opt) {
    PhaseTimer timer;
    ds.validate();
    const auto specs = build_layer_specs(opt.model, ds.num_features(), ds.num_classes);
    const uint32_t L = uint32_t(specs.size());
    validate_run(ds, plan, sa, L);
    timer.mark("validate");
    const uint32_t S = sa.num_stages, K = plan.num_chunks, W = S * G;
    const VertexId n = ds.num_vertices();
    uint64_t split_count[3] = {0, 0, 0};
    for (uint8_t s : ds.split)
        if (s >= 1 && s <= 3) ++split_count[s - 1];
    if (split_count[0] == 0) throw std::invalid_argument("train_hybrid: empty train mask");

    std::vector<gp_layer_spec> gspecs;
    for (const auto& s : specs) gspecs.push_back(to_gp(s));
    // normalize_adjacency<float> (graph.cpp:68-98) runs inside gp_upload_graph_raw
    auto params = init_params<float>(specs, opt.seed);
    const uint32_t t0 = opt.resume ? opt.resume->epoch : 0;  // epochs already trained
    if (opt.resume) {
        const auto& rs = *opt.resume;
        if (rs.params.size() != L || rs.adam_m.size() != L || rs.adam_v.size() != L)
            throw std::invalid_argument("resume: state does not match the model's layers");
        for (uint32_t l = 0; l < L; ++l)
            for (const auto* p : {&rs.params[l], &rs.adam_m[l], &rs.adam_v[l]})
                if (p->weight.rows() != specs[l].k_in() || p->weight.cols() != specs[l].out_dim ||
                    p->bias.size() != (specs[l].has_bias() ? specs[l].out_dim : 0u))
                    throw std::invalid_argument("resume: layer " + std::to_string(l) + " has the wrong shape");
        params = rs.params;
        if (!opt.staleness.synchronous_mode && rs.epoch > 0 && rs.history.empty())
            throw std::invalid_argument(
                "resume: stale-mode training reads historical embeddings the state does not hold "
                "(save it with TrainOptions::keep_history, or resume in synchronous mode)");
    }
    timer.mark("init_params");

    int ndev = 0;
    gp_device_count(&ndev);
    if (ndev == 0) throw GpError(GP_ECUDA, "train_pipeline: no CUDA device (the GPU engine has no CPU fallback)");

    Ctxs ctx;
    for (uint32_t w = 0; w < W; ++w) {
        const uint32_t s = w / G, r = w % G;
        gp_stage_config c{};
        c.device = opt.device >= 0 ? opt.device : int(w % uint32_t(ndev));
        c.num_vertices = n;
        c.num_chunks = K;
        c.num_stages = S;
        c.stage = s;
        c.layer_begin = sa.begin(s);
        c.layer_end = sa.end(s);
        c.num_layers = L;
        c.specs = gspecs.data();
        c.hidden = opt.model.hidden;
        c.num_classes = ds.num_classes;
        c.dropout = opt.model.dropout;
        c.seed = opt.seed;
        c.optimizer = opt.optimizer.kind == OptimizerKind::Sgd ? 1u : 0u;
        c.lr = opt.optimizer.lr;
        c.beta1 = opt.optimizer.beta1;
        c.beta2 = opt.optimizer.beta2;
        c.eps = opt.optimizer.eps;
        c.fix_alpha = opt.staleness.fix_alpha;
        c.historical_gradients = opt.staleness.historical_gradients ? 1u : 0u;
        c.synchronous_mode = opt.staleness.synchronous_mode ? 1u : 0u;
        c.group_size = G;
        c.group_rank = r;
        gp_ctx* g = nullptr;
        check(gp_create(&c, &g), nullptr, "gp_create");
        ctx.v.push_back(g);
        timer.mark("gp_create");
        if (G > 1) check(gp_upload_partition(g, part->assignment.data()), g, "gp_upload_partition");
        const int dev0 = opt.device >= 0 ? opt.device : 0;
        if (w == 0 || c.device != dev0) {
            check(gp_upload_graph_raw(g, ds.graph.csr_offsets.data(), ds.graph.csr_neighbors.data(),
                                      ds.graph.csr_neighbors.size(), opt.model.self_loops ? 1 : 0,
                                      plan.chunk_of.data()),
                  g, "gp_upload_graph_raw");
        } else {
            check(gp_share_graph(g, ctx.v[0]), g, "gp_share_graph");
        }
        timer.mark("graph");
        if (s == 0) check(gp_upload_features(g, ds.features.data(), ds.num_features()), g, "gp_upload_features");
        if (s + 1 == S) check(gp_upload_labels(g, ds.labels.data(), ds.split.data()), g, "gp_upload_labels");
        for (uint32_t l = sa.begin(s); l < sa.end(s); ++l)
            check(gp_set_layer_params(g, l, params[l].weight.data(), params[l].bias.empty() ? nullptr : params[l].bias.data()),
                  g, "gp_set_layer_params");
        if (opt.resume)
            for (uint32_t l = sa.begin(s); l < sa.end(s); ++l) {
                const auto& m = opt.resume->adam_m[l];
                const auto& v = opt.resume->adam_v[l];
                check(gp_set_optimizer_state(g, l, m.weight.data(), v.weight.data(), m.bias.empty() ? nullptr : m.bias.data(),
                                             v.bias.empty() ? nullptr : v.bias.data(), opt.resume->optimizer_step),
                      g, "gp_set_optimizer_state");
            }
        if (opt.resume && !opt.staleness.synchronous_mode)
            for (const auto& h : opt.resume->history)
                if (h.worker == w) {
                    const uint32_t li = h.which == GP_BUF_HIST_IN ? 0 : h.layer - sa.begin(s);
                    check(gp_upload_history(g, h.which, li, h.rows.data(), h.rows.size(), t0), g, "gp_upload_history");
                }
        if (opt.profile) gp_set_profiling(g, 1);
        if (opt.fabric.collect_trace) gp_set_trace(g, 1);
        if (s > 0) check(gp_link_local(ctx.v[w - G], g), g, "gp_link_local");  // same rank, previous stage
    }
    if (G > 1)
        for (uint32_t s = 0; s < S; ++s)
            check(gp_link_group(&ctx.v[size_t(s) * G], G), ctx.v[size_t(s) * G], "gp_link_group");

    timer.mark("create+upload");
    const uint32_t T = opt.epochs;
    std::vector<std::vector<gp_epoch_stats>> stats(W, std::vector<gp_epoch_stats>(T));
    std::vector<std::exception_ptr> errs(W);
    StageBarrier barrier(W);
    auto body = [&](uint32_t w) {
        try {
            for (uint32_t t = t0 + 1; t <= t0 + T; ++t) {
                if (!barrier.arrive_and_wait()) return;  // epoch entry sync (engines_impl.hpp:668)
                std::vector<uint32_t> order(K);
                for (uint32_t k = 0; k < K; ++k) order[k] = k;
                if (opt.staleness.shuffle_chunks) order = shuffle_chunk_order(plan, t, opt.seed);
                check(gp_run_epoch(ctx.v[w], t, order.data(), &stats[w][t - t0 - 1]), ctx.v[w], "gp_run_epoch");
                // fill_quality_metrics (engines_impl.hpp:164-171) throws inside the epoch that
                // produced a non-finite loss; a partial sum over this rank's rows suffices
                if (stats[w][t - t0 - 1].has_quality && !std::isfinite(stats[w][t - t0 - 1].loss_sum))
                    throw NumericError("non-finite training loss at epoch " + std::to_string(t));
            }
        } catch (...) {
            errs[w] = std::current_exception();
            barrier.abort();
            for (auto* c : ctx.v) gp_abort(c);
        }
    };
    if (W == 1) {
        body(0);
    } else {
        std::vector<std::thread> pool;
        for (uint32_t w = 0; w < W; ++w) pool.emplace_back(body, w);
        for (auto& th : pool) th.join();
    }
    timer.mark("epochs");
    // Prefer the root cause over "transport aborted" follow-on errors.
    for (uint32_t pass = 0; pass < 2; ++pass)
        for (uint32_t w = 0; w < W; ++w) {
            if (!errs[w]) continue;
            if (pass == 0) {
                try {
                    std::rethrow_exception(errs[w]);
                } catch (const FabricError& e) {
                    if (std::string(e.what()).find("aborted") != std::string::npos) continue;
                    throw;
                }
            }
            std::rethrow_exception(errs[w]);
        }

    TrainResult<float> res;
    // measured trace (Fabric::trace fabric.cpp:256-264): all workers on one
    // timebase, seconds from the first event, stable-sorted by (start, worker)
    std::vector<double> trace_bubble(T, -1.0);
    if (opt.fabric.collect_trace) {
        std::vector<std::vector<gp_trace_event>> ev(W);
        double ns0 = 0;
        bool any = false;
        for (uint32_t w = 0; w < W; ++w) {
            uint64_t cnt = 0;
            gp_get_trace(ctx.v[w], nullptr, 0, &cnt);
            ev[w].resize(cnt);
            gp_get_trace(ctx.v[w], ev[w].data(), cnt, &cnt);
            for (const auto& e : ev[w]) {
                ns0 = any ? std::min(ns0, e.t_start_ns) : e.t_start_ns;
                any = true;
            }
        }
        std::vector<double> lo(T, 0), hi(T, 0), busy(T, 0);
        std::vector<uint8_t> seen(T, 0);
        for (uint32_t w = 0; w < W; ++w)
            for (const auto& e : ev[w]) {
                TraceEvent te{};
                te.worker = worker_id[w];
                te.t_start = (e.t_start_ns - ns0) * 1e-9;
                te.t_end = (e.t_end_ns - ns0) * 1e-9;
                te.kind = TraceEvent::Kind(e.kind);
                te.chunk = e.chunk;
                te.layer_lo = e.layer_lo;
                te.layer_hi = e.layer_hi;
                res.trace.push_back(te);
                if (e.epoch > t0 && e.epoch <= t0 + T) {
                    const uint32_t i = e.epoch - t0 - 1;
                    lo[i] = seen[i] ? std::min(lo[i], te.t_start) : te.t_start;
                    hi[i] = seen[i] ? std::max(hi[i], te.t_end) : te.t_end;
                    seen[i] = 1;
                    if (te.kind == TraceEvent::Kind::Compute) busy[i] += te.t_end - te.t_start;
                }
            }
        std::stable_sort(res.trace.begin(), res.trace.end(), [](const TraceEvent& a, const TraceEvent& b) {
            return a.t_start != b.t_start ? a.t_start < b.t_start : a.worker < b.worker;
        });
        for (uint32_t i = 0; i < T; ++i)
            if (seen[i] && hi[i] > lo[i]) trace_bubble[i] = std::max(0.0, 1.0 - busy[i] / (double(W) * (hi[i] - lo[i])));
    }
    if (node_of.empty())
        for (uint32_t w = 0; w < W; ++w) node_of.push_back(w / 4);
    auto node = [&](uint32_t s, uint32_t r) { return node_of[worker_id[size_t(s) * G + r]]; };
    res.metrics.resize(T);
    res.comm.resize(T);
    for (uint32_t t = 0; t < T; ++t) {
        EpochMetrics& m = res.metrics[t];
        m.epoch = t0 + t + 1;
        // reduce_metrics (engines_impl.hpp:131-151): group rank 0 adds ranks in order
        double loss = 0;
        uint64_t cor[3] = {0, 0, 0};
        for (uint32_t r = 0; r < G; ++r) {
            const gp_epoch_stats& q = stats[size_t(S - 1) * G + r][t];
            loss += q.loss_sum;
            for (int i = 0; i < 3; ++i) cor[i] += q.correct[i];
        }
        m.train_loss = split_count[0] ? loss / double(split_count[0]) : 0.0;  // :164-171
        if (!std::isfinite(m.train_loss)) throw NumericError("non-finite training loss at epoch " + std::to_string(m.epoch));
        m.train_acc = split_count[0] ? double(cor[0]) / double(split_count[0]) : 0.0;
        m.val_acc = split_count[1] ? double(cor[1]) / double(split_count[1]) : 0.0;
        m.test_acc = split_count[2] ? double(cor[2]) / double(split_count[2]) : 0.0;
        EpochComm& e = res.comm[t];
        double span = 0, busy = 0;
        for (uint32_t w = 0; w < W; ++w) {
            const uint32_t s = w / G, r = w % G;
            const auto& st = stats[w][t];
            span = std::max(span, double(st.epoch_ms));
            busy += st.busy_ms;
            // forward goes (s,r) -> (s+1,r), backward (s,r) -> (s-1,r)
            if (s + 1 < S) e.by_tag_link[0][node(s, r) == node(s + 1, r) ? 0 : 1] += st.bytes_sent[0];
            if (s > 0) e.by_tag_link[1][node(s, r) == node(s - 1, r) ? 0 : 1] += st.bytes_sent[1];
            // halo and weight sync stay inside the stage group; one NVSwitch node here
            for (int tag = 2; tag <= 4; ++tag) e.by_tag_link[tag][node(s, r) == node(s, 0) ? 0 : 1] += st.bytes_sent[tag];
        }
        m.comm_bytes_graph = e.graph_bytes();
        m.comm_bytes_pipeline = e.pipeline_bytes();
        m.comm_bytes_weightsync = e.weight_sync_bytes();
        m.wall_time_s = span / 1000.0;
        m.bubble_fraction = (opt.profile && span > 0) ? std::max(0.0, 1.0 - busy / (span * W)) : 0.0;
        if (trace_bubble[t] >= 0) m.bubble_fraction = trace_bubble[t];  // measured compute spans
    }
    // resumable state: every stage's group rank 0 holds its layers' parameters + moments
    res.final_state.epoch = t0 + T;
    res.final_state.params.resize(L);
    res.final_state.adam_m.resize(L);
    res.final_state.adam_v.resize(L);
    for (uint32_t s = 0; s < S; ++s) {
        gp_ctx* g = ctx.v[size_t(s) * G];
        for (uint32_t l = sa.begin(s); l < sa.end(s); ++l) {
            for (auto* p : {&res.final_state.params[l], &res.final_state.adam_m[l], &res.final_state.adam_v[l]}) {
                p->weight = MatF(specs[l].k_in(), specs[l].out_dim);
                if (specs[l].has_bias()) p->bias.assign(specs[l].out_dim, 0.f);
            }
            auto& P = res.final_state.params[l];
            auto& M = res.final_state.adam_m[l];
            auto& V = res.final_state.adam_v[l];
            check(gp_get_layer_params(g, l, P.weight.data(), P.bias.empty() ? nullptr : P.bias.data()), g,
                  "gp_get_layer_params");
            uint64_t step = 0;
            check(gp_get_optimizer_state(g, l, M.weight.data(), V.weight.data(), M.bias.empty() ? nullptr : M.bias.data(),
                                         V.bias.empty() ? nullptr : V.bias.data(), &step),
                  g, "gp_get_optimizer_state");
            res.final_state.optimizer_step = step;
        }
    }
    if (opt.keep_history && !opt.staleness.synchronous_mode) {
        const bool hist = opt.staleness.historical_gradients;
        auto fetch = [&](uint32_t w, uint32_t which, uint32_t layer, uint32_t li, uint32_t width) {
            TrainState::HistoryRows h;
            h.worker = w;
            h.which = which;
            h.layer = layer;
            h.width = width;
            h.rows.resize(size_t(n) * width);
            check(gp_download(ctx.v[w], which, li, h.rows.data(), h.rows.size()), ctx.v[w], "gp_download(history)");
            res.final_state.history.push_back(std::move(h));
        };
        for (uint32_t w = 0; w < W; ++w) {
            const uint32_t s = w / G, lb = sa.begin(s), le = sa.end(s);
            if (s > 0 && specs[lb].kind != LayerKind::Dense) fetch(w, GP_BUF_HIST_IN, lb, 0, specs[lb].in_dim);
            for (uint32_t l = lb; l < le; ++l) {
                if (l + 1 < le && specs[l + 1].kind != LayerKind::Dense)
                    fetch(w, GP_BUF_HIST_H, l, l - lb, specs[l].out_dim);
                if (hist && l > 0 && specs[l].kind != LayerKind::Dense) {
                    const uint32_t din = specs[l].in_dim;
                    fetch(w, GP_BUF_HIST_DAGG, l, l - lb,
                          specs[l].kind == LayerKind::SageConv ? ((din + 7u) & ~7u) + din : din);
                }
            }
        }
    }
    res.worker_params.resize(W);
    for (uint32_t w = 0; w < W; ++w) {
        const uint32_t s = w / G;
        WorkerParams<float>& wp = res.worker_params[worker_id[w]];
        wp.layer_begin = sa.begin(s);
        wp.layer_end = sa.end(s);
        for (uint32_t l = sa.begin(s); l < sa.end(s); ++l) {
            LayerParams<float> p;
            p.weight = MatF(specs[l].k_in(), specs[l].out_dim);
            if (specs[l].has_bias()) p.bias.assign(specs[l].out_dim, 0.f);
            check(gp_get_layer_params(ctx.v[w], l, p.weight.data(), p.bias.empty() ? nullptr : p.bias.data()),
                  ctx.v[w], "gp_get_layer_params");
            if (w % G == 0) res.params.push_back(p);  // each group's rank 0 (:901-905)
            wp.params.push_back(std::move(p));
        }
        uint64_t bytes = 0;
        gp_device_bytes(ctx.v[w], &bytes);
        res.peak_buffer_bytes = std::max(res.peak_buffer_bytes, bytes);
        gp_profile pr{};
        gp_get_profile(ctx.v[w], &pr);
        for (int k = 0; k < GP_K_NUM; ++k) {
            res.profile.ms[k] += pr.ms[k];
            res.profile.launches[k] += pr.launches[k];
            res.profile.alg_bytes[k] += pr.alg_bytes[k];
            res.profile.flops[k] += pr.flops[k];
            res.profile.gather_bytes[k] += pr.gather_bytes[k];
            res.profile.span_ms[k] += pr.span_ms[k];
        }
    }
    timer.mark("results");
    ctx.destroy();
    timer.mark("destroy");
    return res;
}

TrainResult<float> run_pipeline_f32(const Dataset& ds, const ChunkPlan& plan, const StageAssignment& sa,
                                    const TrainOptions<float>& opt) {
    std::vector<uint32_t> ids(sa.num_stages);
    for (uint32_t s = 0; s < sa.num_stages; ++s) ids[s] = s;  // assign_groups(S, 4, S, 1)
    return run_hybrid_f32(ds, nullptr, plan, sa, 1, ids, opt.fabric.node_of, opt);
}

}  // namespace

template <typename T>
TrainResult<T> train_pipeline(const Dataset& ds, const ChunkPlan& plan, const StageAssignment& sa,
                              const TrainOptions<T>& opt) {
    static_assert(std::is_same_v<T, float>, "the GPU engine computes in fp32");
    return run_pipeline_f32(ds, plan, sa, opt);
}

template <typename T>
TrainResult<T> train_sequential(const Dataset& ds, const TrainOptions<T>& opt) {
    // The S=1, K=1 pipeline reproduces train_sequential bitwise in the
    // reference (test_engines.cpp:103-113); it is the GPU engine's full-graph mode.
    ds.validate();
    const uint32_t L = uint32_t(build_layer_specs(opt.model, ds.num_features(), ds.num_classes).size());
    ChunkPlan whole = chunk_plan_from_assignment(ds.num_vertices(), std::vector<uint32_t>(ds.num_vertices(), 0));
    return train_pipeline<T>(ds, whole, make_stage_assignment(L, 1), opt);
}

template <typename T>
TrainResult<T> train_hybrid(const Dataset& ds, const Partition& part, const ChunkPlan& plan,
                            const StageAssignment& sa, const GroupMap& gmap, const TrainOptions<T>& opt) {
    ds.validate();
    const uint32_t S = sa.num_stages, G = gmap.group_size;
    if (gmap.num_workers != S * G || gmap.num_groups() != S)
        throw std::invalid_argument("train_hybrid: worker count != stages * group_size");
    if (part.num_parts != G) throw std::invalid_argument("train_hybrid: partition parts != group size");
    if (plan.chunk_of.size() != ds.num_vertices() || part.assignment.size() != ds.num_vertices())
        throw std::invalid_argument("train_hybrid: plan/partition do not cover the graph");
    if (G > 8) throw std::invalid_argument("train_hybrid: group size must be <= 8");
    static_assert(std::is_same_v<T, float>, "the GPU engine computes in fp32");
    std::vector<uint32_t> ids(size_t(S) * G);
    for (uint32_t s = 0; s < S; ++s)
        for (uint32_t r = 0; r < G; ++r) ids[size_t(s) * G + r] = gmap.groups[s][r];
    return run_hybrid_f32(ds, G > 1 ? &part : nullptr, plan, sa, G, ids,
                          opt.fabric.node_of.empty() ? gmap.node_of : opt.fabric.node_of, opt);
}

template <typename T>
TrainResult<T> train_graph_parallel(const Dataset& ds, const Partition& part, const TrainOptions<T>& opt) {
    ds.validate();
    if (part.assignment.size() != ds.num_vertices())
        throw std::invalid_argument("train_graph_parallel: partition does not cover the graph");
    const uint32_t P = part.num_parts, L = uint32_t(build_layer_specs(opt.model, ds.num_features(), ds.num_classes).size());
    ChunkPlan whole = chunk_plan_from_assignment(ds.num_vertices(), std::vector<uint32_t>(ds.num_vertices(), 0));
    GroupMap gmap = assign_groups(P, 4, 1, P);
    return train_hybrid<T>(ds, part, whole, make_stage_assignment(L, 1), gmap, opt);
}

template TrainResult<float> train_sequential<float>(const Dataset&, const TrainOptions<float>&);
template TrainResult<float> train_graph_parallel<float>(const Dataset&, const Partition&, const TrainOptions<float>&);
template TrainResult<float> train_pipeline<float>(const Dataset&, const ChunkPlan&, const StageAssignment&,
                                                  const TrainOptions<float>&);
template TrainResult<float> train_hybrid<float>(const Dataset&, const Partition&, const ChunkPlan&,
                                                const StageAssignment&, const GroupMap&, const TrainOptions<float>&);

}  // namespace gnnsim

// ref_driver — runs the UNMODIFIED reference (gnnsim, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) and dumps its
// outputs as "blob" files (named, typed arrays) that the parity tests and the
// golden-fixture generator read. TEST INFRASTRUCTURE ONLY: nothing in the
// product imports, links or executes this.
//
// Sub-commands (key=value arguments):
//   graph   spec=... out=...                 CSR, normalised adjacency, dataset arrays
//   chunks  spec=... K=.. seed=.. out=...    make_chunks + partition_vertices(K)
//   shuffle K=.. seed=.. epochs=.. out=...   shuffle_chunk_order for epochs 1..T
//   forward spec=... model=.. layers=.. hidden=.. seed=.. epoch=.. out=...
//                                            whole-graph forward+backward at one epoch
//                                            with init params (layer_forward/backward)
//   train   spec=... model=.. layers=.. hidden=.. S=.. K=.. chunk_seed=.. epochs=..
//           seed=.. dropout=.. fix_alpha=.. shuffle=.. sync=.. hist=.. mode=seq|pipe
//           out=...                           metrics + final params
//   save    spec=... dir=...                 save_dataset (reference writer)
//   epochs  spec=... model=.. layers=.. hidden=.. S=.. K=.. epochs=.. out=...
//                                            timed whole train_pipeline epochs (CPU baseline)
//   ckpt    model=.. layers=.. hidden=.. F=.. C=.. seed=.. lo=.. hi=.. path=.. out=...
//                                            save_stage_checkpoint of init_params(seed)
//   analytics in=EVENTS dir=DIR out=...      bubble_analysis of the trace in EVENTS (one
//                                            "worker kind chunk lo hi t0 t1" per line),
//                                            volume_* / crossover_report of fixed inputs,
//                                            and the reference writers' files in DIR
//
// Dataset spec strings:
//   er:N:P:GSEED:F:C:FSEED   generate_er (graph.cpp:119-156) + hashed features
//   sbm:B:BS:PIN:POUT:SEED   generate_sbm (dataset.cpp:147-191)
//   g8:F:C                   the test_helpers.hpp:28-50 toy graph
//   dir:PATH                 load_dataset (dataset.cpp:64-119)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gnnsim/analytics.hpp"
#include "gnnsim/engines.hpp"
#include "gnnsim/partition.hpp"

using namespace gnnsim;

namespace {

// ---- blob writer: [u32 nlen][name][u8 dtype][u8 ndim][u64 dims...][raw] ----
struct Blob {
    std::ofstream out;
    explicit Blob(const std::string& path) : out(path, std::ios::binary | std::ios::trunc) {
        if (!out) throw std::runtime_error("cannot write " + path);
        out.write("GPBLOB01", 8);
    }
    void put(const std::string& name, uint8_t dtype, const std::vector<uint64_t>& dims,
             const void* data, size_t bytes) {
        uint32_t n = uint32_t(name.size());
        out.write(reinterpret_cast<const char*>(&n), 4);
        out.write(name.data(), n);
        uint8_t nd = uint8_t(dims.size());
        out.write(reinterpret_cast<const char*>(&dtype), 1);
        out.write(reinterpret_cast<const char*>(&nd), 1);
        for (uint64_t d : dims) out.write(reinterpret_cast<const char*>(&d), 8);
        out.write(static_cast<const char*>(data), std::streamsize(bytes));
    }
    // dtype codes: 1=u8 2=u32 3=u64 4=f32 5=f64 6=i64
    void u8(const std::string& n, const std::vector<uint8_t>& v) { put(n, 1, {v.size()}, v.data(), v.size()); }
    void u32(const std::string& n, const std::vector<uint32_t>& v) { put(n, 2, {v.size()}, v.data(), v.size() * 4); }
    void u64(const std::string& n, const std::vector<uint64_t>& v) { put(n, 3, {v.size()}, v.data(), v.size() * 8); }
    void f32(const std::string& n, const std::vector<float>& v) { put(n, 4, {v.size()}, v.data(), v.size() * 4); }
    void f64(const std::string& n, const std::vector<double>& v) { put(n, 5, {v.size()}, v.data(), v.size() * 8); }
    void mat(const std::string& n, const MatF& m) {
        put(n, 4, {m.rows(), m.cols()}, m.data(), m.size() * 4);
    }
};

using Args = std::map<std::string, std::string>;

std::string arg(const Args& a, const std::string& k, const std::string& def = "") {
    auto it = a.find(k);
    if (it == a.end()) {
        if (def.empty()) throw std::invalid_argument("missing argument " + k);
        return def;
    }
    return it->second;
}
uint64_t argu(const Args& a, const std::string& k, const std::string& def = "") {
    return std::stoull(arg(a, k, def));
}
double argd(const Args& a, const std::string& k, const std::string& def = "") {
    return std::stod(arg(a, k, def));
}

std::vector<std::string> split(const std::string& s, char c) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string t;
    while (std::getline(ss, t, c)) out.push_back(t);
    return out;
}

// Synthetic node features / labels / split for generated graphs. The reference
// has no generator at these shapes; this definition is shared
// verbatim by the product (csrc/host/dataset.cpp) and the C oracle.
void fill_hashed_features(Dataset& d, uint32_t F, uint32_t C, uint64_t fseed) {
    const VertexId n = d.graph.num_vertices;
    d.features = MatF(n, F);
    for (uint64_t v = 0; v < n; ++v)
        for (uint64_t j = 0; j < F; ++j)
            d.features.at(v, j) = float(hash_unit(mix64(fseed, v * F + j)) * 2.0 - 1.0);
    d.num_classes = C;
    d.labels.resize(n);
    d.split.resize(n);
    for (uint64_t v = 0; v < n; ++v) {
        d.labels[v] = uint32_t(mix64(fseed, 0x4C42ull, v) % C);
        const uint64_t r = mix64(fseed, 0x5350ull, v) % 10;
        d.split[v] = r < 6 ? 1 : (r < 8 ? 2 : 3);
    }
}

Dataset make_dataset(const std::string& spec) {
    auto p = split(spec, ':');
    if (p.empty()) throw std::invalid_argument("empty spec");
    if (p[0] == "er") {
        if (p.size() != 7) throw std::invalid_argument("er:N:P:GSEED:F:C:FSEED");
        Dataset d;
        d.graph = generate_er(VertexId(std::stoul(p[1])), std::stod(p[2]), std::stoull(p[3]));
        fill_hashed_features(d, uint32_t(std::stoul(p[4])), uint32_t(std::stoul(p[5])),
                             std::stoull(p[6]));
        d.validate();
        return d;
    }
    if (p[0] == "sbm") {
        if (p.size() != 6) throw std::invalid_argument("sbm:B:BS:PIN:POUT:SEED");
        return generate_sbm(uint32_t(std::stoul(p[1])), uint32_t(std::stoul(p[2])),
                            std::stod(p[3]), std::stod(p[4]), std::stoull(p[5]));
    }
    if (p[0] == "g8") {
        // test_helpers.hpp:28-50
        const uint32_t F = p.size() > 1 ? uint32_t(std::stoul(p[1])) : 2;
        const uint32_t C = p.size() > 2 ? uint32_t(std::stoul(p[2])) : 2;
        Dataset d;
        d.graph = build_graph(8, {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {2, 5}});
        d.features = MatF(8, F);
        std::mt19937_64 eng(7);
        std::uniform_real_distribution<float> u(-1.f, 1.f);
        for (size_t i = 0; i < d.features.size(); ++i) d.features.data()[i] = u(eng);
        d.num_classes = C;
        d.labels.resize(8);
        for (int v = 0; v < 8; ++v) d.labels[v] = uint32_t(v) % C;
        d.split.assign(8, 1);
        d.split[6] = 2;
        d.split[7] = 3;
        return d;
    }
    if (p[0] == "dir") return load_dataset(spec.substr(4));
    throw std::invalid_argument("unknown spec kind " + p[0]);
}

ModelConfig model_from(const Args& a) {
    ModelConfig m;
    m.kind = parse_model_kind(arg(a, "model", "gcn"));
    m.layers = uint32_t(argu(a, "layers", "2"));
    m.hidden = uint32_t(argu(a, "hidden", "16"));
    m.dropout = argd(a, "dropout", "0.5");
    m.gcnii_alpha = argd(a, "alpha", "0.1");
    m.gcnii_lambda = argd(a, "lambda", "0.5");
    m.self_loops = argu(a, "self_loops", "1") != 0;
    return m;
}

void dump_params(Blob& b, const std::string& prefix, const std::vector<LayerParams<float>>& ps) {
    for (size_t l = 0; l < ps.size(); ++l) {
        b.mat(prefix + "W" + std::to_string(l), ps[l].weight);
        b.f32(prefix + "b" + std::to_string(l), ps[l].bias);
    }
}

void cmd_graph(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    Blob b(arg(a, "out"));
    b.u64("csr_offsets", d.graph.csr_offsets);
    b.u32("csr_neighbors", d.graph.csr_neighbors);
    b.u32("degrees", d.graph.degrees);
    b.u64("num_edges", {d.graph.num_edges});
    auto m = normalize_adjacency<float>(d.graph, argu(a, "self_loops", "1") != 0);
    b.u64("norm_offsets", m.offsets);
    b.u32("norm_cols", m.cols);
    b.f32("norm_vals", m.vals);
    b.mat("features", d.features);
    b.u32("labels", d.labels);
    b.u8("split", d.split);
    b.u32("num_classes", {d.num_classes});
}

void cmd_chunks(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    const uint32_t K = uint32_t(argu(a, "K"));
    const uint64_t seed = argu(a, "seed");
    Blob b(arg(a, "out"));
    ChunkPlan plan = make_chunks(d.graph, K, seed);
    b.u32("chunk_of", plan.chunk_of);
    Partition part = partition_vertices(d.graph, K, seed);
    b.u32("assignment", part.assignment);
    std::vector<uint64_t> bsizes;
    std::vector<uint32_t> bflat;
    for (const auto& bs : part.boundary_sets) {
        bsizes.push_back(bs.size());
        bflat.insert(bflat.end(), bs.begin(), bs.end());
    }
    b.u64("boundary_sizes", bsizes);
    b.u32("boundary_flat", bflat);
    b.u64("edge_cut", {part.edge_cut(d.graph)});
}

void cmd_shuffle(const Args& a) {
    ChunkPlan plan;
    plan.num_chunks = uint32_t(argu(a, "K"));
    const uint64_t seed = argu(a, "seed");
    const uint32_t T = uint32_t(argu(a, "epochs"));
    std::vector<uint32_t> all;
    for (uint32_t t = 1; t <= T; ++t) {
        auto o = shuffle_chunk_order(plan, t, seed);
        all.insert(all.end(), o.begin(), o.end());
    }
    Blob b(arg(a, "out"));
    b.u32("orders", all);
    std::vector<uint32_t> ranges;
    for (uint32_t L : {1u, 3u, 8u, 16u, 64u})
        for (uint32_t S = 1; S <= std::min(L, 8u); ++S) {
            auto sa = make_stage_assignment(L, S);
            for (auto [lo, hi] : sa.ranges) {
                ranges.push_back(L);
                ranges.push_back(S);
                ranges.push_back(lo);
                ranges.push_back(hi);
            }
        }
    b.u32("stage_ranges", ranges);
}

// Whole-graph forward + backward at epoch `epoch` with freshly initialised
// parameters, using the reference's whole-matrix ops (nn.hpp:297-361). This is
// exactly train_sequential's first epoch (engines_impl.hpp:226-283) with the
// per-layer activations exposed.
void cmd_forward(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    ModelConfig mc = model_from(a);
    const uint64_t seed = argu(a, "seed", "1");
    const uint64_t epoch = argu(a, "epoch", "1");
    auto specs = build_layer_specs(mc, d.num_features(), d.num_classes);
    auto params = init_params<float>(specs, seed);
    auto adj = build_adj_bundle<float>(d.graph, mc.self_loops);
    const uint32_t L = uint32_t(specs.size());
    const VertexId n = d.num_vertices();
    const bool needs_h0 = model_needs_h0(specs);
    // full=0: only the loss, parameter gradients and per-layer checksums (full-size graphs)
    const bool full = argu(a, "full", "1") != 0;
    Blob b(arg(a, "out"));
    if (full) dump_params(b, "init_", params);
    std::vector<ForwardCache<float>> caches;
    std::vector<DropMask<float>> masks;
    for (uint32_t l = 0; l < L; ++l) {
        masks.push_back(DropMask<float>::make(mc.dropout, seed, epoch, l, n, specs[l].in_dim));
        const MatF& src = l == 0 ? d.features : caches[l - 1].out;
        const MatF* h0 = needs_h0 && l > 0 ? &caches[0].out : nullptr;
        caches.push_back(layer_forward(specs[l], params[l], adj, src, h0, masks[l]));
        if (full) {
            b.mat("pre" + std::to_string(l), caches[l].pre);
            b.mat("h" + std::to_string(l), caches[l].out);
        }
    }
    // Loss head on the training rows, as train_sequential does.
    std::vector<uint8_t> train_mask = d.mask(Split::Train);
    auto loss = softmax_xent(caches[L - 1].out, d.labels, train_mask);
    b.f64("loss", {loss.loss});
    if (full) b.mat("grad_logits", loss.grad_logits);
    // Backward: reproduce train_sequential's loop (engines_impl.hpp:250-277),
    // dumping dz/dagg/grad_in per layer and param grads.
    std::vector<MatF> dz(L), dagg(L), dh(L);
    for (uint32_t l = 0; l < L; ++l) {
        dz[l] = MatF(n, specs[l].out_dim);
        dagg[l] = MatF(n, specs[l].k_in());
        dh[l] = MatF(n, specs[l].out_dim);
    }
    MatF dh0;
    if (needs_h0) dh0 = MatF(n, mc.hidden);
    dh[L - 1] = loss.grad_logits;
    for (int l = int(L) - 1; l >= 0; --l) {
        const auto& spec = specs[l];
        if (l == 0 && needs_h0)
            for (VertexId v = 0; v < n; ++v)
                for (uint32_t j = 0; j < mc.hidden; ++j) dh[0].at(v, j) += dh0.at(v, j);
        for (VertexId v = 0; v < n; ++v)
            kernel::backward_out_row(spec, params[l], dh[l].row(v), caches[l].out.row(v),
                                     dz[l].row(v), dagg[l].row(v),
                                     needs_h0 && spec.kind == LayerKind::Gcn2Conv ? dh0.row(v)
                                                                                  : nullptr);
        if (l > 0)
            for (VertexId u = 0; u < n; ++u)
                kernel::backward_prev_row(spec, adj, u,
                                          [&](VertexId v2) { return dagg[l].row(v2); },
                                          dagg[l].row(u), masks[l], dh[l - 1].row(u));
    }
    auto rows = std::vector<VertexId>(n);
    for (VertexId v = 0; v < n; ++v) rows[v] = v;
    for (uint32_t l = 0; l < L; ++l) {
        if (full) {
            b.mat("dz" + std::to_string(l), dz[l]);
            if (l > 0) b.mat("dagg" + std::to_string(l), dagg[l]);
            b.mat("dh" + std::to_string(l), dh[l]);
        } else {
            // fp64 column sums of the activations and gradients (size-independent checks)
            auto colsum = [](const MatF& m) {
                std::vector<double> s(m.cols(), 0.0);
                for (size_t r = 0; r < m.rows(); ++r)
                    for (size_t c = 0; c < m.cols(); ++c) s[c] += double(m.at(r, c));
                return s;
            };
            b.f64("sum_h" + std::to_string(l), colsum(caches[l].out));
            b.f64("sum_pre" + std::to_string(l), colsum(caches[l].pre));
            b.f64("sum_dz" + std::to_string(l), colsum(dz[l]));
        }
        auto g = param_grads_for_rows(specs[l], rows, caches[l].pre, dz[l]);
        b.mat("gW" + std::to_string(l), g.weight);
        b.f32("gb" + std::to_string(l), g.bias);
    }
    if (needs_h0 && full) b.mat("dh0", dh0);
}

void cmd_train(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    TrainOptions<float> opt;
    opt.model = model_from(a);
    opt.epochs = uint32_t(argu(a, "epochs", "1"));
    opt.seed = argu(a, "seed", "1");
    opt.optimizer.kind = arg(a, "optimizer", "adam") == "sgd" ? OptimizerKind::Sgd : OptimizerKind::Adam;
    opt.optimizer.lr = argd(a, "lr", "0.001");
    opt.staleness.shuffle_chunks = argu(a, "shuffle", "1") != 0;
    opt.staleness.fix_alpha = uint32_t(argu(a, "fix_alpha", "10"));
    opt.staleness.historical_gradients = argu(a, "hist", "0") != 0;
    opt.staleness.synchronous_mode = argu(a, "sync", "0") != 0;
    opt.fabric.mode = arg(a, "fabric", "det") == "conc" ? Fabric::Mode::Concurrent
                                                        : Fabric::Mode::Deterministic;
    // full-size pipelines fill for minutes before the last stage's first message arrives
    opt.fabric.watchdog_seconds = argd(a, "watchdog", "60");
    const std::string mode = arg(a, "mode", "pipe");
    TrainResult<float> res;
    std::vector<uint32_t> chunk_of;
    const auto t0 = std::chrono::steady_clock::now();
    if (mode == "seq") {
        res = train_sequential(d, opt);
    } else if (mode == "graph") {
        Partition part = partition_vertices(d.graph, uint32_t(argu(a, "G", "2")), argu(a, "part_seed", "1"));
        res = train_graph_parallel(d, part, opt);
    } else {
        const uint32_t S = uint32_t(argu(a, "S", "1"));
        const uint32_t K = uint32_t(argu(a, "K", "1"));
        const uint32_t G = uint32_t(argu(a, "G", "1"));
        ChunkPlan plan = K == 1 ? chunk_plan_from_assignment(d.num_vertices(),
                                                             std::vector<uint32_t>(d.num_vertices(), 0))
                                : make_chunks(d.graph, K, argu(a, "chunk_seed", "1"));
        chunk_of = plan.chunk_of;
        const uint32_t L = uint32_t(build_layer_specs(opt.model, d.num_features(), d.num_classes).size());
        auto sa = make_stage_assignment(L, S);
        if (G == 1) {
            res = train_pipeline(d, plan, sa, opt);
        } else {
            Partition part = partition_vertices(d.graph, G, argu(a, "part_seed", "1"));
            GroupMap gmap = assign_groups(S * G, 4, S, G);
            res = train_hybrid(d, part, plan, sa, gmap, opt);
        }
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    Blob b(arg(a, "out"));
    std::vector<double> mt;
    std::vector<uint64_t> comm;
    for (const auto& m : res.metrics) {
        mt.insert(mt.end(), {double(m.epoch), m.train_loss, m.train_acc, m.val_acc, m.test_acc});
        comm.insert(comm.end(), {m.comm_bytes_graph, m.comm_bytes_pipeline, m.comm_bytes_weightsync});
    }
    b.f64("metrics", mt);
    b.u64("comm", comm);
    b.u32("chunk_of", chunk_of);
    b.f64("seconds", {secs});
    b.u64("peak_buffer_bytes", {res.peak_buffer_bytes});
    dump_params(b, "", res.params);
}

// save_stage_checkpoint of init_params(seed) for layers [lo, hi) (nn.hpp:511-531).
void cmd_ckpt(const Args& a) {
    const ModelConfig m = model_from(a);
    const auto specs = build_layer_specs(m, uint32_t(std::stoul(arg(a, "F"))), uint32_t(std::stoul(arg(a, "C"))));
    const auto params = init_params<float>(specs, std::stoull(arg(a, "seed", "1")));
    save_stage_checkpoint(arg(a, "path"), specs, params, std::stoul(arg(a, "lo", "0")),
                          std::stoul(arg(a, "hi", std::to_string(specs.size()))));
    Blob b(arg(a, "out"));
    b.u64("num_layers", {specs.size()});
}

// save_assignment of make_chunks(K) and partition_vertices(K) (partition.cpp:250-256)
void cmd_assign(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    const uint32_t K = uint32_t(argu(a, "K"));
    const uint64_t seed = argu(a, "seed");
    ChunkPlan plan = make_chunks(d.graph, K, seed);
    save_assignment(arg(a, "dir") + "/chunks.txt", plan.num_chunks, plan.chunk_of);
    Partition p = partition_vertices(d.graph, K, seed);
    save_assignment(arg(a, "dir") + "/parts.txt", p.num_parts, p.assignment);
    Blob b(arg(a, "out"));
    b.u32("chunk_of", plan.chunk_of);
}

void cmd_save(const Args& a) {
    Dataset d = make_dataset(arg(a, "spec"));
    save_dataset(d, arg(a, "dir"));
}

// CPU baseline (bench.py --impl reference and cpu_baseline): whole epochs of the
// reference's own train_pipeline<float> (engines_impl.hpp:911-920) through its
// public API, Fabric::Mode::Concurrent (one OS thread per stage worker,
// fabric.cpp:395-422). The call's own setup (adjacency bundle, feature cast,
// stash allocation) is timed by an epochs=0 call and subtracted; dataset
// generation and make_chunks are timed separately.
void cmd_epochs(const Args& a) {
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
    auto t0 = clk::now();
    Dataset d = make_dataset(arg(a, "spec"));
    const double gen_s = secs(t0);
    const uint32_t S = uint32_t(argu(a, "S", "1"));
    const uint32_t K = uint32_t(argu(a, "K", "1"));
    t0 = clk::now();
    ChunkPlan plan = K == 1 ? chunk_plan_from_assignment(d.num_vertices(), std::vector<uint32_t>(d.num_vertices(), 0))
                            : make_chunks(d.graph, K, argu(a, "chunk_seed", "1"));
    const double chunk_s = secs(t0);
    TrainOptions<float> opt;
    opt.model = model_from(a);
    opt.seed = argu(a, "seed", "1");
    opt.fabric.mode = Fabric::Mode::Concurrent;
    // a deep stage's first message can take minutes at full size: the reference's 60 s fabric
    // watchdog would abort the timing run
    opt.fabric.watchdog_seconds = argd(a, "watchdog", "36000");
    const uint32_t L = uint32_t(build_layer_specs(opt.model, d.num_features(), d.num_classes).size());
    const auto sa = make_stage_assignment(L, S);
    opt.epochs = 0;
    t0 = clk::now();
    (void)train_pipeline(d, plan, sa, opt);
    const double setup_s = secs(t0);
    opt.epochs = uint32_t(argu(a, "epochs", "1"));
    t0 = clk::now();
    const TrainResult<float> res = train_pipeline(d, plan, sa, opt);
    const double total_s = secs(t0);
    Blob b(arg(a, "out"));
    b.f64("gen_s", {gen_s});
    b.f64("chunk_s", {chunk_s});
    b.f64("setup_s", {setup_s});
    b.f64("total_s", {total_s});
    b.f64("epoch_s", {(total_s - setup_s) / double(opt.epochs)});
    b.f64("loss", {res.metrics.empty() ? 0.0 : res.metrics.back().train_loss});
    b.u64("threads", {S});
}

void cmd_analytics(const Args& a) {
    std::ifstream in(arg(a, "in"));
    if (!in) throw std::runtime_error("cannot read events");
    std::vector<TraceEvent> tr;
    uint32_t w, k;
    int32_t c, lo, hi;
    double t0, t1;
    while (in >> w >> k >> c >> lo >> hi >> t0 >> t1) tr.push_back({w, t0, t1, TraceEvent::Kind(k), c, lo, hi});
    const std::string dir = arg(a, "dir");
    Blob b(arg(a, "out"));
    const BubbleReport br = bubble_analysis(tr);
    b.f64("bubble", {br.measured_bubble, br.ideal_bubble, double(br.stages), double(br.chunks), br.span});
    write_trace_jsonl(dir + "/trace.jsonl", tr);
    // volumes / crossover on the paper-shaped inputs (Reddit: N, L, H; alpha values)
    std::vector<double> vols;
    std::string cross;
    for (double alpha : {0.0, 0.35, 2.5}) {
        CommModelInput g, p, h;
        g.n = p.n = h.n = 232965;
        g.layers = p.layers = h.layers = 64;
        g.hidden = p.hidden = h.hidden = 100;
        g.ways = 8;
        g.alpha = alpha;
        p.stages = 8;
        p.vecs = 2;
        h.stages = 4;
        h.ways = 2;
        h.alpha = alpha / 3;
        h.vecs = 2;
        const CrossoverReport r = crossover_report(g, p, h);
        vols.insert(vols.end(), {r.bytes_graph, r.bytes_pipeline, r.bytes_hybrid});
        cross += r.winner + "|" + (r.tie ? "tie" : "-") + "|";
        for (const auto& o : r.ordering) cross += o + ",";
        for (const auto& q : r.inequalities) cross += "|" + q;
        cross += "\n";
    }
    b.f64("volumes", vols);
    b.u8("crossover", std::vector<uint8_t>(cross.begin(), cross.end()));
    // writers: a fixed ledger / metrics / compare set
    std::vector<CommReportRow> rows;
    for (uint32_t e = 0; e < 3; ++e)
        for (uint32_t t = 0; t < kNumTags; ++t)
            for (uint32_t l = 0; l < 2; ++l) {
                const uint64_t bytes = ((e + 1) * 1000003ull * (t + 1) + l * 77) % 5 == 0 ? 0 : (e + 1) * 123456789ull * (t + 1) + l;
                if (bytes) rows.push_back({e, MsgTag(t), LinkClass(l), bytes, double(bytes) / double(1ull << 30)});
            }
    write_comm_report_csv(dir + "/comm_report.csv", rows);
    std::vector<EpochMetrics> ms;
    for (uint32_t e = 1; e <= 3; ++e) {
        EpochMetrics m;
        m.epoch = e;
        m.train_loss = 3.7 / e;
        m.train_acc = 0.1 * e;
        m.val_acc = 0.09 * e;
        m.test_acc = 0.08 * e;
        m.comm_bytes_graph = 11 * e;
        m.comm_bytes_pipeline = 373000000ull * e;
        m.comm_bytes_weightsync = 7 * e;
        m.wall_time_s = 0.4 + e * 1e-3;
        m.bubble_fraction = 0.18 / e;
        ms.push_back(m);
    }
    write_metrics_csv(dir + "/metrics.csv", ms);
    std::vector<CompareRow> cr = {{"pipeline", 232965, 64, 100, 8, 1, 0, 2, 2.6e9, 2600000123ull, 4.7e-8},
                                  {"graph", 1000, 4, 16, 1, 3, 0.25, 1, 128000, 127990, 7.8125e-5}};
    write_compare_csv(dir + "/compare.csv", cr);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_driver <cmd> key=value...\n");
        return 2;
    }
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        auto eq = s.find('=');
        if (eq == std::string::npos) {
            std::fprintf(stderr, "bad argument %s\n", argv[i]);
            return 2;
        }
        a[s.substr(0, eq)] = s.substr(eq + 1);
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "graph") cmd_graph(a);
        else if (cmd == "chunks") cmd_chunks(a);
        else if (cmd == "shuffle") cmd_shuffle(a);
        else if (cmd == "forward") cmd_forward(a);
        else if (cmd == "train") cmd_train(a);
        else if (cmd == "save") cmd_save(a);
        else if (cmd == "assign") cmd_assign(a);
        else if (cmd == "epochs") cmd_epochs(a);
        else if (cmd == "analytics") cmd_analytics(a);
        else if (cmd == "ckpt") cmd_ckpt(a);
        else {
            std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
            return 2;
        }
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "invalid argument: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
    return 0;
}

// gs_* — flat C wrappers over the C++ API (include/gnnpipe.h, host section).
// Exceptions map to the gp_status codes of the reference's error classes.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "gnnsim_b200.hpp"

using namespace gnnsim;

struct gs_dataset {
    Dataset d;
};
struct gs_result {
    TrainResult<float> r;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return GP_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return GP_EINVAL;
    } catch (const NumericError& e) {
        g_err = e.what();
        return GP_ENUMERIC;
    } catch (const FabricError& e) {
        g_err = e.what();
        return GP_EFABRIC;
    } catch (const GpError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GP_ERUNTIME;
    }
}

ModelConfig model_of(const gs_model_config* m) {
    if (!m) throw std::invalid_argument("null model config");
    ModelConfig c;
    switch (m->kind) {
        case 0: c.kind = ModelKind::GCN; break;
        case 1: c.kind = ModelKind::Sage; break;
        case 2: c.kind = ModelKind::GCNII; break;
        default: throw std::invalid_argument("unknown model kind");
    }
    c.layers = m->layers;
    c.hidden = m->hidden;
    c.dropout = m->dropout;
    c.gcnii_alpha = m->gcnii_alpha;
    c.gcnii_lambda = m->gcnii_lambda;
    c.self_loops = m->self_loops != 0;
    return c;
}

TrainOptions<float> options_of(const gs_train_options* o) {
    if (!o) throw std::invalid_argument("null train options");
    TrainOptions<float> t;
    t.model = model_of(&o->model);
    t.optimizer.kind = o->optimizer == 1 ? OptimizerKind::Sgd : OptimizerKind::Adam;
    t.optimizer.lr = o->lr;
    t.optimizer.beta1 = o->beta1;
    t.optimizer.beta2 = o->beta2;
    t.optimizer.eps = o->eps;
    t.epochs = o->epochs;
    t.seed = o->seed;
    t.staleness.shuffle_chunks = o->shuffle_chunks != 0;
    t.staleness.fix_alpha = o->fix_alpha;
    t.staleness.historical_gradients = o->historical_gradients != 0;
    t.staleness.synchronous_mode = o->synchronous_mode != 0;
    t.device = o->device;
    t.profile = o->profile != 0;
    t.fabric.collect_trace = o->collect_trace != 0;
    return t;
}

// options + the resume state named by o->resume_path (shapes from the dataset)
TrainOptions<float> options_for(const gs_train_options* o, const Dataset& d) {
    TrainOptions<float> t = options_of(o);
    t.keep_history = o->save_state_path && *o->save_state_path;  // a saved state resumes exactly
    if (o->resume_path && *o->resume_path)
        t.resume = std::make_shared<TrainState>(
            load_train_state(o->resume_path, build_layer_specs(t.model, d.num_features(), d.num_classes)));
    return t;
}

gs_result* finish(std::unique_ptr<gs_result> own, const gs_train_options* o) {
    if (o->save_state_path && *o->save_state_path) save_train_state(o->save_state_path, own->r.final_state);
    return own.release();
}

CommModelInput cmi(const gs_comm_model_input* in) {
    if (!in) throw std::invalid_argument("null input");
    CommModelInput c;
    c.n = in->n;
    c.layers = in->layers;
    c.hidden = in->hidden;
    c.stages = in->stages;
    c.ways = in->ways;
    c.alpha = in->alpha;
    c.vecs = in->vecs;
    c.bytes_per_value = in->bytes_per_value;
    return c;
}
}  // namespace

extern "C" {

const char* gs_last_error(void) { return g_err.c_str(); }

int gs_dataset_from_edges(uint32_t n, const uint32_t* uv, uint64_t m, const float* x, uint32_t F,
                          const uint32_t* labels, uint32_t C, const uint8_t* split, gs_dataset** out) {
    return guarded([&]() {
        auto* h = new gs_dataset();
        std::unique_ptr<gs_dataset> own(h);
        std::vector<std::pair<VertexId, VertexId>> e(m);
        for (uint64_t i = 0; i < m; ++i) e[i] = {uv[2 * i], uv[2 * i + 1]};
        h->d.graph = build_graph(n, std::move(e));
        h->d.features = MatF(n, F);
        if (x && F) std::memcpy(h->d.features.data(), x, size_t(n) * F * 4);
        h->d.num_classes = C;
        h->d.labels.assign(labels, labels + n);
        h->d.split.assign(split, split + n);
        h->d.validate();
        *out = own.release();
    });
}

int gs_dataset_synthetic_er(uint32_t n, double p, uint64_t gseed, uint32_t F, uint32_t C, uint64_t fseed,
                            gs_dataset** out) {
    return guarded([&]() {
        auto own = std::make_unique<gs_dataset>();
        own->d = synthetic_er_dataset(n, p, gseed, F, C, fseed);
        *out = own.release();
    });
}

int gs_dataset_load(const char* dir, gs_dataset** out) {
    return guarded([&]() {
        auto own = std::make_unique<gs_dataset>();
        own->d = load_dataset(dir);
        *out = own.release();
    });
}

int gs_dataset_save(const gs_dataset* d, const char* dir) {
    return guarded([&]() { save_dataset(d->d, dir); });
}

void gs_dataset_free(gs_dataset* d) { delete d; }

int gs_dataset_shape(const gs_dataset* d, uint32_t* n, uint64_t* m, uint32_t* F, uint32_t* C) {
    return guarded([&]() {
        if (n) *n = d->d.graph.num_vertices;
        if (m) *m = d->d.graph.num_edges;
        if (F) *F = d->d.num_features();
        if (C) *C = d->d.num_classes;
    });
}

int gs_dataset_graph(const gs_dataset* d, uint64_t* offsets, uint32_t* neighbors, uint32_t* degrees) {
    return guarded([&]() {
        const Graph& g = d->d.graph;
        if (offsets) std::memcpy(offsets, g.csr_offsets.data(), g.csr_offsets.size() * 8);
        if (neighbors) std::memcpy(neighbors, g.csr_neighbors.data(), g.csr_neighbors.size() * 4);
        if (degrees) std::memcpy(degrees, g.degrees.data(), g.degrees.size() * 4);
    });
}

int gs_dataset_arrays(const gs_dataset* d, float* x, uint32_t* labels, uint8_t* split) {
    return guarded([&]() {
        if (x) std::memcpy(x, d->d.features.data(), d->d.features.size() * 4);
        if (labels) std::memcpy(labels, d->d.labels.data(), d->d.labels.size() * 4);
        if (split) std::memcpy(split, d->d.split.data(), d->d.split.size());
    });
}

int gs_normalize_adjacency(const gs_dataset* d, int self_loops, uint64_t* offsets, uint32_t* cols, float* vals) {
    return guarded([&]() {
        auto m = normalize_adjacency<float>(d->d.graph, self_loops != 0);
        if (offsets) std::memcpy(offsets, m.offsets.data(), m.offsets.size() * 8);
        if (cols) std::memcpy(cols, m.cols.data(), m.cols.size() * 4);
        if (vals) std::memcpy(vals, m.vals.data(), m.vals.size() * 4);
    });
}

int gs_make_chunks(const gs_dataset* d, uint32_t K, uint64_t seed, uint32_t* chunk_of) {
    return guarded([&]() {
        auto plan = make_chunks(d->d.graph, K, seed);
        std::memcpy(chunk_of, plan.chunk_of.data(), plan.chunk_of.size() * 4);
    });
}

int gs_partition_vertices(const gs_dataset* d, uint32_t parts, uint64_t seed, uint32_t* assignment,
                          uint64_t* edge_cut, uint64_t* boundary_total) {
    return guarded([&]() {
        auto p = partition_vertices(d->d.graph, parts, seed);
        if (assignment) std::memcpy(assignment, p.assignment.data(), p.assignment.size() * 4);
        if (edge_cut) *edge_cut = p.edge_cut(d->d.graph);
        if (boundary_total) *boundary_total = p.boundary_total();
    });
}

int gs_shuffle_chunk_order(uint32_t K, uint64_t epoch, uint64_t seed, uint32_t* order) {
    return guarded([&]() {
        ChunkPlan plan;
        plan.num_chunks = K;
        auto o = shuffle_chunk_order(plan, epoch, seed);
        std::memcpy(order, o.data(), o.size() * 4);
    });
}

int gs_save_assignment(const char* path, uint32_t num_parts, const uint32_t* assignment, uint64_t n) {
    return guarded([&]() {
        if (!path || (n && !assignment)) throw std::invalid_argument("null argument");
        save_assignment(path, num_parts, std::vector<uint32_t>(assignment, assignment + n));
    });
}

int gs_load_assignment(const char* path, uint32_t* num_parts, uint32_t* assignment, uint64_t cap, uint64_t* n) {
    return guarded([&]() {
        if (!path) throw std::invalid_argument("null path");
        auto [parts, a] = load_assignment(path);
        if (num_parts) *num_parts = parts;
        if (n) *n = a.size();
        if (assignment) {
            if (cap < a.size()) throw std::invalid_argument("gs_load_assignment: buffer too small");
            std::memcpy(assignment, a.data(), a.size() * 4);
        }
    });
}

int gs_make_stage_assignment(uint32_t layers, uint32_t stages, uint32_t* ranges) {
    return guarded([&]() {
        auto sa = make_stage_assignment(layers, stages);
        for (uint32_t s = 0; s < stages; ++s) {
            ranges[2 * s] = sa.begin(s);
            ranges[2 * s + 1] = sa.end(s);
        }
    });
}

int gs_num_layers(const gs_model_config* m, uint32_t* L) {
    return guarded([&]() { *L = uint32_t(build_layer_specs(model_of(m), 1, 1).size()); });
}

int gs_build_layer_specs(const gs_model_config* m, uint32_t F, uint32_t C, gp_layer_spec* out) {
    return guarded([&]() {
        auto specs = build_layer_specs(model_of(m), F, C);
        for (size_t l = 0; l < specs.size(); ++l) {
            out[l].kind = uint32_t(specs[l].kind);
            out[l].in_dim = specs[l].in_dim;
            out[l].out_dim = specs[l].out_dim;
            out[l].relu = specs[l].relu;
            out[l].alpha = specs[l].alpha;
            out[l].beta = specs[l].beta;
        }
    });
}

int gs_init_params(const gs_model_config* m, uint32_t F, uint32_t C, uint64_t seed, float* flat) {
    return guarded([&]() {
        auto specs = build_layer_specs(model_of(m), F, C);
        auto ps = init_params<float>(specs, seed);
        size_t at = 0;
        for (const auto& p : ps) {
            std::memcpy(flat + at, p.weight.data(), p.weight.size() * 4);
            at += p.weight.size();
            std::memcpy(flat + at, p.bias.data(), p.bias.size() * 4);
            at += p.bias.size();
        }
    });
}

int gs_train_pipeline(const gs_dataset* d, const uint32_t* chunk_of, uint32_t K, uint32_t S,
                      const gs_train_options* o, gs_result** out) {
    return guarded([&]() {
        TrainOptions<float> opt = options_for(o, d->d);
        const uint32_t L = uint32_t(build_layer_specs(opt.model, d->d.num_features(), d->d.num_classes).size());
        ChunkPlan plan = chunk_plan_from_assignment(d->d.num_vertices(),
                                                    std::vector<uint32_t>(chunk_of, chunk_of + d->d.num_vertices()));
        if (plan.num_chunks != K) throw std::invalid_argument("chunk_of does not use exactly K chunks");
        auto own = std::make_unique<gs_result>();
        own->r = train_pipeline<float>(d->d, plan, make_stage_assignment(L, S), opt);
        *out = finish(std::move(own), o);
    });
}

int gs_train_hybrid(const gs_dataset* d, const uint32_t* part_of, const uint32_t* chunk_of, uint32_t K, uint32_t S,
                    const gs_train_options* o, gs_result** out) {
    return guarded([&]() {
        TrainOptions<float> opt = options_for(o, d->d);
        const VertexId n = d->d.num_vertices();
        const uint32_t L = uint32_t(build_layer_specs(opt.model, d->d.num_features(), d->d.num_classes).size());
        Partition part = partition_from_assignment(d->d.graph, std::vector<uint32_t>(part_of, part_of + n));
        ChunkPlan plan = chunk_plan_from_assignment(n, std::vector<uint32_t>(chunk_of, chunk_of + n));
        if (plan.num_chunks != K) throw std::invalid_argument("chunk_of does not use exactly K chunks");
        const uint32_t G = part.num_parts;
        GroupMap gmap = assign_groups(S * G, 4, S, G);
        auto own = std::make_unique<gs_result>();
        own->r = train_hybrid<float>(d->d, part, plan, make_stage_assignment(L, S), gmap, opt);
        *out = finish(std::move(own), o);
    });
}

int gs_train_graph_parallel(const gs_dataset* d, const uint32_t* part_of, const gs_train_options* o,
                            gs_result** out) {
    return guarded([&]() {
        const VertexId n = d->d.num_vertices();
        Partition part = partition_from_assignment(d->d.graph, std::vector<uint32_t>(part_of, part_of + n));
        auto own = std::make_unique<gs_result>();
        own->r = train_graph_parallel<float>(d->d, part, options_for(o, d->d));
        *out = finish(std::move(own), o);
    });
}

int gs_train_sequential(const gs_dataset* d, const gs_train_options* o, gs_result** out) {
    return guarded([&]() {
        auto own = std::make_unique<gs_result>();
        own->r = train_sequential<float>(d->d, options_for(o, d->d));
        *out = finish(std::move(own), o);
    });
}

int gs_result_metrics(const gs_result* r, uint32_t* epochs, double* metrics, uint64_t* comm) {
    return guarded([&]() {
        if (epochs) *epochs = uint32_t(r->r.metrics.size());
        for (size_t t = 0; t < r->r.metrics.size(); ++t) {
            const auto& m = r->r.metrics[t];
            if (metrics) {
                double* row = metrics + 7 * t;
                row[0] = m.epoch;
                row[1] = m.train_loss;
                row[2] = m.train_acc;
                row[3] = m.val_acc;
                row[4] = m.test_acc;
                row[5] = m.wall_time_s;
                row[6] = m.bubble_fraction;
            }
            if (comm) {
                comm[3 * t] = m.comm_bytes_graph;
                comm[3 * t + 1] = m.comm_bytes_pipeline;
                comm[3 * t + 2] = m.comm_bytes_weightsync;
            }
        }
    });
}

int gs_result_params(const gs_result* r, float* flat) {
    return guarded([&]() {
        size_t at = 0;
        for (const auto& p : r->r.params) {
            std::memcpy(flat + at, p.weight.data(), p.weight.size() * 4);
            at += p.weight.size();
            std::memcpy(flat + at, p.bias.data(), p.bias.size() * 4);
            at += p.bias.size();
        }
    });
}

int gs_result_profile(const gs_result* r, gp_profile* out) {
    return guarded([&]() { *out = r->r.profile; });
}

int gs_result_trace(const gs_result* r, gs_trace_event* out, uint64_t cap, uint64_t* count) {
    return guarded([&]() {
        const auto& tr = r->r.trace;
        if (count) *count = tr.size();
        for (uint64_t i = 0; out && i < std::min<uint64_t>(cap, tr.size()); ++i) {
            const auto& e = tr[i];
            out[i] = gs_trace_event{e.worker, uint32_t(e.kind), e.chunk, e.layer_lo, e.layer_hi, 0u, e.t_start, e.t_end};
        }
    });
}

int gs_result_ledger(const gs_result* r, uint64_t* out) {
    return guarded([&]() {
        for (size_t t = 0; t < r->r.comm.size(); ++t)
            for (uint32_t tag = 0; tag < kNumTags; ++tag)
                for (uint32_t l = 0; l < 2; ++l) out[(t * kNumTags + tag) * 2 + l] = r->r.comm[t].by_tag_link[tag][l];
    });
}

namespace {
std::vector<TraceEvent> trace_of(const gs_trace_event* ev, uint64_t n) {
    if (n && !ev) throw std::invalid_argument("null trace");
    std::vector<TraceEvent> v(n);
    for (uint64_t i = 0; i < n; ++i) {
        if (ev[i].kind > 3) throw std::invalid_argument("unknown trace event kind");
        v[i] = TraceEvent{ev[i].worker, ev[i].t_start, ev[i].t_end, TraceEvent::Kind(ev[i].kind), ev[i].chunk,
                          ev[i].layer_lo, ev[i].layer_hi};
    }
    return v;
}
}  // namespace

int gs_write_metrics_csv(const char* path, const double* metrics, const uint64_t* comm, uint32_t epochs) {
    return guarded([&]() {
        if (!path || (epochs && (!metrics || !comm))) throw std::invalid_argument("null argument");
        std::vector<EpochMetrics> m(epochs);
        for (uint32_t t = 0; t < epochs; ++t) {
            const double* row = metrics + 7 * size_t(t);
            m[t].epoch = uint32_t(row[0]);
            m[t].train_loss = row[1];
            m[t].train_acc = row[2];
            m[t].val_acc = row[3];
            m[t].test_acc = row[4];
            m[t].wall_time_s = row[5];
            m[t].bubble_fraction = row[6];
            m[t].comm_bytes_graph = comm[3 * size_t(t)];
            m[t].comm_bytes_pipeline = comm[3 * size_t(t) + 1];
            m[t].comm_bytes_weightsync = comm[3 * size_t(t) + 2];
        }
        write_metrics_csv(path, m);
    });
}

int gs_write_trace_jsonl(const char* path, const gs_trace_event* events, uint64_t n) {
    return guarded([&]() {
        if (!path) throw std::invalid_argument("null path");
        write_trace_jsonl(path, trace_of(events, n));
    });
}

int gs_write_comm_report_csv(const char* path, const uint64_t* ledger, uint32_t epochs) {
    return guarded([&]() {
        if (!path || (epochs && !ledger)) throw std::invalid_argument("null argument");
        std::vector<CommReportRow> rows;
        for (uint32_t t = 0; t < epochs; ++t) {
            EpochComm e;
            for (uint32_t tag = 0; tag < kNumTags; ++tag)
                for (uint32_t l = 0; l < 2; ++l) e.by_tag_link[tag][l] = ledger[(size_t(t) * kNumTags + tag) * 2 + l];
            for (const auto& r : ledger_report(e, t)) rows.push_back(r);
        }
        write_comm_report_csv(path, rows);
    });
}

int gs_bubble_analysis(const gs_trace_event* events, uint64_t n, gs_bubble_report* out) {
    return guarded([&]() {
        if (!out) throw std::invalid_argument("null output");
        const BubbleReport b = bubble_analysis(trace_of(events, n));
        *out = gs_bubble_report{b.measured_bubble, b.ideal_bubble, b.stages, b.chunks, b.span};
    });
}

int gs_comm_volumes(const gs_comm_model_input* in, double* graph, double* pipeline, double* hybrid) {
    return guarded([&]() {
        const CommModelInput c = cmi(in);
        if (graph) *graph = volume_graph(c);
        if (pipeline) *pipeline = volume_pipeline(c);
        if (hybrid) *hybrid = volume_hybrid(c);
    });
}

int gs_crossover_report(const gs_comm_model_input* g, const gs_comm_model_input* p, const gs_comm_model_input* h,
                        double* bytes, char* text, uint64_t cap) {
    return guarded([&]() {
        const CrossoverReport r = crossover_report(cmi(g), cmi(p), cmi(h));
        if (bytes) {
            bytes[0] = r.bytes_graph;
            bytes[1] = r.bytes_pipeline;
            bytes[2] = r.bytes_hybrid;
        }
        std::string t = r.winner + "\n";
        for (size_t i = 0; i < r.ordering.size(); ++i) t += (i ? "," : "") + r.ordering[i];
        t += std::string("\n") + (r.tie ? "1" : "0");
        for (const auto& q : r.inequalities) t += "\n" + q;
        if (text && cap) {
            const size_t m = std::min<size_t>(cap - 1, t.size());
            std::memcpy(text, t.data(), m);
            text[m] = 0;
        }
    });
}

int gs_write_compare_csv(const char* path, const char* modes, const double* vals, const uint64_t* measured,
                         uint64_t n) {
    return guarded([&]() {
        if (!path || (n && (!modes || !vals || !measured))) throw std::invalid_argument("null argument");
        std::vector<CompareRow> rows;
        std::string all(modes ? modes : ""), cur;
        std::vector<std::string> names;
        for (char ch : all) {
            if (ch == '\n') names.push_back(cur), cur.clear();
            else cur += ch;
        }
        names.push_back(cur);
        if (names.size() < n) throw std::invalid_argument("fewer mode names than rows");
        for (uint64_t i = 0; i < n; ++i) {
            const double* v = vals + 9 * i;
            rows.push_back({names[i], v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], measured[i], v[8]});
        }
        write_compare_csv(path, rows);
    });
}

int gs_save_stage_checkpoint(const char* path, const gs_model_config* m, uint32_t F, uint32_t C, const float* flat,
                             uint32_t lo, uint32_t hi) {
    return guarded([&]() {
        if (!path || !flat) throw std::invalid_argument("null argument");
        const auto specs = build_layer_specs(model_of(m), F, C);
        if (lo >= hi || hi > specs.size()) throw std::invalid_argument("bad layer range");
        std::vector<LayerParams<float>> params(specs.size());
        size_t at = 0;
        for (size_t l = 0; l < specs.size(); ++l) {
            params[l].weight = MatF(specs[l].k_in(), specs[l].out_dim);
            std::memcpy(params[l].weight.data(), flat + at, params[l].weight.size() * 4);
            at += params[l].weight.size();
            if (specs[l].has_bias()) {
                params[l].bias.assign(flat + at, flat + at + specs[l].out_dim);
                at += specs[l].out_dim;
            }
        }
        save_stage_checkpoint(path, specs, params, lo, hi);
    });
}

int gs_load_checkpoint(const char* path, char* names, uint64_t names_cap, uint64_t* shapes, float* data,
                       uint64_t* n_tensors, uint64_t* n_floats) {
    return guarded([&]() {
        if (!path) throw std::invalid_argument("null path");
        const auto ts = load_checkpoint(path);
        std::string all;
        uint64_t floats = 0;
        for (size_t i = 0; i < ts.size(); ++i) {
            all += (i ? "\n" : "") + ts[i].name;
            if (shapes) {
                shapes[2 * i] = ts[i].rows;
                shapes[2 * i + 1] = ts[i].cols;
            }
            if (data) std::memcpy(data + floats, ts[i].data.data(), ts[i].data.size() * 4);
            floats += ts[i].data.size();
        }
        if (n_tensors) *n_tensors = ts.size();
        if (n_floats) *n_floats = floats;
        if (names && names_cap) {
            if (all.size() + 1 > names_cap)
                throw std::invalid_argument("gs_load_checkpoint: names buffer needs " + std::to_string(all.size() + 1) +
                                            " bytes (gs_checkpoint_names_bytes)");
            std::memcpy(names, all.data(), all.size());
            names[all.size()] = 0;
        }
    });
}

int gs_checkpoint_names_bytes(const char* path, uint64_t* bytes) {
    return guarded([&]() {
        if (!path || !bytes) throw std::invalid_argument("null argument");
        uint64_t b = 1;
        for (const auto& t : load_checkpoint(path)) b += t.name.size() + 1;
        *bytes = b;
    });
}

int gs_result_peak_bytes(const gs_result* r, uint64_t* out) {
    return guarded([&]() { *out = r->r.peak_buffer_bytes; });
}

void gs_result_free(gs_result* r) { delete r; }

}  // extern "C"

// gnnsim_b200.hpp — C++ API of the B200 engine, source-compatible with the
// reference's public surface for the chunk-pipelined training path
// (proj/include/gnnsim/{graph,dataset,partition,nn,engines}.hpp), so a caller
// of gnnsim::train_pipeline<float> (e.g. proj/tools/gnnsim.cpp:293) can link
// this library instead. Host preprocessing (CSR, normalisation, chunking,
// schedule, init) is bit-exact with the reference; the trainers run every
// per-row kernel on the GPU through the gp_* C-ABI (include/gnnpipe.h).
//
// Only T = float is provided for the trainers (the GPU computes in fp32);
// T = double remains a CPU-oracle concern.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <span>
#include <stdexcept>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "gnnpipe.h"

namespace gnnsim {

using VertexId = uint32_t;

// ---------------------------------------------------------------- randomness
// rng.hpp:9-38 — splitmix64 finaliser and its keyed variants.
inline uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) { return mix64(mix64(a) ^ b); }
inline uint64_t mix64(uint64_t a, uint64_t b, uint64_t c) { return mix64(mix64(a, b) ^ c); }
inline uint64_t mix64(uint64_t a, uint64_t b, uint64_t c, uint64_t d) { return mix64(mix64(a, b, c) ^ d); }
inline double hash_unit(uint64_t h) { return double(h >> 11) * 0x1.0p-53; }
inline std::mt19937_64 make_engine(uint64_t seed) { return std::mt19937_64(mix64(seed)); }
inline std::mt19937_64 make_engine(uint64_t seed, uint64_t stream) {
    return std::mt19937_64(mix64(seed, stream));
}

// ---------------------------------------------------------------- dense rows
template <typename T>
class Mat {
  public:
    Mat() = default;
    Mat(size_t r, size_t c) : r_(r), c_(c), v_(r * c, T{0}) {}
    size_t rows() const { return r_; }
    size_t cols() const { return c_; }
    size_t size() const { return v_.size(); }
    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }
    T* row(size_t i) { return v_.data() + i * c_; }
    const T* row(size_t i) const { return v_.data() + i * c_; }
    T& at(size_t i, size_t j) { return v_[i * c_ + j]; }
    const T& at(size_t i, size_t j) const { return v_[i * c_ + j]; }
    void fill(T x) { std::fill(v_.begin(), v_.end(), x); }
    void zero() { fill(T{0}); }
    bool same_shape(const Mat& o) const { return r_ == o.r_ && c_ == o.c_; }

  private:
    size_t r_ = 0, c_ = 0;
    std::vector<T> v_;
};
using MatF = Mat<float>;
using MatD = Mat<double>;

// ---------------------------------------------------------------- graph / CSR
// graph.hpp:15-30: undirected, both directions stored, rows sorted ascending,
// no duplicates, no self-loops.
struct Graph {
    VertexId num_vertices = 0;
    uint64_t num_edges = 0;
    std::vector<uint64_t> csr_offsets;
    std::vector<VertexId> csr_neighbors;
    std::vector<VertexId> degrees;
    std::span<const VertexId> neighbors(VertexId v) const {
        return {csr_neighbors.data() + csr_offsets[v], csr_neighbors.data() + csr_offsets[v + 1]};
    }
    VertexId degree(VertexId v) const { return degrees[v]; }
    void validate() const;
};

Graph build_graph(VertexId num_vertices, std::vector<std::pair<VertexId, VertexId>> edges);
Graph generate_er(VertexId n, double p, uint64_t seed);

template <typename T>
struct CsrMatrix {
    VertexId n = 0;
    std::vector<uint64_t> offsets;
    std::vector<VertexId> cols;
    std::vector<T> vals;
    size_t row_size(VertexId v) const { return offsets[v + 1] - offsets[v]; }
};
template <typename T>
CsrMatrix<T> normalize_adjacency(const Graph& g, bool add_self_loops = true);

// ---------------------------------------------------------------- dataset
enum class Split : uint8_t { Unused = 0, Train = 1, Val = 2, Test = 3 };

struct Dataset {
    Graph graph;
    MatF features;
    std::vector<uint32_t> labels;
    uint32_t num_classes = 0;
    std::vector<uint8_t> split;
    VertexId num_vertices() const { return graph.num_vertices; }
    uint32_t num_features() const { return uint32_t(features.cols()); }
    std::vector<uint8_t> mask(Split s) const;
    size_t mask_count(Split s) const;
    void validate() const;
};
Dataset load_dataset(const std::string& dir);
void save_dataset(const Dataset& d, const std::string& dir);
// Synthetic shapes of BASELINE.json: generate_er graph plus
// x[v,j] = 2*hash_unit(mix64(fseed, v*F+j)) - 1, label = mix64(fseed,0x4C42,v) % C,
// split by mix64(fseed,0x5350,v) % 10 (60/20/20).
// Stochastic block model dataset (dataset.cpp:147-191): blocks of block_size vertices,
// edge probability p_in inside a block and p_out across; one-hot-plus-noise features,
// label = block, 60/20/20 split by position in the block.
Dataset generate_sbm(uint32_t num_blocks, uint32_t block_size, double p_in, double p_out, uint64_t seed);
Dataset synthetic_er_dataset(VertexId n, double p, uint64_t graph_seed, uint32_t F, uint32_t C,
                             uint64_t feature_seed);

// ---------------------------------------------------------------- partitioning
struct Partition {
    uint32_t num_parts = 0;
    std::vector<uint32_t> assignment;
    std::vector<std::vector<VertexId>> inner_sets;
    std::vector<std::vector<VertexId>> boundary_sets;
    uint64_t boundary_total() const;
    uint64_t edge_cut(const Graph& g) const;
};
Partition partition_vertices(const Graph& g, uint32_t num_parts, uint64_t seed);
Partition partition_from_assignment(const Graph& g, std::vector<uint32_t> assignment);
// E|B_i| for an ER(n, p) graph cut into m equal parts (partition.cpp:206-211)
double expected_boundary(double n, double m, double p);

struct ChunkPlan {
    uint32_t num_chunks = 0;
    std::vector<uint32_t> chunk_of;
    std::vector<std::vector<VertexId>> chunks;
    std::vector<uint32_t> epoch_order;
};
ChunkPlan make_chunks(const Graph& g, uint32_t num_chunks, uint64_t seed);
ChunkPlan chunk_plan_from_assignment(VertexId n, std::vector<uint32_t> chunk_of);
std::vector<uint32_t> shuffle_chunk_order(const ChunkPlan& plan, uint64_t epoch, uint64_t seed);
// chunks.txt / parts.txt (partition.cpp:250-269): the part count on the first line, then
// one part id per vertex line; load returns {parts, assignment}
void save_assignment(const std::string& path, uint32_t num_parts, const std::vector<uint32_t>& assignment);
std::pair<uint32_t, std::vector<uint32_t>> load_assignment(const std::string& path);

// ---------------------------------------------------------------- model
enum class ModelKind { GCN, Sage, GCNII };
enum class LayerKind { Dense, GcnConv, SageConv, Gcn2Conv };
enum class OptimizerKind { Adam, Sgd };
ModelKind parse_model_kind(const std::string& s);
std::string model_kind_name(ModelKind k);

struct ModelConfig {
    ModelKind kind = ModelKind::GCN;
    uint32_t layers = 2;
    uint32_t hidden = 16;
    double dropout = 0.5;
    double gcnii_alpha = 0.1;
    double gcnii_lambda = 0.5;
    bool self_loops = true;
};

struct LayerSpec {
    LayerKind kind = LayerKind::Dense;
    uint32_t in_dim = 0, out_dim = 0;
    bool relu = true;
    double alpha = 0.0, beta = 0.0;
    bool aggregates() const { return kind != LayerKind::Dense; }
    bool has_bias() const { return kind != LayerKind::Gcn2Conv; }
    uint32_t k_in() const { return kind == LayerKind::SageConv ? 2 * in_dim : in_dim; }
};

std::vector<LayerSpec> build_layer_specs(const ModelConfig& cfg, uint32_t in_features,
                                         uint32_t num_classes);
bool model_needs_h0(const std::vector<LayerSpec>& specs);
uint64_t param_count(const std::vector<LayerSpec>& specs);

template <typename T>
struct LayerParams {
    Mat<T> weight;
    std::vector<T> bias;
};

// Glorot-uniform init, one engine per layer (matrix.hpp:53-59, nn.hpp:60-72).
template <typename T>
std::vector<LayerParams<T>> init_params(const std::vector<LayerSpec>& specs, uint64_t seed) {
    std::vector<LayerParams<T>> out(specs.size());
    for (size_t l = 0; l < specs.size(); ++l) {
        out[l].weight = Mat<T>(specs[l].k_in(), specs[l].out_dim);
        const double lim = std::sqrt(6.0 / double(out[l].weight.rows() + out[l].weight.cols()));
        auto eng = make_engine(seed, mix64(0x57454947ull, l));
        std::uniform_real_distribution<double> u(-lim, lim);
        T* w = out[l].weight.data();
        for (size_t i = 0, e = out[l].weight.size(); i < e; ++i) w[i] = T(u(eng));
        if (specs[l].has_bias()) out[l].bias.assign(specs[l].out_dim, T{0});
    }
    return out;
}

// ---------------------------------------------------------------- checkpoints (nn.hpp:497-531)
// One file per stage: u64 header length, JSON header {"tensors":[{"cols","name","rows"}...]},
// then the tensors as little-endian f32 (byte-compatible with the reference's files).
void save_checkpoint(const std::string& path, const std::vector<std::string>& names,
                     const std::vector<const float*>& data,
                     const std::vector<std::pair<uint64_t, uint64_t>>& shapes);
struct CheckpointTensor {
    std::string name;
    uint64_t rows = 0, cols = 0;
    std::vector<float> data;
};
std::vector<CheckpointTensor> load_checkpoint(const std::string& path);

template <typename T>
void save_stage_checkpoint(const std::string& path, const std::vector<LayerSpec>& specs,
                           const std::vector<LayerParams<T>>& params, size_t lo, size_t hi) {
    (void)specs;
    std::vector<std::string> names;
    std::vector<std::vector<float>> store;
    std::vector<std::pair<uint64_t, uint64_t>> shapes;
    for (size_t l = lo; l < hi; ++l) {
        const auto& w = params[l].weight;
        store.emplace_back(w.data(), w.data() + w.size());
        names.push_back("layer" + std::to_string(l) + ".weight");
        shapes.push_back({w.rows(), w.cols()});
        if (!params[l].bias.empty()) {
            store.emplace_back(params[l].bias.begin(), params[l].bias.end());
            names.push_back("layer" + std::to_string(l) + ".bias");
            shapes.push_back({1, params[l].bias.size()});
        }
    }
    std::vector<const float*> ptrs;
    for (const auto& v : store) ptrs.push_back(v.data());
    save_checkpoint(path, names, ptrs, shapes);
}

template <typename T>
struct OptimizerConfig {
    OptimizerKind kind = OptimizerKind::Adam;
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
};

// ---------------------------------------------------------------- fabric types
enum class MsgTag : uint32_t { ForwardEmb = 0, BackwardGrad, GraphBoundaryFwd, GraphBoundaryBwd, WeightSync, Control };
constexpr uint32_t kNumTags = 6;

struct GroupMap {
    uint32_t num_workers = 1, workers_per_node = 4, group_size = 1;
    std::vector<uint32_t> node_of, group_of, rank_in_group;
    std::vector<std::vector<uint32_t>> groups;
    uint32_t num_groups() const { return uint32_t(groups.size()); }
    uint32_t spanning_groups() const;  // groups whose workers sit on more than one node
};
GroupMap assign_groups(uint32_t num_workers, uint32_t workers_per_node, uint32_t num_stages,
                       uint32_t group_size);

struct EpochComm {
    uint64_t by_tag_link[kNumTags][2] = {{0}};
    uint64_t id_bytes = 0;
    uint64_t by_tag(uint32_t t) const { return by_tag_link[t][0] + by_tag_link[t][1]; }
    uint64_t graph_bytes() const { return by_tag(2) + by_tag(3); }
    uint64_t pipeline_bytes() const { return by_tag(0) + by_tag(1); }
    uint64_t weight_sync_bytes() const { return by_tag(4); }
};

struct TraceEvent {
    uint32_t worker;
    double t_start, t_end;
    enum class Kind { Compute, Send, Recv, Idle } kind;
    int32_t chunk = -1, layer_lo = -1, layer_hi = -1;
};

class FabricError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

// Only the knobs the GPU engine honours; Mode is accepted for source
// compatibility (stages always run concurrently, one host thread each).
struct FabricOptions {
    enum class Mode { Deterministic, Concurrent } mode = Mode::Deterministic;
    std::vector<uint32_t> node_of;
    double watchdog_seconds = 600.0;
    bool collect_trace = false;
};
// Fabric (fabric.hpp:150-160) is the reference's simulated worker substrate; here only
// its option types remain, so callers' `opt.fabric.mode = Fabric::Mode::Concurrent`
// compiles. Both modes produce identical results in the reference too (fabric.hpp:146-149).
class Fabric {
  public:
    using Mode = FabricOptions::Mode;
    using Options = FabricOptions;
};

// ---------------------------------------------------------------- engines
struct StageAssignment {
    uint32_t num_stages = 1;
    std::vector<std::pair<uint32_t, uint32_t>> ranges;
    uint32_t begin(uint32_t s) const { return ranges[s].first; }
    uint32_t end(uint32_t s) const { return ranges[s].second; }
};
StageAssignment make_stage_assignment(uint32_t layers, uint32_t stages);

struct StalenessConfig {
    bool shuffle_chunks = true;
    uint32_t fix_alpha = 10;
    bool historical_gradients = false;
    bool synchronous_mode = false;
};

struct EpochMetrics {
    uint32_t epoch = 0;
    double train_loss = 0, train_acc = 0, val_acc = 0, test_acc = 0;
    uint64_t comm_bytes_graph = 0, comm_bytes_pipeline = 0, comm_bytes_weightsync = 0;
    double wall_time_s = 0;      // measured device time of the epoch (max over stages)
    double bubble_fraction = 0;  // 1 - sum(stage busy) / (S * span), profiling runs only
};

class NumericError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

// CUDA / NCCL failure reported by the gp_* layer (no reference counterpart).
struct GpError : std::runtime_error {
    gp_status code;
    GpError(gp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <typename T>
struct WorkerParams {
    uint32_t layer_begin = 0, layer_end = 0;
    std::vector<LayerParams<T>> params;
};

// Resumable training state (extension: the reference's checkpoints are
// parameters only and there is no resume path). epoch = last completed epoch;
// adam_m / adam_v mirror params (Optimizer m_/v_, nn.hpp:431-495).
// history: the historical-embedding rows the next epoch reads stale values from
// (h_snap / in_snap / dagg_snap after the snapshot rule, engines_impl.hpp:671-679),
// one entry per worker and buffer, original vertex order; empty in synchronous mode.
struct TrainState {
    uint32_t epoch = 0;
    uint64_t optimizer_step = 0;
    std::vector<LayerParams<float>> params, adam_m, adam_v;
    struct HistoryRows {
        uint32_t worker = 0, which = 0, layer = 0, width = 0;  // which: GP_BUF_HIST_*; layer: global
        std::vector<float> rows;                                // N x width
    };
    std::vector<HistoryRows> history;
};
// Stored in the checkpoint format: layerL.weight/.bias (as save_stage_checkpoint),
// layerL.{weight,bias}.adam_{m,v}, train.state = [epoch, optimizer_step], and
// history.wW.kK.lL (N x width) for each history entry.
void save_train_state(const std::string& path, const TrainState& st);
TrainState load_train_state(const std::string& path, const std::vector<LayerSpec>& specs);

template <typename T>
struct TrainResult {
    std::vector<EpochMetrics> metrics;
    std::vector<LayerParams<T>> params;
    std::vector<WorkerParams<T>> worker_params;
    std::vector<TraceEvent> trace;
    std::vector<EpochComm> comm;
    uint64_t peak_buffer_bytes = 0;  // max per-stage device footprint
    gp_profile profile{};            // summed over stages (profiling runs)
    TrainState final_state;          // parameters + optimizer state after the last epoch
};

template <typename T>
struct TrainOptions {
    ModelConfig model;
    OptimizerConfig<T> optimizer;
    uint32_t epochs = 1;
    uint64_t seed = 1;
    StalenessConfig staleness;
    FabricOptions fabric;
    int device = 0;        // first CUDA device (stages round-robin over visible GPUs)
    bool profile = false;  // per-kernel device timing
    // Continue from a saved state: parameters, optimizer moments and (stale mode) the
    // historical-embedding rows are restored and epochs run from resume->epoch + 1
    // (dropout keys, chunk order and the snapshot schedule continue), so a resumed run
    // equals an uninterrupted one. Stale-mode resume without history is rejected.
    std::shared_ptr<const TrainState> resume;
    // Put the historical-embedding rows into final_state.history (N x H per stashed
    // layer and worker, read back from the device after the last epoch).
    bool keep_history = false;
};

template <typename T>
TrainResult<T> train_sequential(const Dataset& ds, const TrainOptions<T>& opt);
template <typename T>
TrainResult<T> train_pipeline(const Dataset& ds, const ChunkPlan& plan, const StageAssignment& stages,
                              const TrainOptions<T>& opt);
template <typename T>
TrainResult<T> train_hybrid(const Dataset& ds, const Partition& part, const ChunkPlan& plan,
                            const StageAssignment& stages, const GroupMap& gmap,
                            const TrainOptions<T>& opt);
// Graph parallelism (engines.hpp:83-87): the reference's hybrid engine at S = 1,
// K = 1 reproduces it bitwise (test_engines.cpp:238-251), and so does this one.
template <typename T>
TrainResult<T> train_graph_parallel(const Dataset& ds, const Partition& part, const TrainOptions<T>& opt);

// ---------------------------------------------------------------- run outputs and analytics
// (fabric.hpp/fabric.cpp:20-35, :136-182; analytics.hpp/analytics.cpp; engines.cpp:23-38)
const char* tag_name(MsgTag t);
enum class LinkClass : uint32_t { IntraNode = 0, InterNode = 1 };
const char* link_class_name(LinkClass c);
const char* trace_kind_name(TraceEvent::Kind k);

struct CommReportRow {
    uint32_t epoch;
    MsgTag tag;
    LinkClass link;
    uint64_t bytes;
    double gib;  // bytes / 2^30
};
// Non-zero (tag, link) cells of one closed epoch (ledger_report fabric.cpp:136-146).
std::vector<CommReportRow> ledger_report(const EpochComm& e, uint32_t epoch);
void write_comm_report_csv(const std::string& path, const std::vector<CommReportRow>& rows);
void write_trace_jsonl(const std::string& path, const std::vector<TraceEvent>& events);
void write_metrics_csv(const std::string& path, const std::vector<EpochMetrics>& metrics);

struct CommModelInput {
    double n = 0, layers = 0, hidden = 0, stages = 1, ways = 1, alpha = 0, vecs = 1;
    double bytes_per_value = 4;
};
constexpr double kGiB = 1024.0 * 1024.0 * 1024.0;
double volume_pipeline(const CommModelInput& in);  // 2 (S-1) N H vecs * bytes
double volume_graph(const CommModelInput& in);     // 2 alpha L N H * bytes
double volume_hybrid(const CommModelInput& in);    // graph + pipeline

struct CrossoverReport {
    double bytes_graph = 0, bytes_pipeline = 0, bytes_hybrid = 0;
    std::vector<std::string> ordering;
    bool tie = false;
    std::vector<std::string> inequalities;
    std::string winner;
};
CrossoverReport crossover_report(const CommModelInput& graph_in, const CommModelInput& pipe_in,
                                 const CommModelInput& hybrid_in);

struct BubbleReport {
    double measured_bubble = 0;  // idle fraction of workers x span
    double ideal_bubble = 0;     // (S-1) / (K+S-1)
    uint32_t stages = 0;
    uint32_t chunks = 0;
    double span = 0;
};
BubbleReport bubble_analysis(const std::vector<TraceEvent>& trace);

struct CompareRow {
    std::string mode;
    double n, layers, hidden, stages, ways, alpha, vecs;
    double predicted_bytes;
    uint64_t measured_bytes;
    double rel_error;
};
void write_compare_csv(const std::string& path, const std::vector<CompareRow>& rows);

extern template TrainResult<float> train_sequential<float>(const Dataset&, const TrainOptions<float>&);
extern template TrainResult<float> train_pipeline<float>(const Dataset&, const ChunkPlan&,
                                                         const StageAssignment&, const TrainOptions<float>&);
extern template TrainResult<float> train_graph_parallel<float>(const Dataset&, const Partition&,
                                                               const TrainOptions<float>&);
extern template TrainResult<float> train_hybrid<float>(const Dataset&, const Partition&, const ChunkPlan&,
                                                       const StageAssignment&, const GroupMap&,
                                                       const TrainOptions<float>&);

}  // namespace gnnsim

/*
 * gnnpipe.h — C-ABI of the B200 chunk-pipelined GNN training engine.
 *
 * Two layers, both plain C (extern "C", PODs, pointers + sizes, status codes):
 *
 *   gp_*  DEVICE ENGINE (libgpcuda.so, sm_100a). One gp_ctx per pipeline stage.
 *         It replaces the per-worker body of the reference trainer
 *         (proj/src/engines_impl.hpp:564-898) — the chunk loop, the per-row
 *         kernels it calls (proj/include/gnnsim/nn.hpp:140-293, matrix.hpp:63-86),
 *         the historical-embedding store (engines_impl.hpp:580-617, :671-679,
 *         :735-782), the optimizer step (nn.hpp:456-490) and the stage messages
 *         (engines_impl.hpp:690-724 -> fabric.cpp:288-359).
 *
 *   gs_*  HOST API (libgnnsim_b200.so, C++). Flat C wrappers over the C++ mirror
 *         of the reference API (namespace gnnsim, csrc/include/gnnsim_b200.hpp):
 *         build_graph, normalize_adjacency, generate_er, load/save_dataset,
 *         make_chunks, partition_vertices, shuffle_chunk_order,
 *         make_stage_assignment, build_layer_specs, init_params, and
 *         train_pipeline / train_sequential. The C++ trainers call the gp_* ABI.
 *
 * Status codes map the reference's exception classes
 * (std::invalid_argument, NumericError engines.hpp:48-51, FabricError
 * fabric.hpp:139-142); gp_last_error()/gs_last_error() return the message.
 * There is no CPU fallback: without a CUDA device gp_create fails with
 * GP_ECUDA.
 */
#ifndef GNNPIPE_H
#define GNNPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GP_ABI_VERSION 1u

typedef enum {
    GP_OK = 0,
    GP_EINVAL = 1,    /* std::invalid_argument in the reference            */
    GP_ENUMERIC = 2,  /* gnnsim::NumericError (non-finite loss)            */
    GP_EFABRIC = 3,   /* gnnsim::FabricError (transport / watchdog)        */
    GP_ECUDA = 4,     /* CUDA or NCCL failure, or no device                */
    GP_ERUNTIME = 5   /* anything else (std::runtime_error)                */
} gp_status;

/* Mirrors LayerKind (nn.hpp:16). SageConv is outside the hot-path scope
 * and is rejected with GP_EINVAL. */
typedef enum { GP_DENSE = 0, GP_GCNCONV = 1, GP_SAGECONV = 2, GP_GCN2CONV = 3 } gp_layer_kind;

/* Mirrors LayerSpec (nn.hpp:32-44). */
typedef struct {
    uint32_t kind;    /* gp_layer_kind */
    uint32_t in_dim;
    uint32_t out_dim;
    uint32_t relu;
    double alpha;     /* Gcn2Conv only */
    double beta;      /* Gcn2Conv only */
} gp_layer_spec;

/* What one stage worker of train_hybrid needs (engines_impl.hpp:564-617). */
typedef struct {
    int32_t device;              /* CUDA ordinal */
    uint32_t num_vertices;       /* N (< 2^26)                                  */
    uint32_t num_chunks;         /* K (1..64)                                   */
    uint32_t num_stages;         /* S                                           */
    uint32_t stage;              /* s                                           */
    uint32_t layer_begin;        /* [lb, le) global layers owned by s           */
    uint32_t layer_end;
    uint32_t num_layers;         /* L                                           */
    const gp_layer_spec* specs;  /* all L specs (copied)                        */
    uint32_t hidden;             /* H = width of h0 (GCNII)                     */
    uint32_t num_classes;        /* C                                           */
    double dropout;              /* ModelConfig::dropout (nn.hpp:26)            */
    uint64_t seed;               /* TrainOptions::seed                          */
    uint32_t optimizer;          /* 0 Adam, 1 SGD (OptimizerKind nn.hpp:17)    */
    double lr, beta1, beta2, eps;/* OptimizerConfig (nn.hpp:432-438)            */
    uint32_t fix_alpha;          /* StalenessConfig (engines.hpp:28-33)         */
    uint32_t historical_gradients;
    uint32_t synchronous_mode;
    uint32_t group_size;         /* G graph partitions per stage (0/1 = pure pipeline) */
    uint32_t group_rank;         /* r: this worker owns Partition::inner_sets[r]      */
} gp_stage_config;

typedef struct gp_ctx gp_ctx;

/* Per-epoch results of one stage (gp_run_epoch). Quality fields are valid on
 * the last stage only (SplitStats, engines_impl.hpp:29-37, :816-825). */
typedef struct {
    uint32_t epoch;
    uint32_t has_quality;
    double loss_sum;             /* sum of train-row xent in double            */
    uint64_t correct[3];         /* train / val / test correct counts          */
    uint64_t bytes_sent[6];      /* by MsgTag (fabric.hpp:14-21), 4 B/value    */
    uint64_t msgs_sent[6];
    float epoch_ms;              /* CUDA events on the stage compute stream    */
    float busy_ms;               /* sum of this stage's kernel times (profiling) */
    uint64_t kernel_launches;    /* kernels this stage launched in the epoch   */
} gp_epoch_stats;

/* Per-kernel-class device time (profiling mode), summed since last reset. */
enum {
    GP_K_REMASK = 0, GP_K_FWD_AGG = 1, GP_K_FWD_DENSE = 2, GP_K_BWD_AGG = 3,
    GP_K_BWD_DENSE = 4, GP_K_XENT = 5, GP_K_PGRAD = 6, GP_K_OPTIM = 7,
    GP_K_XFER = 8, GP_K_NUM = 9
};
typedef struct {
    double ms[GP_K_NUM];         /* summed kernel durations (CUDA events)      */
    uint64_t launches[GP_K_NUM];
    double alg_bytes[GP_K_NUM];  /* algorithmic HBM bytes       */
    double flops[GP_K_NUM];
    double gather_bytes[GP_K_NUM]; /* bytes gathered through L2 by SpMMs        */
    double span_ms[GP_K_NUM];    /* time at least one launch of the class ran   */
                                 /* (union of its launch intervals; concurrent  */
                                 /* launches on the wavefront streams overlap)  */
} gp_profile;

/* Buffers readable through gp_download (parity tests; original vertex order). */
enum {
    GP_BUF_H = 0,        /* h_cur[i]   layer output                 (N x out) */
    GP_BUF_PRE = 1,      /* pre[i]     pre-transform rows           (N x k_in)*/
    GP_BUF_DZ = 2,       /* dz[i]                                   (N x out) */
    GP_BUF_DAGG = 3,     /* dagg[i] (unscaled)                      (N x k_in)*/
    GP_BUF_DH0 = 4,      /* dh0_run                                 (N x H)   */
    GP_BUF_HSNAP = 5,    /* h_snap[i]                               (N x out) */
    GP_BUF_IN = 6,       /* in_cur (stage input)                    (N x in0) */
    GP_BUF_DH_IN = 7,    /* dh_in  (gradient sent upstream)         (N x in0) */
    GP_BUF_GATHER = 8,   /* masked gather source of layer i         (N x in)  */
    /* historical-embedding state the next epoch reads stale rows from (resume):
     * h_snap[i] / in_snap / dagg_snap[i] after the snapshot rule of
     * engines_impl.hpp:671-679 (readable with gp_download, restorable with
     * gp_upload_history) */
    GP_BUF_HIST_H = 9,   /* (N x out)  */
    GP_BUF_HIST_IN = 10, /* (N x in0)  */
    GP_BUF_HIST_DAGG = 11 /* (N x k_in), historical-gradient ablation */
};

/* ---- lifecycle ---------------------------------------------------------- */
uint32_t gp_abi_version(void);
gp_status gp_create(const gp_stage_config* cfg, gp_ctx** out);
void gp_destroy(gp_ctx* ctx);
const char* gp_last_error(const gp_ctx* ctx); /* ctx may be NULL: thread-local */
gp_status gp_device_count(int* out);

/* ---- data (caller-owned host buffers, copied) ---------------------------- */
/* Normalised adjacency (CsrMatrix<float>, graph.hpp:37-45 as produced by
 * normalize_adjacency graph.cpp:68-98) and the chunk plan (ChunkPlan::chunk_of,
 * partition.hpp:39-44). The engine renumbers vertices chunk-contiguously on
 * device; neighbour order inside each row is preserved. */
gp_status gp_upload_graph(gp_ctx* ctx, const uint64_t* offsets, const uint32_t* cols,
                          const float* vals, uint64_t nnz, const uint32_t* chunk_of);
/* Same, from the graph itself (Graph::csr_offsets / csr_neighbors, graph.hpp:15-34:
 * strictly ascending neighbours, no self loops): normalize_adjacency<float>
 * (graph.cpp:68-98) is applied row by row while the packed CSR is built, with the
 * same double-precision expression, so the uploaded matrix is bit-identical and no
 * N-sized host copy of it is made. Single-partition stages ship the raw lists and
 * build the packed CSR on the device (GP_GRAPH_BUILD). num_neighbors = 2E. */
gp_status gp_upload_graph_raw(gp_ctx* ctx, const uint64_t* offsets, const uint32_t* neighbors,
                              uint64_t num_neighbors, int self_loops, const uint32_t* chunk_of);
/* Hybrid (train_hybrid, engines_impl.hpp:515-909, G > 1): the vertex partition
 * (Partition::assignment, partition.hpp:13-21). Call before gp_upload_graph. */
gp_status gp_upload_partition(gp_ctx* ctx, const uint32_t* part_of);
/* Reuse another stage's device graph (same device) instead of a second copy. */
gp_status gp_share_graph(gp_ctx* ctx, const gp_ctx* owner);
/* Dataset::features (dataset.hpp:17) N x F row-major; stage 0 only. */
gp_status gp_upload_features(gp_ctx* ctx, const float* x, uint32_t num_features);
/* Dataset::labels / split (dataset.hpp:18-20); last stage only. */
gp_status gp_upload_labels(gp_ctx* ctx, const uint32_t* labels, const uint8_t* split);
/* LayerParams (nn.hpp:54-58): W k_in x out row-major, b out (NULL if none). */
gp_status gp_set_layer_params(gp_ctx* ctx, uint32_t layer, const float* W, const float* b);
gp_status gp_get_layer_params(gp_ctx* ctx, uint32_t layer, float* W, float* b);
/* ParamGrads of the last epoch (nn.hpp:264-293, Gcn2Conv already scaled by beta). */
gp_status gp_get_layer_grads(gp_ctx* ctx, uint32_t layer, float* W, float* b);
/* Optimizer state of a layer (Optimizer m_/v_ and step count t_, nn.hpp:431-495),
 * for checkpoint/resume (the reference's checkpoints hold parameters only,
 * nn.hpp:497-531). mb/vb are ignored for layers without a bias; step is the
 * stage's optimizer step count (one per epoch). */
gp_status gp_get_optimizer_state(gp_ctx* ctx, uint32_t layer, float* mW, float* vW, float* mb, float* vb,
                                 uint64_t* step);
gp_status gp_set_optimizer_state(gp_ctx* ctx, uint32_t layer, const float* mW, const float* vW,
                                 const float* mb, const float* vb, uint64_t step);

/* ---- transport (stage boundaries, engines_impl.hpp:690-724) -------------- */
/* Same process: upstream stage s and downstream stage s+1 exchange chunk rows
 * with device-to-device copies ordered by CUDA events (one host thread per
 * stage, like Fabric::Mode::Concurrent fabric.cpp:401-422). */
gp_status gp_link_local(gp_ctx* upstream, gp_ctx* downstream);
/* One process per GPU: NCCL send/recv over NVLink. Each stage boundary is a
 * 2-rank communicator (rank 0 = upstream stage). Pass NULL for a missing side. */
gp_status gp_nccl_unique_id(uint8_t out[128]);
gp_status gp_link_nccl(gp_ctx* ctx, const uint8_t* up_id, const uint8_t* down_id);
/* One process per GPU: CUDA-IPC peer-memory rings (replaces the reference's
 * in-process fabric channels, WorkerCtx::send/recv fabric.cpp:288-359, for stages in different
 * processes of one node). The receiving side of each direction owns a ring of
 * message slots; the sender pushes chunk rows into the peer's slot with the copy
 * engine over NVLink and signals with in-stream memory ops, so the transfer
 * overlaps the next chunk's kernels without taking SMs. Protocol:
 *   1. gp_ipc_export after gp_upload_graph: fills an opaque blob per boundary
 *      (up: shared with stage s-1, down: with stage s+1; NULL for a missing side);
 *   2. exchange blobs out of band (any control plane);
 *   3. gp_link_ipc(ctx, blob exported as `down` by stage s-1, blob exported as
 *      `up` by stage s+1). Both processes may use the same device. */
#define GP_IPC_BLOB_BYTES 256
gp_status gp_ipc_export(gp_ctx* ctx, uint8_t* up_blob, uint8_t* down_blob);
gp_status gp_link_ipc(gp_ctx* ctx, const uint8_t* up_peer_blob, const uint8_t* down_peer_blob);
/* Hybrid: join the G workers of one stage group (same process). Halo rows of each
 * aggregating layer (exchange_rows, engines_impl.hpp:626-643) are pulled by the
 * receiver from its peers' buffers after an event handshake; weight gradients
 * are folded in rank order at rank 0 and broadcast (group_weight_sync :102-128). */
gp_status gp_link_group(gp_ctx** members, uint32_t group_size);
/* Hybrid group across processes (one process per GPU; replaces the in-process
 * group channels of exchange_rows engines_impl.hpp:626-643 and group_weight_sync
 * :102-128). Each member maps its peers' activation / gradient-table / weight-
 * gradient buffers over CUDA IPC and pulls halo rows straight from them after an
 * in-stream counter handshake; rank 0 folds weight gradients in rank order.
 *   1. after gp_upload_graph (and before the first epoch): gp_group_export fills
 *      this member's blob (call with blob = NULL to get the length);
 *   2. exchange blobs out of band within the stage group;
 *   3. gp_link_group_ipc(ctx, blobs, lengths): blobs[r] = member r's blob (own entry
 *      ignored). Stage links between groups use gp_ipc_export / gp_link_ipc. */
gp_status gp_group_export(gp_ctx* ctx, uint8_t* blob, uint64_t capacity, uint64_t* length);
gp_status gp_link_group_ipc(gp_ctx* ctx, const uint8_t* const* blobs, const uint64_t* lengths);
/* Abort a blocked local transport (error propagation across stage threads). */
void gp_abort(gp_ctx* ctx);

/* ---- epochs -------------------------------------------------------------- */
/* One epoch t (1-based) with the host-computed chunk order (shuffle_chunk_order
 * partition.cpp:239-248, so schedule order stays bit-exact). Blocks until the
 * stage's work for the epoch is complete. */
gp_status gp_run_epoch(gp_ctx* ctx, uint32_t t, const uint32_t* order, gp_epoch_stats* out);

/* ---- introspection / profiling ------------------------------------------ */
gp_status gp_download(gp_ctx* ctx, uint32_t which, uint32_t local_layer, float* out,
                      uint64_t count);
gp_status gp_set_profiling(gp_ctx* ctx, int enable);
/* CUDA events around every launch of one kernel class (GP_K_*) in normal epochs (the
 * chunk wavefront stays on), accumulated into gp_get_profile; GP_K_NUM times every class,
 * -1 turns it off. Used by bench.py to time the dominant kernel inside the timed region. */
gp_status gp_set_live_timing(gp_ctx* ctx, int kernel_class);
/* Device bytes gp_create + the uploads would allocate for this stage (the stash
 * layout under the current GP_LEAN / GP_MERGED_G switches, graph with nnz_norm
 * normalised entries, features of width num_features on stage 0, labels on the
 * last stage). Needs no device: a memory plan for configurations larger than the
 * GPUs at hand (reference: peak_buffer_bytes, engines_impl.hpp:891-896). */
gp_status gp_stage_footprint(const gp_stage_config* cfg, uint64_t nnz_norm, uint32_t num_features,
                             uint64_t* bytes);
/* Restore one history buffer (GP_BUF_HIST_*, original vertex order, N x width)
 * before resuming at epoch resume_epoch + 1. Extension: the reference has no
 * resume path (its checkpoints are parameters only, nn.hpp:497-531). */
gp_status gp_upload_history(gp_ctx* ctx, uint32_t which, uint32_t local_layer, const float* rows,
                            uint64_t count, uint32_t resume_epoch);

/* Trace of a stage's epochs (replaces the simulated-clock trace of the fabric,
 * TraceEvent fabric.hpp, Fabric::trace fabric.cpp:256-264; collect_trace
 * fabric.cpp:222-227). Kinds follow TraceEvent::Kind. Times are the device's
 * %globaltimer in nanoseconds (one timebase for all stages of a node, anchored
 * once per epoch per stage by a one-thread stamp kernel: cross-stage times agree
 * to a few microseconds); a
 * compute span covers one chunk's layers [layer_lo, layer_hi] of the stage
 * (chunk -1: the whole partition in synchronous mode, or the epoch-close
 * parameter step). Tracing runs chunks serially (no wavefront). */
enum { GP_TRACE_COMPUTE = 0, GP_TRACE_SEND = 1, GP_TRACE_RECV = 2, GP_TRACE_IDLE = 3 };
typedef struct {
    uint32_t epoch;
    uint32_t kind;
    int32_t chunk;
    int32_t layer_lo;
    int32_t layer_hi;
    uint32_t reserved;
    double t_start_ns;
    double t_end_ns;
} gp_trace_event;
gp_status gp_set_trace(gp_ctx* ctx, int enable);
/* Copies up to `cap` resolved events (all epochs since the last clear) into
 * `out` (may be NULL) and stores the total in *count. */
gp_status gp_get_trace(gp_ctx* ctx, gp_trace_event* out, uint64_t cap, uint64_t* count);
gp_status gp_clear_trace(gp_ctx* ctx);
gp_status gp_get_profile(gp_ctx* ctx, gp_profile* out);
gp_status gp_reset_profile(gp_ctx* ctx);
gp_status gp_device_bytes(gp_ctx* ctx, uint64_t* out); /* stash footprint */
/* Device timestamps on the stage's compute stream (bench timing): record event
 * `slot` (0..15); gp_elapsed synchronises and returns ms between two slots. */
gp_status gp_mark(gp_ctx* ctx, uint32_t slot);
gp_status gp_elapsed(gp_ctx* ctx, uint32_t slot_a, uint32_t slot_b, float* ms);
gp_status gp_synchronize(gp_ctx* ctx);

/* ====================== host API (libgnnsim_b200.so) ===================== */

typedef struct gs_dataset gs_dataset;
typedef struct gs_result gs_result;

typedef struct {
    uint32_t kind;        /* 0 gcn, 1 sage, 2 gcnii (ModelKind nn.hpp:15) */
    uint32_t layers;
    uint32_t hidden;
    double dropout;
    double gcnii_alpha;
    double gcnii_lambda;
    uint32_t self_loops;
} gs_model_config;        /* ModelConfig nn.hpp:22-30 */

typedef struct {
    gs_model_config model;
    uint32_t optimizer;   /* 0 Adam, 1 SGD */
    double lr, beta1, beta2, eps;
    uint32_t epochs;
    uint64_t seed;
    uint32_t shuffle_chunks, fix_alpha, historical_gradients, synchronous_mode;
    int32_t device;       /* first CUDA device; stages are placed round-robin */
    uint32_t profile;     /* collect per-kernel device times                  */
    uint32_t collect_trace; /* FabricOptions::collect_trace (fabric.hpp): measured trace */
    const char* resume_path;     /* NULL/"" or a save_state_path file: continue from it   */
    const char* save_state_path; /* NULL/"" or where to write the final TrainState       */
} gs_train_options;       /* TrainOptions engines.hpp:69-77 (+ resume, an extension) */

/* TraceEvent (fabric.hpp): seconds from the first event of the run. */
typedef struct {
    uint32_t worker;
    uint32_t kind;        /* GP_TRACE_* (TraceEvent::Kind order) */
    int32_t chunk, layer_lo, layer_hi;
    uint32_t reserved;
    double t_start, t_end;
} gs_trace_event;

typedef struct {
    double measured_bubble, ideal_bubble;
    uint32_t stages, chunks;
    double span;
} gs_bubble_report;       /* BubbleReport analytics.hpp:47-54 */

typedef struct {
    double n, layers, hidden, stages, ways, alpha, vecs, bytes_per_value;
} gs_comm_model_input;    /* CommModelInput analytics.hpp:14-24 */

const char* gs_last_error(void);

/* Graph / dataset (graph.cpp:33-66, :119-156; dataset.cpp:64-145). */
int gs_dataset_from_edges(uint32_t n, const uint32_t* uv, uint64_t m, const float* x,
                          uint32_t F, const uint32_t* labels, uint32_t C, const uint8_t* split,
                          gs_dataset** out);
int gs_dataset_synthetic_er(uint32_t n, double p, uint64_t graph_seed, uint32_t F, uint32_t C,
                            uint64_t feature_seed, gs_dataset** out);
int gs_dataset_load(const char* dir, gs_dataset** out);
int gs_dataset_save(const gs_dataset* d, const char* dir);
void gs_dataset_free(gs_dataset* d);
int gs_dataset_shape(const gs_dataset* d, uint32_t* n, uint64_t* m, uint32_t* F, uint32_t* C);
int gs_dataset_graph(const gs_dataset* d, uint64_t* offsets, uint32_t* neighbors,
                     uint32_t* degrees);
int gs_dataset_arrays(const gs_dataset* d, float* x, uint32_t* labels, uint8_t* split);
int gs_normalize_adjacency(const gs_dataset* d, int self_loops, uint64_t* offsets,
                           uint32_t* cols, float* vals);

/* Partitioning and schedule (partition.cpp, engines.cpp:8-21). */
int gs_make_chunks(const gs_dataset* d, uint32_t K, uint64_t seed, uint32_t* chunk_of);
int gs_partition_vertices(const gs_dataset* d, uint32_t parts, uint64_t seed,
                          uint32_t* assignment, uint64_t* edge_cut, uint64_t* boundary_total);
int gs_shuffle_chunk_order(uint32_t K, uint64_t epoch, uint64_t seed, uint32_t* order);
int gs_make_stage_assignment(uint32_t layers, uint32_t stages, uint32_t* ranges /* 2*S */);
/* chunks.txt / parts.txt (save_assignment / load_assignment, partition.cpp:250-269);
 * load: call with assignment = NULL for the count n, then with a buffer of cap >= n. */
int gs_save_assignment(const char* path, uint32_t num_parts, const uint32_t* assignment, uint64_t n);
int gs_load_assignment(const char* path, uint32_t* num_parts, uint32_t* assignment, uint64_t cap, uint64_t* n);

/* Model (nn.cpp:28-71, nn.hpp:60-72). */
int gs_num_layers(const gs_model_config* m, uint32_t* L);
int gs_build_layer_specs(const gs_model_config* m, uint32_t F, uint32_t C, gp_layer_spec* out);
int gs_init_params(const gs_model_config* m, uint32_t F, uint32_t C, uint64_t seed,
                   float* flat /* concat of W_l then b_l per layer */);

/* Trainers (engines.hpp:79-99): run on the GPU through gp_*. */
int gs_train_pipeline(const gs_dataset* d, const uint32_t* chunk_of, uint32_t K, uint32_t S,
                      const gs_train_options* opt, gs_result** out);
int gs_train_sequential(const gs_dataset* d, const gs_train_options* opt, gs_result** out);
/* train_hybrid (engines.hpp:96-99): S stages x G graph partitions; part_of is
 * Partition::assignment (G = max + 1), groups as assign_groups(S*G, 4, S, G). */
int gs_train_hybrid(const gs_dataset* d, const uint32_t* part_of, const uint32_t* chunk_of, uint32_t K,
                    uint32_t S, const gs_train_options* opt, gs_result** out);
/* train_graph_parallel (engines.hpp:83-87) = hybrid at S = 1, K = 1. */
int gs_train_graph_parallel(const gs_dataset* d, const uint32_t* part_of, const gs_train_options* opt,
                            gs_result** out);
/* T x {epoch, train_loss, train_acc, val_acc, test_acc, wall_time_s, bubble_fraction} */
int gs_result_metrics(const gs_result* r, uint32_t* epochs, double* metrics,
                      uint64_t* comm /* T x {graph, pipeline, weightsync} */);
int gs_result_params(const gs_result* r, float* flat);
int gs_result_profile(const gs_result* r, gp_profile* out);
/* Checkpoints (nn.hpp:497-531, nn.cpp:82-124): save_stage_checkpoint of layers
 * [lo, hi) from flat parameters (gs_init_params layout); load_checkpoint returns
 * newline-separated names, (rows, cols) pairs and the concatenated data (call
 * with NULL buffers first to get n_tensors / n_floats). */
int gs_save_stage_checkpoint(const char* path, const gs_model_config* m, uint32_t F, uint32_t C,
                             const float* flat, uint32_t lo, uint32_t hi);
int gs_load_checkpoint(const char* path, char* names, uint64_t names_cap, uint64_t* shapes, float* data,
                       uint64_t* n_tensors, uint64_t* n_floats);
/* Bytes gs_load_checkpoint's newline-separated names need (incl. the NUL). */
int gs_checkpoint_names_bytes(const char* path, uint64_t* bytes);
/* Measured trace (collect_trace runs): copies up to cap events, *count = total. */
int gs_result_trace(const gs_result* r, gs_trace_event* out, uint64_t cap, uint64_t* count);
/* Communication ledger: T x 6 tags x 2 link classes (EpochComm::by_tag_link). */
int gs_result_ledger(const gs_result* r, uint64_t* out);

/* Run outputs and analytics (engines.cpp:23-38, fabric.cpp:136-182,
 * analytics.cpp:12-103). */
int gs_write_metrics_csv(const char* path, const double* metrics /* T x 7 as gs_result_metrics */,
                         const uint64_t* comm /* T x 3 */, uint32_t epochs);
int gs_write_trace_jsonl(const char* path, const gs_trace_event* events, uint64_t n);
int gs_write_comm_report_csv(const char* path, const uint64_t* ledger /* T x 6 x 2 */, uint32_t epochs);
int gs_bubble_analysis(const gs_trace_event* events, uint64_t n, gs_bubble_report* out);
int gs_comm_volumes(const gs_comm_model_input* in, double* graph, double* pipeline, double* hybrid);
/* crossover_report (analytics.cpp:26-56): bytes[3] = graph, pipeline, hybrid;
 * text = "winner\nordering (comma-separated)\ntie 0|1\ninequality lines...". */
int gs_crossover_report(const gs_comm_model_input* graph_in, const gs_comm_model_input* pipe_in,
                        const gs_comm_model_input* hybrid_in, double* bytes, char* text, uint64_t cap);
/* write_compare_csv (analytics.cpp:88-103): modes = n newline-separated names;
 * vals = n x 9 (N, L, H, S, W, alpha, vecs, predicted_bytes, rel_error). */
int gs_write_compare_csv(const char* path, const char* modes, const double* vals, const uint64_t* measured,
                         uint64_t n);
int gs_result_peak_bytes(const gs_result* r, uint64_t* out);
void gs_result_free(gs_result* r);

#ifdef __cplusplus
}
#endif
#endif /* GNNPIPE_H */

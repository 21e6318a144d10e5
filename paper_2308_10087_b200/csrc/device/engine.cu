// Stage engine: the device-resident state and epoch schedule of one pipeline
// stage, exported through the gp_* C-ABI (include/gnnpipe.h).
//
// Reference mapping (proj/src/engines_impl.hpp, train_hybrid's worker body):
//   stash allocation  :580-612  -> Stage::alloc()
//   snapshot          :671-679  -> pointer swaps in run_epoch()
//   dropout masks     :681-683  -> DropKey per (t, l), hashed on device
//   forward chunk loop:784-814  -> run_epoch() forward section
//   metrics           :816-825  -> k_xent_stats / k_xent_fold
//   backward loop     :827-870  -> run_epoch() backward section
//   param grads + step:872-878  -> k_pgrad_* + k_adam
//   stage messages    :690-724  -> Transport (local D2D, CUDA-IPC peer rings, or NCCL)
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>  // types and the config initializer only; libnccl.so.2 is dlopen'ed
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../../include/gnnpipe.h"
#include "dense_tile.cuh"
#include "rows8.cuh"
#include "tc_pgrad.cuh"
#include "tc_xform.cuh"

namespace gp {
namespace {

thread_local std::string g_tls_error;

struct Error : std::runtime_error {
    gp_status code;
    Error(gp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GP_CUDA(expr)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            throw ::gp::Error(GP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
    } while (0)

inline uint32_t pad8(uint32_t d) { return (d + 7u) & ~7u; }

// ------------------------------------------------------------------ NCCL (dlopen)
// NCCL is resolved at run time so single-GPU use never depends on it and the
// process shares whichever libnccl.so.2 torch may already have loaded.
struct NcclApi {
    typedef int (*GetUniqueId)(void*);
    typedef int (*CommInitRank)(void**, int, const void*, int);  // id passed by value (128 B)
    typedef int (*CommDestroy)(void*);
    typedef int (*SendRecv)(const void*, size_t, int, int, void*, cudaStream_t);
    typedef int (*Group)();
    typedef const char* (*ErrStr)(int);
    void* h = nullptr;
    GetUniqueId get_unique_id = nullptr;
    void* comm_init_rank = nullptr;
    CommDestroy comm_destroy = nullptr;
    SendRecv send = nullptr;
    void* recv = nullptr;
    Group group_start = nullptr, group_end = nullptr;
    ErrStr err = nullptr;
    // non-blocking communicators: init with a watchdog instead of blocking forever on
    // a peer that never joins (NCCL >= 2.14)
    typedef int (*CommInitRankConfig)(void**, int, ncclUniqueId, int, ncclConfig_t*);
    typedef int (*CommGetAsyncError)(void*, int*);
    typedef int (*CommAbort)(void*);
    CommInitRankConfig init_config = nullptr;
    CommGetAsyncError async_error = nullptr;
    CommAbort abort_comm = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return false;
        get_unique_id = (GetUniqueId)dlsym(h, "ncclGetUniqueId");
        comm_init_rank = dlsym(h, "ncclCommInitRank");
        comm_destroy = (CommDestroy)dlsym(h, "ncclCommDestroy");
        send = (SendRecv)dlsym(h, "ncclSend");
        recv = dlsym(h, "ncclRecv");
        group_start = (Group)dlsym(h, "ncclGroupStart");
        group_end = (Group)dlsym(h, "ncclGroupEnd");
        err = (ErrStr)dlsym(h, "ncclGetErrorString");
        init_config = (CommInitRankConfig)dlsym(h, "ncclCommInitRankConfig");
        async_error = (CommGetAsyncError)dlsym(h, "ncclCommGetAsyncError");
        abort_comm = (CommAbort)dlsym(h, "ncclCommAbort");
        return get_unique_id && comm_init_rank && comm_destroy && send && recv && group_start &&
               group_end;
    }
};
NcclApi g_nccl;

struct NcclId {
    char b[128];
};
typedef int (*NcclInitFn)(void**, int, NcclId, int);
typedef int (*NcclRecvFn)(void*, size_t, int, int, void*, cudaStream_t);
constexpr int kNcclFloat = 7;  // ncclFloat32

void nccl_check(int r, const char* what) {
    if (r != 0 && r != ncclInProgress)
        throw Error(GP_ECUDA, std::string(what) + ": " + (g_nccl.err ? g_nccl.err(r) : "nccl error"));
}

// Seconds a non-blocking NCCL operation may stay in progress (GP_NCCL_TIMEOUT, default 120).
double nccl_timeout() {
    const char* e = std::getenv("GP_NCCL_TIMEOUT");
    return e ? std::atof(e) : 120.0;
}

// Poll a non-blocking communicator until its pending operation (init, or the enqueue of a
// grouped send/recv) leaves ncclInProgress; abort it and raise GP_EFABRIC on a timeout (a
// peer that never joins) and GP_ECUDA on an NCCL error (e.g. two ranks on one device).
void nccl_wait(void*& comm, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; ++spin) {
        int state = 0;
        const int r = g_nccl.async_error(comm, &state);
        if (r != 0) state = r;
        if (state == 0) return;
        if (state != ncclInProgress) {
            g_nccl.abort_comm(comm);
            comm = nullptr;
            throw Error(GP_ECUDA, std::string(what) + ": " + (g_nccl.err ? g_nccl.err(state) : "nccl error"));
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > nccl_timeout()) {
            g_nccl.abort_comm(comm);
            comm = nullptr;
            throw Error(GP_EFABRIC, std::string(what) + ": timed out after " + std::to_string(nccl_timeout()) +
                                        " s (GP_NCCL_TIMEOUT; the peer rank never joined)");
        }
        // an enqueue normally completes within microseconds: spin first, then back off
        if (spin < 1000) std::this_thread::yield();
        else std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

// One 2-rank communicator per stage boundary, created non-blocking.
void* nccl_comm_init(const uint8_t* id_bytes, int rank, const char* what) {
    if (!g_nccl.init_config || !g_nccl.async_error || !g_nccl.abort_comm)
        throw Error(GP_ECUDA, "libnccl.so.2 lacks the non-blocking communicator API (NCCL >= 2.14)");
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    void* comm = nullptr;
    const int r = g_nccl.init_config(&comm, 2, id, rank, &cfg);
    if (r != 0 && r != ncclInProgress) {
        if (comm) g_nccl.abort_comm(comm);
        throw Error(GP_ECUDA, std::string(what) + ": " + (g_nccl.err ? g_nccl.err(r) : "nccl error"));
    }
    nccl_wait(comm, what);
    return comm;
}

// ------------------------------------------------------------------ stream memory ops
// cuStreamWaitValue32 / cuStreamWriteValue32 (driver API, resolved through the
// runtime so nothing links libcuda directly): the IPC transport's flags are
// waited on and bumped in-stream, so no host thread sits in the data path.
struct MemOps {
    typedef CUresult (*Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    Fn wait = nullptr, write = nullptr;
    std::mutex mu;
    void load() {
        std::lock_guard<std::mutex> lk(mu);
        if (wait && write) return;
        for (int i = 0; i < 2; ++i) {
            void* f = nullptr;
            cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
            const char* sym = i == 0 ? "cuStreamWaitValue32" : "cuStreamWriteValue32";
            if (cudaGetDriverEntryPointByVersion(sym, &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !f)
                throw Error(GP_ECUDA, std::string(sym) + " unavailable");
            (i == 0 ? wait : write) = (Fn)f;
        }
    }
};
MemOps g_memops;


void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw Error(GP_ECUDA, std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}

// ------------------------------------------------------------------ transport
struct Piece {
    float* ptr;
    size_t floats;
};

struct Stage;

// One direction of one stage boundary inside a process: FIFO of posted chunk
// sends (the reference channel (src,dst,tag) is a FIFO deque, fabric.cpp:190).
struct LocalQueue {
    struct Msg {
        uint32_t chunk;
        cudaEvent_t ready;
        std::vector<Piece> src;
        int device;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Msg> q;
    bool aborted = false;
};

struct LocalLink {
    LocalQueue fwd, bwd;
};

// Hybrid group (G workers of one stage): one FIFO per (src, dst, kind).
// kind 0 = forward halo, 1 = backward halo, 2 = weight-gradient sync.
struct GroupLink {
    uint32_t G = 1;
    std::vector<Stage*> members;
    std::vector<LocalQueue> q;  // (src * G + dst) * 3 + kind
    explicit GroupLink(uint32_t g) : G(g), q(size_t(g) * g * 3) {}
    LocalQueue& at(uint32_t src, uint32_t dst, uint32_t kind) { return q[(size_t(src) * G + dst) * 3 + kind]; }
};

// Host copy of the renumbered graph, shared by the contexts that share the
// device graph (needed to derive each rank's halo lists).
struct HostGraph {
    std::vector<uint64_t> blk_nnz;  // (G*K row blocks) x (K column chunks) CSR entry counts
    std::vector<uint64_t> rp;       // renumbered row pointers
    std::vector<uint32_t> col;      // renumbered columns
    std::vector<uint32_t> part;     // new id -> partition
    std::vector<uint32_t> chunk;    // new id -> chunk
    std::vector<uint32_t> bstart;   // (G x (K+1)) block starts: rows of (rank r, chunk k)
};

// One stage boundary between processes over CUDA IPC (one process per GPU on a
// node; NVLink P2P between GPUs, plain device memory when both share one).
// Each side owns a region {ready @0, ack @128, ring of R message slots @4096}:
// the sender pushes a message into the receiver's ring with the copy engine
// (no SMs taken from the stage's kernels) and bumps the receiver's `ready`
// counter with an in-stream write; the receiver waits on `ready` in its compute
// stream, unpacks the slot and bumps the sender's `ack`, which the sender waits
// on before reusing a slot. Counters are message sequence numbers (1-based,
// monotone over the run), so each direction stays a FIFO like the reference
// channel (fabric.cpp:190).
constexpr size_t kIpcReady = 0, kIpcAck = 128, kIpcRing = 4096;
constexpr uint32_t kIpcMagic = 0x50495047u;  // "GPIP"

struct IpcBlob {
    uint32_t magic, version, stage, role;  // role 0: up boundary (receives fwd), 1: down (receives bwd)
    uint32_t n, K, R, pad0;
    uint64_t slot_floats, bytes, ptr;
    int32_t pid, device;
    cudaIpcMemHandle_t handle;
};
static_assert(sizeof(IpcBlob) <= GP_IPC_BLOB_BYTES, "IPC blob too large");

struct IpcSide {
    char* own = nullptr;  // own region (allocated by export)
    uint64_t own_slot = 0, own_bytes = 0;
    uint32_t own_R = 0;
    char* peer = nullptr;  // peer region (opened from the peer's blob)
    bool peer_opened = false;  // true: cudaIpcOpenMemHandle (close on destroy)
    uint64_t peer_slot = 0;
    uint32_t peer_R = 0;
    uint32_t send_seq = 0, recv_seq = 0;
    cudaStream_t stream = nullptr;   // send stream (copy engine work overlaps the next chunk)
    cudaStream_t rstream = nullptr;  // receive stream: waits/unpacks/acks in message order
    bool linked() const { return peer != nullptr; }
};

// Hybrid group across processes (gp_group_export / gp_link_group_ipc): every
// member maps its peers' activation, gradient-table and weight-gradient buffers
// (CUDA IPC; NVLink P2P between GPUs) and a small counter region. A halo message
// is "rows of chunk k of buffer X are final": the sender bumps a counter in each
// peer's region with an in-stream write, the receiver waits on it in-stream and
// pulls the halo rows straight from the peer's buffer (k_pull_rows). Buffers are
// matched by export index; all members swap cur/snapshot buffers at the same
// epochs, so "my current buffer j" is "peer's current buffer j".
constexpr uint32_t kGroupMagic = 0x52475047u;  // "GPGR"
constexpr uint32_t kGroupKinds = 5;            // 0 fwd halo, 1 bwd halo, 2 grads ready, 3 fold done, 4 copied
constexpr uint32_t kGroupMaxRanks = 8;

struct IpcGroup {
    bool linked = false;
    char* own_flags = nullptr;                  // kGroupKinds x kGroupMaxRanks u32 counters
    std::vector<char*> own_bufs;                // export order
    std::vector<std::vector<char*>> peer_bufs;  // [rank][export index]
    std::vector<char*> peer_flags;              // [rank]
    std::vector<char*> opened;                  // IPC mappings to close
    uint32_t post_seq[kGroupKinds] = {};
    uint32_t recv_seq[kGroupKinds][kGroupMaxRanks] = {};
    uint32_t sync_seq = 0;
    static size_t off(uint32_t kind, uint32_t src) { return (size_t(kind) * kGroupMaxRanks + src) * 4; }
};

struct Transport {
    // Forward: upstream stage sends chunk rows of its last layer (+h0).
    std::shared_ptr<LocalLink> up_local, down_local;  // links to s-1 and s+1
    std::shared_ptr<GroupLink> group;                 // hybrid peers (same stage)
    void* up_comm = nullptr;                          // NCCL 2-rank comms
    void* down_comm = nullptr;
    cudaStream_t up_stream = nullptr, down_stream = nullptr;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_next = 0;
    IpcSide ipc_up, ipc_down;  // cross-process boundaries (gp_link_ipc)
    IpcGroup ipcg;             // cross-process hybrid group (gp_link_group_ipc)
};

// ------------------------------------------------------------------ stage
struct LayerDev {
    gp_layer_spec spec;
    uint32_t l;          // global layer id
    uint32_t din, dout;  // in_dim, out_dim
    uint32_t sin, sout;  // padded strides
    // transform width and the stride of pre / bg: din, sin for Dense/GCN/GCNII;
    // SageConv (k_in = 2 din) keeps its two halves 32-byte aligned: own half at
    // column 0, aggregated half at sgap = pad8(din), so kw = sgap + din
    bool sage = false;
    uint32_t kin = 0, kw = 0, skw = 0, sgap = 0;
    float *Wg = nullptr, *WTg = nullptr;  // SageConv: W and W^T in the gapped layout
    bool agg;
    float *W = nullptr, *b = nullptr, *gW = nullptr, *gb = nullptr;
    float* WT = nullptr;  // W^T, refreshed whenever W changes (set_params, optimizer step)
    float *mW = nullptr, *vW = nullptr, *mb = nullptr, *vb = nullptr;
    float *h = nullptr, *hs = nullptr;   // h_cur / h_snap
    float *pre = nullptr, *dz = nullptr;
    float *G = nullptr;                  // masked gather source (input of this layer): rows of done chunks
    float *Gs = nullptr;                 // masked snapshot rows (rows of not-done chunks); == G if cur == snap
    float *bg = nullptr, *bgs = nullptr; // backward gather source (+ snapshot, hist mode)
    // tcgen05 row transforms (tc_xform.cuh): prepared W' operands, forward and backward
    bool tc = false;
    float *xf_fwd = nullptr, *xf_bwd = nullptr;
};

struct Stage {
    gp_stage_config cfg{};
    std::vector<gp_layer_spec> specs;
    uint32_t n = 0, K = 0, S = 1, s = 0, lb = 0, le = 0, len = 0, H = 0, C = 0;
    bool first = true, last = true, needs_h0 = false, sync = false, hist = false;
    int device = 0;
    std::string err;
    cudaStream_t cs = nullptr;       // compute stream (the current one: see the backward wavefront)
    static constexpr int kMaxWave = 16;
    cudaStream_t cs_side[kMaxWave] = {};  // extra compute streams of the chunk wavefront
    // streams in the chunk wavefront (GP_WAVE=1..16; default 12 from K = 32 on, 8 from 16, else
    // 4). Reddit shape, one B200: K = 32: 16 streams 0.428, 12: 0.429, 8: 0.433, 6: 0.443, 4:
    // 0.449, 3: 0.457 s/epoch (2: 0.466 in round 1); K = 16: 12: 0.407, 8: 0.404, 6: 0.405, 4:
    // 0.419; K = 8: 4 streams 0.376 vs 6: 0.388; K = 4: 4 = 6.
    int wave_w = 4;
    // GP_REMASK_OVERLAP=1 (default): the epoch-start snapshot remasks of layers >= 1 run on
    // their own stream, each waited for only by the kernels that write or read that layer's
    // gather table, so they overlap the first chunk's first layers instead of preceding them
    bool remask_overlap = true;
    cudaStream_t cs_prep = nullptr;
    // GP_MERGED_G=1: one gather table per layer (G == Gs). A row of G holds the
    // snapshot until its chunk rewrites it, so the forward gathers read a single
    // table (half the L2 footprint); the wavefront then also orders "chunk j+1
    // writes G_{i+1}" after "chunk j's layer i+1 gather" (wave_reads_done).
    bool merged_g = true;
    bool host_timing = false;  // GP_HOST_TIMING=1: per-epoch enqueue vs device time on stderr
    // GP_TC_MIX=1: Gcn2Conv identity mix in the tcgen05 epilogue from the unsplit input row
    // (forward h error vs fp64 3-8x lower: median 3-9e-8 vs 2e-7 of max|row|; 1.5 % slower
    // epoch: 0.366 vs 0.360 s at K = 4); 0 (default): folded into W' = beta W + (1 - beta) I
    bool tc_mix_epi = false;
    // GP_LEAN=1 (default): four N x H buffers per layer instead of seven. dz is written
    // in place over the layer's output h (the backward reads h[v] only for its own
    // ReLU mask, in the same lane, right before writing dz[v]); the backward gather
    // table bg_i lives in the forward gather table G_i (dead once the stage's forward
    // is complete, rebuilt at the next epoch start); snapshots are copies taken at
    // the end of epoch t when epoch t+1 refreshes (engines_impl.hpp:671-679), since
    // h no longer survives the backward. GP_LEAN=0 keeps h, dz, G and bg apart and
    // snapshots by pointer swap (the round-1 layout; tests that read activations
    // after an epoch use it).
    bool lean = true;
    // GP_TC_XFORM=1 (default): the GCN / GCNII row transforms (pre.W', dz.W'^T and their
    // epilogues) run on tcgen05 (3xTF32, fp32-level); 0: the bit-exact CUDA-core tiles
    bool use_tc_xform = true;
    // GP_XF_PAD: launches of at least this many rows stage A with the padded (conflict-free)
    // k-core stride (tc_xform.cuh); 1 (default) = always, 0 = never (the dense stride)
    uint32_t xf_pad_rows = 0;
    // GP_GRAPH_BUILD: where a single-partition upload of raw neighbour lists packs the
    // normalised CSR: "device" (k_build_edges), "host" (the builder hybrid groups and
    // precomputed values always use), default: the device from 64 MB of packed entries
    int graph_build = 0;  // 0 auto, 1 device, 2 host
    bool tc_dense = true;  // GP_TC_DENSE=0: Dense layers keep the fused CUDA-core GEMV kernels
    bool state_restored = false;  // gp_set_history: the snapshot rows were loaded
    // lean layout, epoch t with t % fix_alpha == 0 (the next epoch refreshes the snapshot):
    // tcgen05 forward epilogues write each row of h into hs as well (dual_done[i] marks the
    // layers), so copy_snapshots only copies the rest (single-process stages: hybrid halo rows
    // land in h outside the epilogue)
    bool dual_snap = false;
    std::vector<uint8_t> dual_done;
    // forward wavefront hooks (merged_g): after the kernel gathering from G_i, and
    // before the kernel writing rows of G_i
    std::function<void(uint32_t)> on_gather_done, before_g_write;
    std::vector<LayerDev> L;

    // graph (renumbered chunk-contiguous)
    std::shared_ptr<void> graph_owner;
    uint64_t* rowptr = nullptr;
    uint2* edges = nullptr;
    // SageConv mean adjacency (graph neighbours without the self loop): rowptr_m,
    // edges_m weighted 1/deg(row) (mean, graph.cpp:100-112), edges_mt weighted
    // 1/deg(col) (mean_t, nn.hpp:85-98); only when this stage has a SageConv layer
    bool has_sage = false;
    uint64_t* rowptr_m = nullptr;
    uint2* edges_m = nullptr;
    uint2* edges_mt = nullptr;
    uint32_t* orig = nullptr;          // new -> original id (device)
    // GP_BWD_CSR=1 (default): the backward gathers of a stale-mode epoch read a per-epoch
    // done-filtered copy of the own rows' CSR (k_done_csr) instead of filtering each batch
    bool bwd_csr = true;
    bool bwd_csr_ready = false;        // built for the current epoch's backward order
    uint64_t* rowptr_f = nullptr;
    uint2* edges_f = nullptr;
    unsigned long long* scan_tmp = nullptr;  // per-tile totals of the row-count scan
    uint32_t scan_tiles = 0;
    uint32_t* id_rows = nullptr;       // own rows in ascending original id (reductions)
    std::vector<uint32_t> perm;        // original -> new (host)
    std::vector<uint32_t> inv;         // new -> original (host)
    uint64_t nnz = 0;
    bool graph_ready = false;
    // hybrid: vertices renumbered by (partition, chunk, id); block (r, k) contiguous
    uint32_t G = 1, grank = 0;
    std::vector<uint32_t> part_host;             // original id -> partition (before upload)
    std::shared_ptr<HostGraph> hg;
    std::vector<uint32_t> bstart;                // (G x (K+1))
    uint32_t* pull_idx = nullptr;                // halo rows to pull, grouped by (peer, chunk)
    std::vector<uint32_t> pull_off;              // (G x (K+1)) offsets into pull_idx
    std::vector<uint64_t> push_cnt;              // (K x G) rows this rank pushes to each peer
    uint32_t row_begin(uint32_t k) const { return bstart[size_t(grank) * (K + 1) + k]; }
    uint32_t row_end(uint32_t k) const { return bstart[size_t(grank) * (K + 1) + k + 1]; }
    uint32_t own_begin() const { return row_begin(0); }
    uint32_t own_end() const { return row_begin(K); }

    // stage-level buffers
    float* x0 = nullptr;               // features (stage 0)
    uint32_t F = 0, sx = 0;
    float *in_cur = nullptr, *in_snap = nullptr;  // stage input (s > 0)
    uint32_t in0 = 0, sin0 = 0;
    float* h0 = nullptr;               // received h0 (s > 0, GCNII)
    float* dh0 = nullptr;              // dh0_run (GCNII)
    float* dtop = nullptr;             // incoming gradient of the last local layer
    float* dh_in = nullptr;            // gradient sent upstream (s > 0)
    uint32_t* labels = nullptr;
    uint8_t* split = nullptr;
    float inv_train = 0.f;
    bool labels_ready = false, x_ready = false;
    float* ws = nullptr;               // pgrad workspace
    float* wsb = nullptr;
    uint32_t splits = 1;
    double* part_loss = nullptr;
    unsigned long long* part_correct = nullptr;
    double* red_loss = nullptr;
    unsigned long long* red_correct = nullptr;
    uint32_t xent_blocks = 0;
    uint64_t step = 0;
    uint32_t last_epoch = 0;
    uint64_t dev_bytes = 0;
    std::vector<void*> allocs;

    Transport tr;
    // profiling
    bool profiling = false;
    // gp_set_live_timing: CUDA events around every launch of one kernel class during normal
    // (wavefront) epochs, accumulated like the profiling epoch's; -1 = off
    int live_cls = -1;

    // ---- trace (FabricOptions::collect_trace, fabric.cpp:222-227, :256-264) ----
    // Per epoch: one anchor (event + %globaltimer stamp) and a pair of timing
    // events per trace record; resolved to globaltimer nanoseconds after the
    // epoch's synchronize. Tracing runs the chunks serially (no wavefront), so a
    // stage's compute spans never overlap, as in the reference's worker clock.
    bool tracing = false;
    struct TraceRec {
        uint32_t epoch, kind;
        int32_t chunk, llo, lhi;
        cudaEvent_t a, b;
    };
    std::vector<TraceRec> trace_pending;
    std::vector<gp_trace_event> trace_done;
    cudaEvent_t trace_origin = nullptr;
    unsigned long long* trace_stamp = nullptr;  // mapped pinned host slot
    uint32_t trace_epoch = 0;
    gp_profile prof{};
    struct Timed {
        int cls;
        cudaEvent_t a, b;
        double bytes, flops, gather;
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> ev_free;
    uint64_t launches = 0;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    cudaEvent_t marks[16] = {};
    int num_sms = 148;
    std::map<std::pair<const void*, size_t>, int> occ_cache;
    std::atomic<bool> aborted{false};

    // ---- memory -----------------------------------------------------------
    // The stage's stash (every buffer alloc() lays out) is one cudaMalloc'd arena
    // carved in 256-byte aligned pieces: ~500 separate allocations of a Reddit-shape
    // stage cost 0.16-1.2 s to create and 0.14-0.5 s to free on the B200, the arena
    // ~10 ms each (tools/alloc_bench.cu). Hybrid workers (G > 1) export their layer
    // buffers over CUDA IPC, whose handles name whole allocations, so they keep one
    // allocation per buffer. Later allocations (graph, IPC rings, ...) are separate.
    bool arena_sizing = false;
    char* arena = nullptr;
    size_t arena_need = 0, arena_off = 0, arena_cap = 0;
    template <typename T>
    T* dalloc(size_t count, bool zero = true) {
        const size_t bytes = (std::max<size_t>(count * sizeof(T), 16) + 255) & ~size_t(255);
        if (arena_sizing) {
            arena_need += bytes;
            return reinterpret_cast<T*>(uintptr_t(256));  // layout pass: never dereferenced
        }
        if (arena && arena_off + bytes <= arena_cap) {  // zeroed with the arena
            char* p = arena + arena_off;
            arena_off += bytes;
            dev_bytes += bytes;
            return reinterpret_cast<T*>(p);
        }
        void* p = nullptr;
        GP_CUDA(cudaMalloc(&p, bytes));
        if (zero) GP_CUDA(cudaMemset(p, 0, bytes));
        allocs.push_back(p);
        dev_bytes += bytes;
        return static_cast<T*>(p);
    }

    ~Stage() {
        if (plan_only) return;  // gp_stage_footprint: nothing was created
        if (device >= 0) cudaSetDevice(device);
        if (tr.ipc_up.linked() || tr.ipc_down.linked() || tr.ipcg.linked) {
            // a dead peer leaves in-stream waits pending: bounded wait, then leak
            try {
                for (cudaStream_t st : {cs, tr.ipc_up.stream, tr.ipc_down.stream, tr.ipc_up.rstream, tr.ipc_down.rstream})
                    if (st) sync_watchdog(st, 30.0);
            } catch (...) {
                return;
            }
            for (char* p : tr.ipcg.opened) cudaIpcCloseMemHandle(p);
            for (IpcSide* x : {&tr.ipc_up, &tr.ipc_down}) {
                if (x->peer_opened) cudaIpcCloseMemHandle(x->peer);
                if (x->stream) cudaStreamDestroy(x->stream);
                if (x->rstream) cudaStreamDestroy(x->rstream);
            }
        }
        if (cs) cudaStreamSynchronize(cs);
        for (auto st : cs_side)
            if (st) cudaStreamSynchronize(st);
        for (void* p : allocs) cudaFree(p);
        for (auto& t : timed) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        for (auto e : ev_free) cudaEventDestroy(e);
        for (auto e : tr.ev_pool) cudaEventDestroy(e);
        for (auto e : marks)
            if (e) cudaEventDestroy(e);
        if (ev_start) cudaEventDestroy(ev_start);
        if (trace_origin) cudaEventDestroy(trace_origin);
        for (int i = 0; i < 2; ++i) {

            if (h2d_done[i]) cudaEventDestroy(h2d_done[i]);
        }
        if (trace_stamp) cudaFreeHost(trace_stamp);
        {
            std::vector<cudaEvent_t> used;
            for (const auto& r : trace_pending) used.insert(used.end(), {r.a, r.b});
            std::sort(used.begin(), used.end());
            used.erase(std::unique(used.begin(), used.end()), used.end());
            for (auto e : used) cudaEventDestroy(e);
        }
        if (ev_end) cudaEventDestroy(ev_end);
        if (tr.up_comm) g_nccl.comm_destroy(tr.up_comm);
        if (tr.down_comm) g_nccl.comm_destroy(tr.down_comm);
        if (tr.up_stream) cudaStreamDestroy(tr.up_stream);
        if (tr.down_stream) cudaStreamDestroy(tr.down_stream);
        if (cs) cudaStreamDestroy(cs);
        for (auto st : cs_side)
            if (st) cudaStreamDestroy(st);
        if (cs_prep) cudaStreamDestroy(cs_prep);
    }

    // ---- configuration ------------------------------------------------------
    void init(const gp_stage_config& c) {
        cfg = c;
        if (!c.specs || c.num_layers == 0) throw Error(GP_EINVAL, "gp_create: no layer specs");
        specs.assign(c.specs, c.specs + c.num_layers);
        cfg.specs = nullptr;
        n = c.num_vertices;
        K = c.num_chunks;
        S = c.num_stages;
        s = c.stage;
        lb = c.layer_begin;
        le = c.layer_end;
        H = c.hidden;
        C = c.num_classes;
        if (n == 0 || n > kColMask) throw Error(GP_EINVAL, "num_vertices must be in [1, 2^26)");
        if (K == 0 || K > kMaxChunks || K > n)
            throw Error(GP_EINVAL, "num_chunks must be in [1, min(64, N)]");
        if (S == 0 || s >= S) throw Error(GP_EINVAL, "bad stage index");
        if (lb >= le || le > c.num_layers) throw Error(GP_EINVAL, "bad layer range");
        if (c.dropout >= 1.0) throw Error(GP_EINVAL, "dropout rate must be < 1");
        len = le - lb;
        first = s == 0;
        last = s + 1 == S;
        sync = c.synchronous_mode != 0;
        hist = c.historical_gradients != 0 && !sync;
        G = c.group_size ? c.group_size : 1;
        grank = c.group_rank;
        if (G > 8 || grank >= G) throw Error(GP_EINVAL, "group_size must be in [1, 8] and group_rank < group_size");
        needs_h0 = false;
        has_sage = false;
        for (uint32_t l = 0; l < c.num_layers; ++l) {
            const auto& sp = specs[l];
            if (sp.kind > GP_GCN2CONV) throw Error(GP_EINVAL, "unknown layer kind");
            if (sp.kind == GP_GCN2CONV) needs_h0 = true;
            if (sp.kind == GP_SAGECONV && l >= c.layer_begin && l < c.layer_end) {
                if (sp.in_dim > kMaxWidth && l > 0)  // layer 0 (features) takes the wide path
                    throw Error(GP_EINVAL, "SageConv hidden width > 128 is not supported by the GPU engine");
                has_sage = true;
            }
        }
        if (first != (lb == 0)) throw Error(GP_EINVAL, "stage 0 must own layer 0");
        if (last != (le == c.num_layers)) throw Error(GP_EINVAL, "last stage must own layer L-1");
        for (uint32_t l = lb; l < le; ++l) {
            const auto& sp = specs[l];
            if (sp.out_dim == 0 || sp.out_dim > kMaxWidth)
                throw Error(GP_EINVAL, "layer output width must be in [1, 128]");
            if (l > 0 && sp.in_dim > kMaxWidth)
                throw Error(GP_EINVAL, "hidden width must be <= 128");
            if (sp.kind == GP_GCN2CONV && sp.in_dim != sp.out_dim)
                throw Error(GP_EINVAL, "Gcn2Conv needs in_dim == out_dim");
        }
        if (needs_h0 && (H == 0 || H > kMaxWidth)) throw Error(GP_EINVAL, "bad hidden width");
        if (const char* e = std::getenv("GP_MERGED_G")) merged_g = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_BWD_CSR")) bwd_csr = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_HOST_TIMING")) host_timing = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_TC_MIX")) tc_mix_epi = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_LEAN")) lean = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_TC_XFORM")) use_tc_xform = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_TC_DENSE")) tc_dense = std::atoi(e) != 0;
        if (plan_only) return;
        device = c.device;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error(GP_ECUDA, "no CUDA device (the GPU engine has no CPU fallback)");
        if (device < 0 || device >= ndev) throw Error(GP_EINVAL, "bad device ordinal");
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
        GP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        wave_w = K >= 32 ? 12 : (K >= 16 ? 8 : 4);
        if (const char* e = std::getenv("GP_WAVE")) wave_w = std::max(1, std::min(kMaxWave, std::atoi(e)));
        for (int w = 1; w < wave_w; ++w) GP_CUDA(cudaStreamCreateWithFlags(&cs_side[w], cudaStreamNonBlocking));
        if (const char* e = std::getenv("GP_REMASK_OVERLAP")) remask_overlap = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_FUSED_STEP")) fused_step = std::atoi(e) != 0;
        if (const char* e = std::getenv("GP_GRAPH_BUILD"))
            graph_build = std::string(e) == "device" ? 1 : std::string(e) == "host" ? 2 : 0;
        if (const char* e = std::getenv("GP_XF_PAD")) {
            const long v = std::atol(e);
            xf_pad_rows = v == 0 ? UINT32_MAX : v == 1 ? 0u : uint32_t(v);
        }
        if (remask_overlap) GP_CUDA(cudaStreamCreateWithFlags(&cs_prep, cudaStreamNonBlocking));
        GP_CUDA(cudaEventCreate(&ev_start));
        GP_CUDA(cudaEventCreate(&ev_end));
        alloc();
        setup_kernels();
    }

    // Device footprint of this configuration without a device: the stash layout pass
    // (alloc_layout in sizing mode) plus the graph, features and labels the uploads
    // allocate (CSR: u64 row pointers + 8-byte packed entries; SageConv mean CSRs).
    bool plan_only = false;
    uint64_t plan_bytes(const gp_stage_config& c, uint64_t nnz_norm, uint32_t F_in) {
        plan_only = true;
        init(c);
        arena_sizing = true;
        arena_need = 0;
        alloc_layout();
        arena_sizing = false;
        uint64_t b = arena_need;
        auto add = [&](uint64_t bytes) { b += (std::max<uint64_t>(bytes, 16) + 255) & ~uint64_t(255); };
        add(8ull * (n + 1));                                  // rowptr
        add(8ull * nnz_norm);                                 // packed {col | chunk, weight}
        add(4ull * n);                                        // new -> original id
        if (has_sage) {
            const uint64_t nnz_m = nnz_norm >= n ? nnz_norm - n : nnz_norm;  // no self loops
            add(8ull * (n + 1));
            add(2 * 8ull * nnz_m);
        }
        if (needs_bwd_csr()) {  // done-filtered backward CSR (own rows; hybrid: a 1/G share)
            add(8ull * (n + 1));
            add(8ull * ((nnz_norm + G - 1) / G));
        }
        if (first) add(4ull * n * pad8(F_in ? F_in : specs[0].in_dim));  // x0
        if (last) add(5ull * n);                              // labels + split
        return b;
    }

    void alloc() {
        if (G == 1) {
            arena_sizing = true;
            arena_need = 0;
            alloc_layout();
            arena_sizing = false;
            GP_CUDA(cudaMalloc(reinterpret_cast<void**>(&arena), arena_need));
            GP_CUDA(cudaMemset(arena, 0, arena_need));
            allocs.push_back(arena);
            arena_cap = arena_need;
            arena_off = 0;
            L.clear();
        }
        alloc_layout();
        arena_cap = arena_off;  // nothing else is carved from it
    }

    void alloc_layout() {
        in0 = specs[lb].in_dim;
        sin0 = pad8(in0);
        L.resize(len);
        for (uint32_t i = 0; i < len; ++i) {
            auto& d = L[i];
            d.spec = specs[lb + i];
            d.l = lb + i;
            d.din = d.spec.in_dim;
            d.dout = d.spec.out_dim;
            d.sin = pad8(d.din);
            d.sout = pad8(d.dout);
            d.agg = d.spec.kind != GP_DENSE;
            d.sage = d.spec.kind == GP_SAGECONV;
            d.kin = d.sage ? 2 * d.din : d.din;
            d.sgap = d.sage ? d.sin : 0;
            d.kw = d.sage ? d.sgap + d.din : d.din;
            d.skw = pad8(d.kw);
            const bool bias = d.spec.kind != GP_GCN2CONV;
            const size_t wn = size_t(d.kin) * d.dout;
            d.W = dalloc<float>(wn);
            d.WT = dalloc<float>(wn);
            if (d.sage) {
                d.Wg = dalloc<float>(size_t(d.kw) * d.dout);
                d.WTg = dalloc<float>(size_t(d.kw) * d.dout);
            }
            d.gW = dalloc<float>(wn);
            d.mW = dalloc<float>(wn);
            d.vW = dalloc<float>(wn);
            if (bias) {
                d.b = dalloc<float>(d.dout);
                d.gb = dalloc<float>(d.dout);
                d.mb = dalloc<float>(d.dout);
                d.vb = dalloc<float>(d.dout);
            }
            if (use_tc_xform && (d.agg || tc_dense) && !d.sage && d.din <= kMaxWidth && d.dout <= kMaxWidth) {
                d.tc = true;
                d.xf_fwd = dalloc<float>(2 * size_t(xf_pad8k(d.din)) * xf_pad16(d.dout));
                d.xf_bwd = dalloc<float>(2 * size_t(xf_pad8k(d.dout)) * xf_pad16(d.din));
            }
            d.h = dalloc<float>(size_t(n) * d.sout);
            if (G == 1 || arena_sizing) d.pre = own_rows_alloc(d.skw);  // G > 1: at graph upload
            d.dz = lean ? d.h : dalloc<float>(size_t(n) * d.sout);
            // gather tables carry one extra all-zero row (row n, see gather_row)
            if (d.agg) {
                d.G = dalloc<float>(size_t(n + 1) * d.sin);
                // stage 0's layer-0 input is x0 (cur == snap); sync mode never reads snapshots
                d.Gs = (first && i == 0) || sync || merged_g ? d.G : dalloc<float>(size_t(n + 1) * d.sin);
            }
            if (!sync && i + 1 < len && specs[lb + i + 1].kind != GP_DENSE)
                d.hs = dalloc<float>(size_t(n) * d.sout);
            if (d.l > 0) {
                // lean: bg_i in G_i's rows (same width for non-SageConv layers; the
                // historical-gradient ablation swaps bg with its snapshot, so it keeps its own)
                d.bg = lean && d.agg && !d.sage && !hist && d.skw == d.sin ? d.G
                                                                        : dalloc<float>(size_t(n + 1) * d.skw);
                if (hist && d.agg) d.bgs = dalloc<float>(size_t(n + 1) * d.skw);
            }
        }
        if (!first) {
            in_cur = dalloc<float>(size_t(n) * sin0);
            if (!sync && L[0].agg) in_snap = dalloc<float>(size_t(n) * sin0);
        }
        if (G == 1 || arena_sizing) alloc_own_stage_rows();  // G > 1: at graph upload
        // pgrad workspace: ~2 waves of CTAs
        splits = std::max<uint32_t>(1, std::min<uint32_t>(2 * num_sms, (n + 63) / 64));
        size_t wmax = 1;
        for (auto& d : L) wmax = std::max(wmax, size_t(d.din) * d.dout);  // per half for SageConv
        ws = dalloc<float>(size_t(splits) * wmax, false);
        wsb = dalloc<float>(size_t(splits) * kMaxWidth, false);
        xent_blocks = uint32_t(std::min<uint64_t>(2ull * num_sms, (n + kWarpsPerBlock - 1) / kWarpsPerBlock));
        part_loss = dalloc<double>(xent_blocks);
        part_correct = dalloc<unsigned long long>(3ull * xent_blocks);
        red_loss = dalloc<double>(1);
        red_correct = dalloc<unsigned long long>(3);
        tickets = dalloc<uint32_t>(kTickets);
        if (!arena_sizing) GP_CUDA(cudaDeviceSynchronize());
    }

    // ---- owner-row buffers ---------------------------------------------------
    // pre, the received h0, dh0 and the incoming / outgoing chunk gradients are only ever
    // touched at this worker's own rows. A hybrid worker (G > 1) allocates them for its own
    // rows [own_begin, own_end) only, once the partition is known (graph upload), and keeps
    // a base pointer offset by own_begin rows, so every kernel indexes them by global row as
    // before. The layout pass (gp_stage_footprint) sizes them at the partitioner's balance
    // cap max(ceil(N/G), floor(1.05 N/G)) (partition.cpp:183-187).
    uint32_t own_rows_planned() const {
        if (G == 1) return n;
        if (graph_ready || !bstart.empty()) return own_end() - own_begin();
        return std::min<uint32_t>(n, std::max<uint32_t>((n + G - 1) / G, uint32_t(1.05 * double(n) / G)));
    }
    float* own_rows_alloc(uint32_t stride) {
        const uint32_t rows = own_rows_planned();
        float* base = dalloc<float>(size_t(rows) * stride);
        if (arena_sizing || G == 1) return base;
        return base - size_t(own_begin()) * stride;
    }
    void alloc_own_stage_rows() {
        if (!first) {
            dh_in = own_rows_alloc(sin0);
            if (needs_h0) h0 = own_rows_alloc(pad8(H));
        }
        if (needs_h0) dh0 = own_rows_alloc(pad8(H));
        // lean: a chunk's incoming gradient (dtop, read first in its backward) and its
        // outgoing one (dh_in, written last) share rows when their strides agree
        dtop = lean && dh_in && L[len - 1].sout == sin0 ? dh_in : own_rows_alloc(L[len - 1].sout);
    }
    // G > 1, after the partition renumbering: the owner-row buffers
    void ensure_own_buffers() {
        if (G == 1 || dtop) return;
        for (auto& d : L) d.pre = own_rows_alloc(d.skw);
        alloc_own_stage_rows();
    }
    bool own_only(const float* p) const {
        if (G == 1 || !p) return false;
        if (p == dh0 || p == h0 || p == dh_in || p == dtop) return true;
        for (const auto& d : L)
            if (p == d.pre) return true;
        return false;
    }

    // Work counters of the dynamically scheduled row kernels (one per launch).
    uint32_t* tickets = nullptr;
    uint32_t ticket_next = 0;
    static constexpr uint32_t kTickets = 16384;
    uint32_t* take_ticket() {
        if (ticket_next == kTickets) {
            zero_words(tickets, kTickets);
            ticket_next = 0;
        }
        return tickets + ticket_next++;
    }

    // Gathers in flight per lane (template NB of the row kernels); GP_NB overrides.
    int nb = 2;
    // Aggregating layers run as two kernels (default): the gather (-> pre / dz)
    // and the register-tiled row transform + epilogue (k_fwd_tile / k_bwd_tile,
    // dense_tile.cuh). GP_SPLIT=0: one fused kernel with a 2-rows-per-warp GEMV
    // (its shared-memory wavefronts compete with the gather). Reddit shape, one
    // B200: split 0.439 vs fused 0.450 s/epoch at K = 4, 0.465 vs 0.519 at K = 32.
    bool split_rows = true;

    // Row kernels stage a weight matrix (+ x rows; <= 100 KB) in shared memory;
    // gathers bypass L1 (no_allocate), so the unified carveout goes to shared memory.
    template <int NB>
    void setup_nb() {
        const int smem_max = int(row_smem_bytes(kMaxWidth, kMaxWidth, 2));
        const void* fns[] = {(const void*)k_fwd8<FWD_DENSE, NB>,
                             (const void*)k_fwd8<FWD_GCN, NB>,
                             (const void*)k_fwd8<FWD_GCN2, NB>,
                             (const void*)k_fwd8<FWD_GCN, NB, true>,
                             (const void*)k_fwd8<FWD_GCN2, NB, true>,
                             (const void*)k_fwd8<FWD_SAGE, NB, true>,
                             (const void*)k_fwd8<FWD_GCN, NB, true, 5>,
                             (const void*)k_fwd8<FWD_GCN2, NB, true, 5>,
                             (const void*)k_fwd8<FWD_SAGE, NB, true, 5>,
                             (const void*)k_bwd8<PREV_TOP, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_AGG, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_AGG_HIST, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_OWN, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_SAGE, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_SAGE_HIST, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_TOP, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_OWN, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_SAGE, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_SAGE_HIST, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_SAGE, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_SAGE_HIST, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_SAGE, OUT_DHIN, NB>,
                             (const void*)k_bwd8<PREV_AGG_ALL, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_AGG_ALL, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_AGG_ALL, OUT_LAYER, NB, true, 5>,
                             (const void*)k_bwd8<PREV_AGG_ALL, OUT_DHIN, NB>,
                             (const void*)k_bwd8<PREV_SAGE_HIST, OUT_DHIN, NB>,
                             (const void*)k_bwd8<PREV_TOP, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_AGG, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_AGG_HIST, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_OWN, OUT_LAYER, NB>,
                             (const void*)k_bwd8<PREV_AGG, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_AGG_HIST, OUT_LAYER, NB, true>,
                             (const void*)k_bwd8<PREV_AGG, OUT_DHIN, NB>,
                             (const void*)k_bwd8<PREV_AGG_HIST, OUT_DHIN, NB>,
                             (const void*)k_bwd8<PREV_OWN, OUT_DHIN, NB>};
        for (const void* f : fns) {
            GP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
            GP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         int(cudaSharedmemCarveoutMaxShared)));
        }
        const void* tiles[] = {(const void*)k_fwd_tile<false, 1>,      (const void*)k_fwd_tile<true, 1>,
                               (const void*)k_fwd_tile<false, 2>,      (const void*)k_fwd_tile<true, 2>,
                               (const void*)k_fwd_tile<false, 4>,      (const void*)k_fwd_tile<true, 4>,
                               (const void*)k_bwd_tile<1>,             (const void*)k_bwd_tile<2>,
                               (const void*)k_bwd_tile<4>,             (const void*)k_fwd_tile<false, 4, 100>,
                               (const void*)k_fwd_tile<true, 4, 100>,  (const void*)k_fwd_tile<false, 4, 128>,
                               (const void*)k_fwd_tile<true, 4, 128>,  (const void*)k_bwd_tile<4, 100>,
                               (const void*)k_bwd_tile<4, 128>};
        GP_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        for (const void* f : tiles) {
            GP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
            GP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         int(cudaSharedmemCarveoutMaxShared)));
        }
    }

    // Parameter gradients on tcgen05 (default) or CUDA cores (GP_PGRAD=simt).
    bool use_tc_pgrad = true;

    // Load every kernel now. With CUDA's lazy module loading the first launch of a
    // kernel loads it, and loading synchronises the context: if another stage of
    // this process has an in-stream wait pending on a value this stage has yet to
    // write (gp_link_ipc peers in one process), that first launch never returns.
    void preload_kernels() {
        const void* fns[] = {(const void*)k_adam,        (const void*)k_copy,          (const void*)k_dense_gemm,
                             (const void*)k_group_fold,  (const void*)k_pgrad_fold,    (const void*)k_pgrad_partial,
                             (const void*)k_pgrad_tc,    (const void*)k_pull_rows,     (const void*)k_remask,
                             (const void*)k_spmm_pre,    (const void*)k_stamp,         (const void*)k_transpose,
                             (const void*)k_xent_fold,   (const void*)k_xent_grad,     (const void*)k_xent_stats,
                             (const void*)k_zero,        (const void*)k_sage_weights,  (const void*)k_tc_prep,
                             (const void*)k_tc_xform<false>, (const void*)k_tc_xform<true>};
        for (const void* f : fns) {
            cudaFuncAttributes a;
            GP_CUDA(cudaFuncGetAttributes(&a, f));
        }
    }

    void zero_words(uint32_t* p, size_t words) {
        const uint32_t blocks = uint32_t(std::min<size_t>(size_t(num_sms) * 4, (words + 255) / 256));
        k_zero<<<std::max<uint32_t>(blocks, 1), 256, 0, cs>>>(p, words);
        GP_CUDA(cudaGetLastError());
    }

    void setup_kernels() {
        preload_kernels();
        if (const char* e = std::getenv("GP_PGRAD")) use_tc_pgrad = std::string(e) != "simt";
        GP_CUDA(cudaFuncSetAttribute(k_pgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GP_CUDA(cudaFuncSetAttribute(k_tc_xform<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kXfSmemMax)));
        GP_CUDA(cudaFuncSetAttribute(k_tc_xform<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kXfSmemMax)));
        if (const char* e = std::getenv("GP_NB")) {
            const int v = std::atoi(e);
            if (v == 2 || v == 4) nb = v;
        }
        if (const char* e = std::getenv("GP_SPLIT")) split_rows = std::string(e) != "0";
        if (const char* e = std::getenv("GP_IPC_SMCOPY")) ipc_smcopy = std::string(e) == "1";
        if (const char* e = std::getenv("GP_OCC5")) occ5_mode = std::string(e) == "auto" ? -1 : (std::atoi(e) ? 1 : 0);
        if (const char* e = std::getenv("GP_TILE_TR")) {
            const int v = std::atoi(e);
            if (v == 1 || v == 2 || v == 4) tile_tr_env = v;
        }
        setup_nb<2>();
        setup_nb<4>();
    }

    // Split gather kernels: 5 resident CTAs (48 registers) by default; GP_OCC5=0 forces the
    // 4-CTA (64-register) build, GP_OCC5=auto takes 5 CTAs for launches with enough row pairs
    // to keep every warp busy. With the single-table gather and tcgen05 transforms (Dense
    // layers too) co-running in the wavefront: 5 CTAs 0.371 vs 0.374 s/epoch at K = 4 (3 runs
    // each), 0.448 vs 0.466 at K = 32.
    int occ5_mode = 1;
    bool use_occ5(uint32_t rows) const {
        if (occ5_mode >= 0) return occ5_mode == 1;
        return uint64_t(rows) / 2 >= 2ull * uint64_t(num_sms) * 5 * kWarpsPerBlock;
    }
    template <int KIND, int NB, bool SPLIT = false>
    void fwd_go(uint32_t rows, size_t smem, const FwdParams& p) {
        if (SPLIT && NB == 2 && use_occ5(rows)) {
            k_fwd8<KIND, NB, SPLIT, 5><<<row_grid(rows, (const void*)k_fwd8<KIND, NB, SPLIT, 5>, smem, 16), kBlock, smem, cs>>>(p);
            return;
        }
        k_fwd8<KIND, NB, SPLIT><<<row_grid(rows, (const void*)k_fwd8<KIND, NB, SPLIT>, smem, 16), kBlock, smem, cs>>>(p);
    }
    template <int KIND, bool SPLIT = false>
    void fwd_nb(uint32_t rows, size_t smem, const FwdParams& p) {
        if (nb == 2) fwd_go<KIND, 2, SPLIT>(rows, smem, p);
        else fwd_go<KIND, 4, SPLIT>(rows, smem, p);
    }
    // Split-path transforms: register-tiled (dense_tile.cuh), one tile of
    // tile_geom(width).tm rows per CTA iteration.
    uint32_t tile_grid(uint32_t rows, const void* fn, size_t smem, uint32_t tm) {
        auto key = std::make_pair(fn, smem);
        auto it = occ_cache.find(key);
        int occ = 0;
        if (it == occ_cache.end()) {
            GP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTileThreads, smem));
            occ_cache[key] = occ = std::max(occ, 1);
        } else {
            occ = it->second;
        }
        const uint64_t want = (uint64_t(rows) + tm - 1) / tm;
        return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(num_sms) * occ)));
    }
    template <bool GCN2, int TR, int WIDTH = 0>
    void fwd_tile_go(uint32_t rows, const FwdParams& p) {
        const size_t smem = tile_smem_bytes(p.din, p.dout, TR);
        const void* fn = (const void*)k_fwd_tile<GCN2, TR, WIDTH>;
        k_fwd_tile<GCN2, TR, WIDTH>
            <<<tile_grid(rows, fn, smem, tile_geom(p.din, p.dout, TR).tm), kTileThreads, smem, cs>>>(p);
    }
    // compile-time geometry for the square H = 100 / 128 transforms (TR = 4)
    static int square_width(uint32_t a, uint32_t b) { return a == b && (a == 100 || a == 128) ? int(a) : 0; }
    int smem_optin = 227 * 1024;
    // rows per thread for a tile launch: by launch size, then down until the
    // staged matrix + double-buffered row tiles fit (SageConv's 2*din-wide transforms)
    int tile_tr_env = 0;  // GP_TILE_TR=1/2/4 forces rows per thread (experiments)
    int tile_tr(uint32_t rows, uint32_t win, uint32_t wout) const {
        int tr = tile_tr_env ? tile_tr_env : tile_rows_per_thread(rows, wout, num_sms);
        // two resident CTAs (one stages rows while the other computes): H = 128 at 4 rows per
        // thread needs 139 KB and would run one CTA per SM
        while (tr > 1 && tile_smem_bytes(win, wout, uint32_t(tr)) > size_t(smem_optin) / 2) tr /= 2;
        if (tile_smem_bytes(win, wout, uint32_t(tr)) > size_t(smem_optin))
            throw Error(GP_EINVAL, "row transform too wide for shared memory");
        return tr;
    }
    template <bool GCN2>
    void fwd_dense_go(uint32_t rows, const FwdParams& p) {
        switch (tile_tr(rows, p.din, p.dout)) {
            case 4:
                if (square_width(p.din, p.dout) == 100) fwd_tile_go<GCN2, 4, 100>(rows, p);
                else if (square_width(p.din, p.dout) == 128) fwd_tile_go<GCN2, 4, 128>(rows, p);
                else fwd_tile_go<GCN2, 4>(rows, p);
                break;
            case 2: fwd_tile_go<GCN2, 2>(rows, p); break;
            default: fwd_tile_go<GCN2, 1>(rows, p); break;
        }
    }
    template <int TR, int WIDTH = 0>
    void bwd_tile_go(uint32_t rows, const BwdParams& p) {
        const size_t smem = tile_smem_bytes(p.dout, p.din, TR);
        const void* fn = (const void*)k_bwd_tile<TR, WIDTH>;
        k_bwd_tile<TR, WIDTH><<<tile_grid(rows, fn, smem, tile_geom(p.dout, p.din, TR).tm), kTileThreads, smem, cs>>>(p);
    }
    void bwd_dense_go(uint32_t rows, const BwdParams& p) {
        switch (tile_tr(rows, p.dout, p.din)) {
            case 4:
                if (square_width(p.din, p.dout) == 100) bwd_tile_go<4, 100>(rows, p);
                else if (square_width(p.din, p.dout) == 128) bwd_tile_go<4, 128>(rows, p);
                else bwd_tile_go<4>(rows, p);
                break;
            case 2: bwd_tile_go<2>(rows, p); break;
            default: bwd_tile_go<1>(rows, p); break;
        }
    }
    template <int PREV, int OUT, int NB, bool SPLIT = false>
    void bwd_go(uint32_t rows, size_t smem, const BwdParams& p) {
        if (SPLIT && NB == 2 && use_occ5(rows)) {
            k_bwd8<PREV, OUT, NB, SPLIT, 5>
                <<<row_grid(rows, (const void*)k_bwd8<PREV, OUT, NB, SPLIT, 5>, smem, 16), kBlock, smem, cs>>>(p);
            return;
        }
        k_bwd8<PREV, OUT, NB, SPLIT>
            <<<row_grid(rows, (const void*)k_bwd8<PREV, OUT, NB, SPLIT>, smem, 16), kBlock, smem, cs>>>(p);
    }
    template <int PREV, int OUT, bool SPLIT = false>
    void bwd_nb(uint32_t rows, size_t smem, const BwdParams& p) {
        if (nb == 2) bwd_go<PREV, OUT, 2, SPLIT>(rows, smem, p);
        else bwd_go<PREV, OUT, 4, SPLIT>(rows, smem, p);
    }

    // ---- graph --------------------------------------------------------------
    // Bulk host->device copy through two pinned 32 MB staging buffers (host memcpy
    // of one chunk overlaps the DMA of the previous one): pageable cudaMemcpy runs at
    // ~1.5 GB/s here, the staged path at PCIe rate. Synchronous on return.
    static constexpr size_t kStageChunk = size_t(32) << 20;
    // The two pinned buffers are process-wide (allocating 64 MB of pinned memory costs tens
    // of ms per engine); an upload holds them through a StagingLease.
    struct StagingPool {
        std::mutex mu;
        char* buf[2] = {nullptr, nullptr};
    };
    static StagingPool& staging_pool() {
        static StagingPool* pool = new StagingPool;  // never freed: lives until process exit
        return *pool;
    }
    struct StagingLease {
        std::unique_lock<std::mutex> lk;
        char* buf[2];
        StagingLease() : lk(staging_pool().mu) {
            for (int i = 0; i < 2; ++i) {
                if (!staging_pool().buf[i]) GP_CUDA(cudaMallocHost(&staging_pool().buf[i], kStageChunk));
                buf[i] = staging_pool().buf[i];
            }
        }
    };
    cudaEvent_t h2d_done[2] = {nullptr, nullptr};
    void h2d(void* dst, const void* src, size_t bytes) {
        if (bytes < (size_t(4) << 20)) {
            GP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
            return;
        }
        StagingLease lease;
        char* const* h2d_stage = lease.buf;
        for (int i = 0; i < 2; ++i)
            if (!h2d_done[i]) GP_CUDA(cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming));
        const char* s8 = static_cast<const char*>(src);
        char* d8 = static_cast<char*>(dst);
        bool used[2] = {false, false};
        for (size_t off = 0, j = 0; off < bytes; off += kStageChunk, ++j) {
            const int b = int(j & 1);
            const size_t len = std::min(kStageChunk, bytes - off);
            if (used[b]) GP_CUDA(cudaEventSynchronize(h2d_done[b]));  // buffer b's previous DMA is done
            std::memcpy(h2d_stage[b], s8 + off, len);
            GP_CUDA(cudaMemcpyAsync(d8 + off, h2d_stage[b], len, cudaMemcpyHostToDevice, cs));
            GP_CUDA(cudaEventRecord(h2d_done[b], cs));
            used[b] = true;
        }
        GP_CUDA(cudaStreamSynchronize(cs));
    }

    // Fill a device CSR-entry array row by row: rows are grouped into chunks of at
    // most kStageChunk bytes, each chunk is filled in a pinned staging buffer by
    // `nth` threads (fill(r, out) writes row r's entries) and DMA'd while the next
    // chunk is filled.
    template <class T, class Fill>
    void stage_rows_h2d(T* dst, const std::vector<uint64_t>& rp, unsigned nth, Fill&& fill) {
        const uint32_t rows = uint32_t(rp.size() - 1);
        if (rp[rows] == 0) return;
        if (rp[rows] * sizeof(T) < (size_t(4) << 20)) {  // small graphs: no pinned staging (its
            std::vector<T> tmp(rp[rows]);                  // allocation costs more than the copy)
            for (uint32_t r = 0; r < rows; ++r) fill(r, tmp.data() + rp[r]);
            GP_CUDA(cudaMemcpy(dst, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice));
            return;
        }
        StagingLease lease;
        char* const* h2d_stage = lease.buf;
        for (int i = 0; i < 2; ++i)
            if (!h2d_done[i]) GP_CUDA(cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming));
        const uint64_t cap = kStageChunk / sizeof(T);
        bool used[2] = {false, false};
        uint32_t r0 = 0;
        for (uint32_t j = 0; r0 < rows; ++j) {
            uint32_t r1 = r0;
            while (r1 < rows && rp[r1 + 1] - rp[r0] <= cap) ++r1;
            if (r1 == r0) {  // one row larger than a chunk: copy it on its own
                std::vector<T> tmp(rp[r0 + 1] - rp[r0]);
                fill(r0, tmp.data());
                GP_CUDA(cudaMemcpy(dst + rp[r0], tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice));
                r0 = r0 + 1;
                continue;
            }
            const int b = int(j & 1);
            if (used[b]) GP_CUDA(cudaEventSynchronize(h2d_done[b]));
            T* buf = reinterpret_cast<T*>(h2d_stage[b]);
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < nth; ++t)
                pool.emplace_back([&, t]() {
                    for (uint32_t r = r0 + t; r < r1; r += nth) fill(r, buf + (rp[r] - rp[r0]));
                });
            for (auto& th : pool) th.join();
            GP_CUDA(cudaMemcpyAsync(dst + rp[r0], buf, (rp[r1] - rp[r0]) * sizeof(T), cudaMemcpyHostToDevice, cs));
            GP_CUDA(cudaEventRecord(h2d_done[b], cs));
            used[b] = true;
            r0 = r1;
        }
        GP_CUDA(cudaStreamSynchronize(cs));
    }

    void upload_partition(const uint32_t* part_of) {
        if (!part_of) throw Error(GP_EINVAL, "null partition");
        if (graph_ready) throw Error(GP_EINVAL, "upload the partition before the graph");
        part_host.assign(part_of, part_of + n);
        for (uint32_t p : part_host)
            if (p >= G) throw Error(GP_EINVAL, "partition id >= group_size");
    }

    // Vertex renumbering: (partition, chunk, original id) order, so that the rows
    // of (rank r, chunk k) form the contiguous block [bstart(r,k), bstart(r,k+1)):
    // stage messages (engines_impl.hpp:690-724) are slices, and a rank's own rows
    // (Partition::inner_sets[r]) are one range. Row content keeps the original
    // ascending neighbour order, so every reduction stays bit-exact.
    // Rows of the normalised adjacency, from an uploaded CSR (off, cols, vals) ...
    struct NormCsr {
        const uint64_t* off;
        const uint32_t* cols;
        const float* vals;
        uint64_t len(uint32_t v) const { return off[v + 1] - off[v]; }
        template <class F>
        bool row(uint32_t v, uint32_t n, F&& f) const {
            for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
                if (cols[i] >= n) return false;
                f(cols[i], vals[i]);
            }
            return true;
        }
    };
    // ... or normalised on the fly from the graph (normalize_adjacency<float>,
    // graph.cpp:68-98: self loop at its sorted position, float(1/sqrt(dv*du)) with
    // dv = deg + 1 in double), so no N-sized host copy of it exists.
    struct RawGraph {
        const uint64_t* off;
        const uint32_t* nbr;
        bool loops;
        uint64_t len(uint32_t v) const { return off[v + 1] - off[v] + (loops ? 1 : 0); }
        template <class F>
        bool row(uint32_t v, uint32_t n, F&& f) const {
            const double extra = loops ? 1.0 : 0.0;
            const double dv = double(off[v + 1] - off[v]) + extra;
            bool pending = loops;
            for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
                const uint32_t u = nbr[i];
                if (u >= n || u == v) return false;
                if (pending && u > v) {
                    f(v, float(1.0 / std::sqrt(dv * dv)));
                    pending = false;
                }
                f(u, float(1.0 / std::sqrt(dv * (double(off[u + 1] - off[u]) + extra))));
            }
            if (pending) f(v, float(1.0 / std::sqrt(dv * dv)));
            return true;
        }
    };

    void upload_graph(const uint64_t* off, const uint32_t* cols, const float* vals, uint64_t nz,
                      const uint32_t* chunk_of) {
        GP_CUDA(cudaSetDevice(device));
        if (!off || !cols || !vals || !chunk_of) throw Error(GP_EINVAL, "null graph array");
        if (off[0] != 0 || off[n] != nz) throw Error(GP_EINVAL, "CSR offsets inconsistent with nnz");
        upload_graph_src(NormCsr{off, cols, vals}, nz, chunk_of);
    }
    void upload_graph_raw(const uint64_t* off, const uint32_t* nbr, uint64_t m2, bool loops, const uint32_t* chunk_of) {
        GP_CUDA(cudaSetDevice(device));
        if (!off || !nbr || !chunk_of) throw Error(GP_EINVAL, "null graph array");
        if (off[0] != 0 || off[n] != m2) throw Error(GP_EINVAL, "graph offsets inconsistent with the neighbour count");
        for (uint32_t v = 0; v < n; ++v)
            if (off[v + 1] < off[v]) throw Error(GP_EINVAL, "graph offsets not monotone");
        upload_graph_src(RawGraph{off, nbr, loops}, m2 + (loops ? n : 0), chunk_of);
    }

    // Raw neighbour lists -> normalised, renumbered, packed CSR on the device (k_build_edges):
    // the host only ships the raw lists (4 bytes per entry instead of 8, no per-entry host
    // arithmetic); the renumbering and row pointers come from the host builder. Sets edges and
    // hg->blk_nnz; throws like the host builder on a bad neighbour.
    void build_edges_device(const RawGraph& src, HostGraph& h, const uint32_t* chunk_of, unsigned nth) {
        const uint64_t m2 = src.off[n];
        auto t_prev = std::chrono::steady_clock::now();
        auto phase = [&](const char* what) {
            if (!host_timing) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[gp graph] %-12s %.1f ms\n", what,
                         std::chrono::duration<double, std::milli>(now - t_prev).count());
            t_prev = now;
        };
        auto tmp = [&](size_t bytes) {
            void* p = nullptr;
            GP_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
            return p;
        };
        struct Free {
            std::vector<void*> v;
            ~Free() {
                for (void* p : v) cudaFree(p);
            }
        } fr;
        auto* d_off = static_cast<uint64_t*>(tmp((size_t(n) + 1) * 8));
        auto* d_nbr = static_cast<uint32_t*>(tmp(m2 * 4));
        auto* d_inv = static_cast<uint32_t*>(tmp(size_t(n) * 4));
        auto* d_perm = static_cast<uint32_t*>(tmp(size_t(n) * 4));
        auto* d_chunk = static_cast<uint32_t*>(tmp(size_t(n) * 4));
        auto* d_rp = static_cast<uint64_t*>(tmp((size_t(n) + 1) * 8));
        auto* d_blk = static_cast<unsigned long long*>(tmp(size_t(K) * K * 8));
        auto* d_bad = static_cast<uint32_t*>(tmp(4));
        fr.v = {d_off, d_nbr, d_inv, d_perm, d_chunk, d_rp, d_blk, d_bad};
        phase("alloc");
        h2d_mt(d_nbr, src.nbr, m2 * 4, nth);
        phase("h2d nbr");
        GP_CUDA(cudaMemcpy(d_off, src.off, (size_t(n) + 1) * 8, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(d_inv, inv.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(d_perm, perm.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(d_chunk, chunk_of, size_t(n) * 4, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(d_rp, h.rp.data(), (size_t(n) + 1) * 8, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemsetAsync(d_blk, 0, size_t(K) * K * 8, cs));
        GP_CUDA(cudaMemsetAsync(d_bad, 0, 4, cs));
        settle_uploads();  // the small copies above went through the legacy stream
        BuildEdgesParams p{d_off, d_nbr, d_inv, d_perm, d_chunk, d_rp, edges, d_blk, d_bad, n, K, src.loops ? 1u : 0u};
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((n + kWarpsPerBlock - 1) / kWarpsPerBlock,
                                                                    uint32_t(num_sms) * 8));
        k_build_edges<<<grid, kBlock, size_t(K) * K * 4, cs>>>(p);
        GP_CUDA(cudaGetLastError());
        uint32_t bad = 0;
        std::vector<uint64_t> blk(size_t(K) * K);
        GP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, cs));
        GP_CUDA(cudaMemcpyAsync(blk.data(), d_blk, blk.size() * 8, cudaMemcpyDeviceToHost, cs));
        GP_CUDA(cudaStreamSynchronize(cs));
        phase("build");
        if (bad) throw Error(GP_EINVAL, "CSR column out of range (or a self loop in the graph)");
        h.blk_nnz = std::move(blk);
    }

    // h2d with the staging copies split over nth threads (large raw arrays)
    void h2d_mt(void* dst, const void* src, size_t bytes, unsigned nth) {
        if (bytes < (size_t(4) << 20) || nth < 2) return h2d(dst, src, bytes);
        StagingLease lease;
        char* const* h2d_stage = lease.buf;
        for (int i = 0; i < 2; ++i)
            if (!h2d_done[i]) GP_CUDA(cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming));
        const char* s8 = static_cast<const char*>(src);
        char* d8 = static_cast<char*>(dst);
        bool used[2] = {false, false};
        for (size_t off = 0, j = 0; off < bytes; off += kStageChunk, ++j) {
            const int b = int(j & 1);
            const size_t len = std::min(kStageChunk, bytes - off);
            if (used[b]) GP_CUDA(cudaEventSynchronize(h2d_done[b]));
            const size_t part = (len / nth + 63) & ~size_t(63);
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < nth; ++t) {
                const size_t a = std::min(len, t * part), z = std::min(len, a + part);
                if (a < z) pool.emplace_back([=]() { std::memcpy(h2d_stage[b] + a, s8 + off + a, z - a); });
            }
            for (auto& th : pool) th.join();
            GP_CUDA(cudaMemcpyAsync(d8 + off, h2d_stage[b], len, cudaMemcpyHostToDevice, cs));
            GP_CUDA(cudaEventRecord(h2d_done[b], cs));
            used[b] = true;
        }
        GP_CUDA(cudaStreamSynchronize(cs));
    }

    template <class Src>
    void upload_graph_src(const Src& src, uint64_t nz, const uint32_t* chunk_of) {
        auto t_prev = std::chrono::steady_clock::now();
        auto phase = [&](const char* what) {
            if (!host_timing) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[gp upload] %-12s %.1f ms\n", what,
                         std::chrono::duration<double, std::milli>(now - t_prev).count());
            t_prev = now;
        };
        if (G > 1 && part_host.size() != n) throw Error(GP_EINVAL, "hybrid: upload the partition first");
        auto partof = [&](uint32_t v) -> uint32_t { return G > 1 ? part_host[v] : 0u; };
        auto h = std::make_shared<HostGraph>();
        const uint32_t KB = K + 1;
        std::vector<uint32_t> count(size_t(G) * KB, 0);
        for (uint32_t v = 0; v < n; ++v) {
            if (chunk_of[v] >= K) throw Error(GP_EINVAL, "chunk id out of range");
            ++count[size_t(partof(v)) * KB + chunk_of[v]];
        }
        h->bstart.assign(size_t(G) * KB, 0);
        uint32_t at = 0;
        for (uint32_t r = 0; r < G; ++r)
            for (uint32_t k = 0; k <= K; ++k) {
                h->bstart[size_t(r) * KB + k] = at;
                if (k < K) at += count[size_t(r) * KB + k];
            }
        perm.assign(n, 0);
        inv.assign(n, 0);
        std::vector<uint32_t> cur(size_t(G) * KB);
        for (uint32_t r = 0; r < G; ++r)
            for (uint32_t k = 0; k < K; ++k) cur[size_t(r) * KB + k] = h->bstart[size_t(r) * KB + k];
        for (uint32_t v = 0; v < n; ++v) inv[cur[size_t(partof(v)) * KB + chunk_of[v]]++] = v;
        // Inside each (rank, chunk) block rows go by descending degree (ties by id):
        // the two rows of a warp then have near-equal lengths (no padded slots on
        // the lighter half) and the dynamic row scheduler hands out the longest
        // rows first. Row contents are untouched, so results stay bit-exact;
        // GP_ROW_ORDER=id keeps plain id order.
        const char* ro = std::getenv("GP_ROW_ORDER");
        if (!(ro && std::string(ro) == "id")) {
            for (size_t b = 0; b + 1 < h->bstart.size(); ++b) {
                if ((b + 1) % KB == 0) continue;  // last entry of a rank's row of starts
                const uint32_t b0 = h->bstart[b], b1 = h->bstart[b + 1];
                std::stable_sort(inv.begin() + b0, inv.begin() + b1,
                                 [&](uint32_t a, uint32_t c) { return src.len(a) > src.len(c); });
            }
        }
        for (uint32_t r = 0; r < n; ++r) perm[inv[r]] = r;
        h->rp.assign(size_t(n) + 1, 0);
        h->part.assign(n, 0);
        h->chunk.assign(n, 0);
        for (uint32_t r = 0; r < n; ++r) {
            const uint32_t v = inv[r];
            if (std::is_same<Src, NormCsr>::value && src.len(v) > nz) throw Error(GP_EINVAL, "CSR offsets not monotone");
            h->rp[r + 1] = h->rp[r] + src.len(v);
            h->part[r] = partof(v);
            h->chunk[r] = chunk_of[v];
        }
        // Packed entries are built straight into the pinned staging chunks and DMA'd
        // chunk by chunk (no N-sized host copy); host columns only for hybrid halos.
        if (G > 1) h->col.resize(nz);
        const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::atomic<bool> bad{false};
        edges = dalloc<uint2>(std::max<uint64_t>(nz, 1), false);
        // CSR entries per (row block (rank, chunk), column chunk): the entries a done-filtered
        // backward gather actually fetches, for the byte / flop accounting
        std::vector<std::atomic<uint64_t>> blk_nnz(size_t(G) * K * K);
        phase("renumber");
        bool built = false;
        if constexpr (std::is_same<Src, RawGraph>::value)
            if (G == 1 && (graph_build == 1 || (graph_build == 0 && nz * 8 >= (size_t(64) << 20)))) {
                build_edges_device(src, *h, chunk_of, nth);
                built = true;
            }
        if (!built) stage_rows_h2d(edges, h->rp, nth, [&](uint32_t r, uint2* out) {
            const uint32_t v = inv[r];
            uint64_t w = 0;
            uint32_t per_chunk[kMaxChunks] = {};
            const bool ok = src.row(v, n, [&](uint32_t u, float val) {
                uint32_t bits;
                std::memcpy(&bits, &val, 4);
                out[w] = make_uint2(perm[u] | (chunk_of[u] << kColBits), bits);
                if (G > 1) h->col[h->rp[r] + w] = perm[u];
                ++per_chunk[chunk_of[u] < K ? chunk_of[u] : 0];
                ++w;
            });
            const size_t blk = (size_t(h->part[r]) * K + h->chunk[r]) * K;
            for (uint32_t c = 0; c < K; ++c)
                if (per_chunk[c]) blk_nnz[blk + c].fetch_add(per_chunk[c], std::memory_order_relaxed);
            if (!ok) bad = true;
        });
        if (!built) {
            h->blk_nnz.resize(blk_nnz.size());
            for (size_t i = 0; i < blk_nnz.size(); ++i) h->blk_nnz[i] = blk_nnz[i].load();
        }
        if (bad) throw Error(GP_EINVAL, "CSR column out of range (or a self loop in the graph)");
        phase("entries");
        if (has_sage) {
            // mean / mean_t (graph.cpp:100-112, nn.hpp:85-98): the normalised rows
            // without the self loop, same renumbering and chunk bits
            std::vector<uint32_t> deg(n, 0);
            for (uint32_t v = 0; v < n; ++v) src.row(v, n, [&](uint32_t u, float) { deg[v] += u != v; });
            std::vector<uint64_t> rpm(size_t(n) + 1, 0);
            for (uint32_t r = 0; r < n; ++r) rpm[r + 1] = rpm[r] + deg[inv[r]];
            std::vector<uint2> em(std::max<uint64_t>(rpm[n], 1)), emt(std::max<uint64_t>(rpm[n], 1));
            for (uint32_t r = 0; r < n; ++r) {
                const uint32_t v = inv[r];
                const float wv = deg[v] ? float(1.0 / double(deg[v])) : 0.f;
                uint64_t w = rpm[r];
                src.row(v, n, [&](uint32_t u, float) {
                    if (u == v) return;
                    const float wu = deg[u] ? float(1.0 / double(deg[u])) : 0.f;
                    uint32_t bv, bu;
                    std::memcpy(&bv, &wv, 4);
                    std::memcpy(&bu, &wu, 4);
                    const uint32_t col = perm[u] | (chunk_of[u] << kColBits);
                    em[w] = make_uint2(col, bv);
                    emt[w] = make_uint2(col, bu);
                    ++w;
                });
            }
            rowptr_m = dalloc<uint64_t>(size_t(n) + 1, false);
            edges_m = dalloc<uint2>(em.size(), false);
            edges_mt = dalloc<uint2>(emt.size(), false);
            GP_CUDA(cudaMemcpy(rowptr_m, rpm.data(), rpm.size() * 8, cudaMemcpyHostToDevice));
            h2d(edges_m, em.data(), em.size() * 8);
            h2d(edges_mt, emt.data(), emt.size() * 8);
        }
        nnz = nz;
        rowptr = dalloc<uint64_t>(size_t(n) + 1, false);
        orig = dalloc<uint32_t>(n, false);
        GP_CUDA(cudaMemcpy(rowptr, h->rp.data(), h->rp.size() * 8, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(orig, inv.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
        hg = h;
        if (G == 1) hg->col.clear();  // only hybrid needs the host columns
        bstart = hg->bstart;
        build_halo();
        build_id_rows();
        phase("rows");
        ensure_own_buffers();
        alloc_bwd_csr();
        settle_uploads();
        phase("buffers");
        graph_ready = true;
    }

    // Own rows in ascending original vertex id: the order param_grads_for_rows and the
    // loss sum visit rows in (nn.hpp:269-293, engines_impl.hpp:725-734, :873-876). Reducing
    // in this order, with split boundaries fixed by the row count alone, makes parameter
    // gradients and the loss independent of the chunk plan (a synchronous pipeline then
    // equals the sequential trainer bit for bit, test_engines.cpp:115-126).
    // A stale-mode backward gather (PREV_AGG) filters by done chunks: layers i >= 1 that
    // aggregate (not SageConv: its filtered gather runs over the mean CSR), and layer 0 on
    // a non-first stage (the dh_in gather)
    bool needs_bwd_csr() const {
        if (!bwd_csr || sync || hist || K < 2) return false;
        for (uint32_t i = 0; i < len; ++i)
            if (L[i].agg && !L[i].sage && (i > 0 || !first)) return true;
        return false;
    }
    uint64_t bwd_csr_cap = 0;
    void alloc_bwd_csr() {
        if (!needs_bwd_csr()) return;
        const uint64_t own_nnz = hg->rp[own_end()] - hg->rp[own_begin()];
        if (rowptr_f && own_nnz <= bwd_csr_cap) return;
        rowptr_f = dalloc<uint64_t>(size_t(n) + 1);  // rowptr_f[own_begin] stays 0
        edges_f = dalloc<uint2>(std::max<uint64_t>(own_nnz, 1), false);
        bwd_csr_cap = own_nnz;
        const uint32_t items = own_end() - own_begin() + 1;
        scan_tiles = (items + kScanTile - 1) / kScanTile;
        scan_tmp = dalloc<unsigned long long>(scan_tiles, false);
    }

    // The epoch's done-filtered backward CSR: chunk order[kk] runs its backward with
    // done = {order[kk], ..., order[K-1]} (engines_impl.hpp:829-866)
    void build_bwd_csr(const std::vector<uint32_t>& ord) {
        bwd_csr_ready = false;
        if (!rowptr_f || !needs_bwd_csr()) return;
        DoneCsrParams p{};
        p.rowptr = rowptr;
        p.edges = edges;
        p.rowptr_f = rowptr_f;
        p.edges_f = edges_f;
        for (uint32_t k = 0; k <= K; ++k) p.rb[k] = row_begin(k);
        uint64_t done = 0;
        for (uint32_t kk = K; kk-- > 0;) p.mask[ord[kk]] = done |= 1ull << ord[kk];
        const dim3 grid(std::max<uint32_t>(1, (uint32_t(num_sms) * 8 + K - 1) / K), K);
        const uint32_t items = own_end() - own_begin() + 1;
        const double eb = double(hg->rp[own_end()] - hg->rp[own_begin()]) * 8.0;
        launch(GP_K_BWD_AGG, eb + double(items) * 16.0, 0, 0, [&]() {
            k_done_csr<true><<<grid, kBlock, 0, cs>>>(p);
            auto* v = reinterpret_cast<unsigned long long*>(rowptr_f + own_begin());
            k_scan_tiles<<<scan_tiles, kScanThreads, 0, cs>>>(v, items, scan_tmp);
            k_scan_totals<<<1, kScanThreads, 0, cs>>>(scan_tmp, scan_tiles);
            k_scan_add<<<scan_tiles, kScanThreads, 0, cs>>>(v, items, scan_tmp);
            k_done_csr<false><<<grid, kBlock, 0, cs>>>(p);
        });
        bwd_csr_ready = true;
    }

    void build_id_rows() {
        std::vector<uint32_t> rows;
        rows.reserve(own_end() - own_begin());
        for (uint32_t v = 0; v < n; ++v) {
            const uint32_t r = perm[v];
            if (r >= own_begin() && r < own_end()) rows.push_back(r);
        }
        if (!id_rows) id_rows = dalloc<uint32_t>(std::max<size_t>(rows.size(), 1), false);
        GP_CUDA(cudaMemcpy(id_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    }

    // Halo lists (chunk_push_sets, engines_impl.hpp:488-499): peer r2 pushes, in
    // chunk k, its rows v (part r2, chunk k) that have a neighbour in my partition;
    // I push mine likewise. Derived from the (symmetric) normalised adjacency.
    void build_halo() {
        pull_off.assign(size_t(G) * (K + 1), 0);
        push_cnt.assign(size_t(K) * G, 0);
        if (G == 1) return;
        const HostGraph& h = *hg;
        std::vector<std::vector<uint32_t>> lists(size_t(G) * K);
        std::vector<uint32_t> seen(G, 0xffffffffu);
        for (uint32_t v = 0; v < n; ++v) {
            const uint32_t pv = h.part[v], kv = h.chunk[v];
            for (uint64_t i = h.rp[v]; i < h.rp[v + 1]; ++i) {
                const uint32_t pu = h.part[h.col[i]];
                if (pu == pv || seen[pu] == v) continue;
                seen[pu] = v;  // v is in B_pu (boundary of pu)
                if (pu == grank) lists[size_t(pv) * K + kv].push_back(v);
                if (pv == grank) ++push_cnt[size_t(kv) * G + pu];
            }
        }
        std::vector<uint32_t> flat;
        for (uint32_t r2 = 0; r2 < G; ++r2)
            for (uint32_t k = 0; k < K; ++k) {
                pull_off[size_t(r2) * (K + 1) + k] = uint32_t(flat.size());
                auto& l = lists[size_t(r2) * K + k];
                flat.insert(flat.end(), l.begin(), l.end());
                pull_off[size_t(r2) * (K + 1) + k + 1] = uint32_t(flat.size());
            }
        pull_idx = dalloc<uint32_t>(std::max<size_t>(flat.size(), 1), false);
        if (!flat.empty()) GP_CUDA(cudaMemcpy(pull_idx, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice));
    }

    void share_graph(const Stage& o) {
        if (!o.graph_ready) throw Error(GP_EINVAL, "owner stage has no graph");
        if (o.n != n || o.K != K || o.device != device || o.G != G)
            throw Error(GP_EINVAL, "graph sharing needs the same N, K, G and device");
        rowptr = o.rowptr;
        edges = o.edges;
        if (has_sage && !o.rowptr_m) throw Error(GP_EINVAL, "graph sharing: owner stage has no SageConv adjacency");
        rowptr_m = o.rowptr_m;
        edges_m = o.edges_m;
        edges_mt = o.edges_mt;
        orig = o.orig;
        perm = o.perm;
        inv = o.inv;
        hg = o.hg;
        bstart = o.bstart;
        nnz = o.nnz;
        build_halo();
        build_id_rows();
        ensure_own_buffers();
        alloc_bwd_csr();
        settle_uploads();
        graph_ready = true;
    }

    void upload_features(const float* x, uint32_t f) {
        GP_CUDA(cudaSetDevice(device));
        if (!first) throw Error(GP_EINVAL, "features belong to stage 0");
        if (!graph_ready) throw Error(GP_EINVAL, "upload the graph first");
        if (f != specs[0].in_dim) throw Error(GP_EINVAL, "feature width != layer 0 in_dim");
        F = f;
        sx = pad8(f);
        if (!x0) x0 = dalloc<float>(size_t(n) * sx, false);
        // rows renumbered and padded straight into the pinned staging chunks
        std::vector<uint64_t> rp(size_t(n) + 1);
        for (uint32_t r = 0; r <= n; ++r) rp[r] = uint64_t(r) * sx;
        const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        stage_rows_h2d(x0, rp, nth, [&](uint32_t r, float* out) {
            std::memcpy(out, x + size_t(inv[r]) * f, size_t(f) * 4);
            std::memset(out + f, 0, size_t(sx - f) * 4);
        });
        settle_uploads();
        x_ready = true;
    }

    void upload_labels(const uint32_t* lab, const uint8_t* sp) {
        GP_CUDA(cudaSetDevice(device));
        if (!last) throw Error(GP_EINVAL, "labels belong to the last stage");
        if (!graph_ready) throw Error(GP_EINVAL, "upload the graph first");
        std::vector<uint32_t> hl(n);
        std::vector<uint8_t> hs(n);
        uint64_t ntrain = 0;
        for (uint32_t r = 0; r < n; ++r) {
            hl[r] = lab[inv[r]];
            hs[r] = sp[inv[r]];
            if (hl[r] >= C) throw Error(GP_EINVAL, "label >= num_classes");
            ntrain += hs[r] == 1;
        }
        if (ntrain == 0) throw Error(GP_EINVAL, "train_hybrid: empty train mask");
        inv_train = float(1.0 / double(ntrain));  // engines_impl.hpp:548
        if (!labels) labels = dalloc<uint32_t>(n, false);
        if (!split) split = dalloc<uint8_t>(n, false);
        GP_CUDA(cudaMemcpy(labels, hl.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(split, hs.data(), n, cudaMemcpyHostToDevice));
        settle_uploads();
        labels_ready = true;
    }

    LayerDev& layer(uint32_t l) {
        if (l < lb || l >= le) throw Error(GP_EINVAL, "layer not owned by this stage");
        return L[l - lb];
    }

    void transpose_w(const LayerDev& d) {
        if (d.sage) {
            const uint32_t nw = d.kw * d.dout;
            launch(GP_K_OPTIM, nw * 12.0, 0, 0, [&]() {
                k_sage_weights<<<(nw + 255) / 256, 256, 0, cs>>>(d.W, d.Wg, d.WTg, d.din, d.dout, d.sgap);
            });
            return;
        }
        const uint32_t nw = d.din * d.dout;
        launch(GP_K_OPTIM, nw * 8.0, 0, 0,
               [&]() { k_transpose<<<(nw + 255) / 256, 256, 0, cs>>>(d.W, d.WT, d.din, d.dout); });
        if (d.tc) {  // W (or, GP_TC_MIX=0, W' = beta W + (1 - beta) I for Gcn2Conv) as tf32 hi / lo
            const bool g2 = d.spec.kind == GP_GCN2CONV && !tc_mix_epi;
            const float beta = float(d.spec.beta), omb = 1.f - beta;
            launch(GP_K_OPTIM, nw * 12.0, 0, 0, [&]() {
                k_tc_prep<<<(nw + 255) / 256, 256, 0, cs>>>(d.W, d.din, d.dout, xf_pad8k(d.din), xf_pad16(d.dout), 0,
                                                            g2, beta, omb, d.xf_fwd);
                k_tc_prep<<<(nw + 255) / 256, 256, 0, cs>>>(d.W, d.dout, d.din, xf_pad8k(d.dout), xf_pad16(d.din), 1,
                                                            g2, beta, omb, d.xf_bwd);
            });
        }
    }

    // tcgen05 transform launch over rows [r0, r1): one CTA per SM (>= 116 KB of shared
    // memory, so a second CTA never waits on TMEM columns), persistent over 128-row tiles
    template <bool BWD>
    void tc_xform_go(TcXformParams x) {
        x.a_lbo = x.r1 - x.r0 >= xf_pad_rows ? kXfLboPad : kXfLboDense;
        const uint32_t ntiles = (x.r1 - x.r0 + kXfM - 1) / kXfM;
        const size_t smem = std::max<size_t>(xf_smem_bytes(x.kpad, x.npad), 116 * 1024);
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(ntiles, uint32_t(num_sms)));
        k_tc_xform<BWD><<<grid, kXfThreads, smem, cs>>>(x);
    }
    TcXformParams tc_fwd_params(const LayerDev& d, const FwdParams& p) const {
        TcXformParams x{};
        x.r0 = p.r0;
        x.r1 = p.r1;
        x.A = p.pre;
        x.astride = p.prestride;
        x.kdim = d.din;
        x.kpad = xf_pad8k(d.din);
        x.ndim = d.dout;
        x.npad = xf_pad16(d.dout);
        x.ostride = p.outstride;
        x.Bop = d.xf_fwd;
        x.bias = p.bias;
        x.relu = p.relu;
        x.out = p.out;
        // lean layout, epoch before a snapshot refresh: the epilogue writes h into the snapshot too
        x.out2 = dual_snap && d.hs ? d.hs : nullptr;
        x.gnext = p.gnext;
        x.gnstride = p.gnstride;
        x.next_mask = p.next_mask;
        x.orig = p.orig;
        tc_mix(d, x);
        return x;
    }
    // Gcn2Conv identity mix in the transform epilogue (GP_TC_MIX=1) or folded into the
    // prepared operand (GP_TC_MIX=0, default)
    void tc_mix(const LayerDev& d, TcXformParams& x) const {
        if (d.spec.kind != GP_GCN2CONV || !tc_mix_epi) return;
        x.mix = 1;
        x.mbeta = float(d.spec.beta);
        x.momb = 1.f - x.mbeta;
    }
    TcXformParams tc_bwd_params(const LayerDev& d, const BwdParams& p) const {
        TcXformParams x{};
        x.r0 = p.r0;
        x.r1 = p.r1;
        x.A = p.dz;
        x.astride = p.dzstride;
        x.kdim = d.dout;
        x.kpad = xf_pad8k(d.dout);
        x.ndim = d.din;
        x.npad = xf_pad16(d.din);
        x.ostride = p.bgstride;
        x.Bop = d.xf_bwd;
        x.gcn2 = p.gcn2;
        x.alpha = p.alpha;
        x.oma = p.oma;
        x.dh0 = p.dh0;
        x.dh0stride = p.dh0stride;
        x.bg = p.bg;
        tc_mix(d, x);
        return x;
    }

    // A cudaMemcpy from pageable host memory may return before its DMA has landed, and the
    // engine's streams are non-blocking (not ordered after the legacy stream): every upload
    // entry point waits for its legacy-stream copies before returning, so no kernel can read a
    // buffer whose upload is still in flight.
    void settle_uploads() { GP_CUDA(cudaStreamSynchronize(cudaStreamLegacy)); }

    void set_params(uint32_t l, const float* W, const float* b) {
        GP_CUDA(cudaSetDevice(device));
        auto& d = layer(l);
        if (d.b && !b) throw Error(GP_EINVAL, "layer has a bias");
        GP_CUDA(cudaStreamSynchronize(cs));
        GP_CUDA(cudaMemcpy(d.W, W, size_t(d.kin) * d.dout * 4, cudaMemcpyHostToDevice));
        if (d.b) GP_CUDA(cudaMemcpy(d.b, b, size_t(d.dout) * 4, cudaMemcpyHostToDevice));
        settle_uploads();  // transpose_w reads W on cs
        transpose_w(d);
        GP_CUDA(cudaStreamSynchronize(cs));
    }

    void get_grads(uint32_t l, float* W, float* b) {
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaStreamSynchronize(cs));
        auto& d = layer(l);
        if (W) GP_CUDA(cudaMemcpy(W, d.gW, size_t(d.kin) * d.dout * 4, cudaMemcpyDeviceToHost));
        if (d.gb && b) GP_CUDA(cudaMemcpy(b, d.gb, size_t(d.dout) * 4, cudaMemcpyDeviceToHost));
    }

    // Optimizer state (Optimizer::m_/v_/t_, nn.hpp:431-495) for checkpoint/resume.
    void get_opt_state(uint32_t l, float* mW, float* vW, float* mb, float* vb, uint64_t* t) {
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaStreamSynchronize(cs));
        auto& d = layer(l);
        const size_t wn = size_t(d.kin) * d.dout * 4;
        if (mW) GP_CUDA(cudaMemcpy(mW, d.mW, wn, cudaMemcpyDeviceToHost));
        if (vW) GP_CUDA(cudaMemcpy(vW, d.vW, wn, cudaMemcpyDeviceToHost));
        if (d.mb && mb) GP_CUDA(cudaMemcpy(mb, d.mb, size_t(d.dout) * 4, cudaMemcpyDeviceToHost));
        if (d.vb && vb) GP_CUDA(cudaMemcpy(vb, d.vb, size_t(d.dout) * 4, cudaMemcpyDeviceToHost));
        if (t) *t = step;
    }
    void set_opt_state(uint32_t l, const float* mW, const float* vW, const float* mb, const float* vb, uint64_t t) {
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaStreamSynchronize(cs));
        auto& d = layer(l);
        const size_t wn = size_t(d.kin) * d.dout * 4;
        if (!mW || !vW) throw Error(GP_EINVAL, "optimizer state: null weight moments");
        GP_CUDA(cudaMemcpy(d.mW, mW, wn, cudaMemcpyHostToDevice));
        GP_CUDA(cudaMemcpy(d.vW, vW, wn, cudaMemcpyHostToDevice));
        if (d.mb) {
            if (!mb || !vb) throw Error(GP_EINVAL, "optimizer state: layer has a bias");
            GP_CUDA(cudaMemcpy(d.mb, mb, size_t(d.dout) * 4, cudaMemcpyHostToDevice));
            GP_CUDA(cudaMemcpy(d.vb, vb, size_t(d.dout) * 4, cudaMemcpyHostToDevice));
        }
        settle_uploads();
        step = t;
    }

    void get_params(uint32_t l, float* W, float* b) {
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaStreamSynchronize(cs));
        auto& d = layer(l);
        if (W) GP_CUDA(cudaMemcpy(W, d.W, size_t(d.kin) * d.dout * 4, cudaMemcpyDeviceToHost));
        if (d.b && b) GP_CUDA(cudaMemcpy(b, d.b, size_t(d.dout) * 4, cudaMemcpyDeviceToHost));
    }

    // ---- launch helpers -------------------------------------------------------
    cudaEvent_t take_event() {
        if (!ev_free.empty()) {
            auto e = ev_free.back();
            ev_free.pop_back();
            return e;
        }
        cudaEvent_t e;
        GP_CUDA(cudaEventCreate(&e));
        return e;
    }

    template <typename F>
    void launch(int cls, double bytes, double flops, double gather, F&& fn) {
        ++launches;
        if (!profiling && cls != live_cls && live_cls != GP_K_NUM) {
            fn();
            GP_CUDA(cudaGetLastError());
            return;
        }
        Timed t{cls, take_event(), take_event(), bytes, flops, gather};
        GP_CUDA(cudaEventRecord(t.a, cs));
        fn();
        GP_CUDA(cudaGetLastError());
        GP_CUDA(cudaEventRecord(t.b, cs));
        timed.push_back(t);
    }

    // Persistent grid: exactly the resident capacity (occupancy x SMs), capped by
    // the number of 8-row blocks, so there is no partial second wave.
    uint32_t row_grid(uint32_t rows, const void* fn, size_t smem, uint32_t rows_per_block = kWarpsPerBlock) {
        auto key = std::make_pair(fn, smem);
        auto it = occ_cache.find(key);
        int occ = 0;
        if (it == occ_cache.end()) {
            GP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, smem));
            occ_cache[key] = occ = std::max(occ, 1);
        } else {
            occ = it->second;
        }
        const uint64_t want = (uint64_t(rows) + rows_per_block - 1) / rows_per_block;
        const uint64_t cap = uint64_t(num_sms) * occ;
        return uint32_t(std::max<uint64_t>(1, std::min(want, cap)));
    }

    DropKey drop_key(uint32_t t, uint32_t l, uint32_t cols) const {
        DropKey k;
        if (cfg.dropout <= 0.0) return k;  // DropMask::off (nn.hpp:115)
        const double keep = 1.0 - cfg.dropout;
        k.enabled = 1;
        k.cols = cols;
        k.scale = float(1.0 / keep);
        k.k2 = mix64(mix64(cfg.seed, t, l));
        k.thr = uint64_t(std::ceil(std::ldexp(keep, 53)));
        return k;
    }

    // Source rows of layer i's input for stale reads: the snapshot.
    const float* snap_src(uint32_t i) const {
        if (i == 0) return first ? x0 : in_snap;
        return L[i - 1].hs;
    }
    uint32_t src_stride(uint32_t i) const { return i == 0 ? (first ? sx : sin0) : L[i - 1].sout; }
    const float* cur_src(uint32_t i) const {
        if (i == 0) return first ? x0 : in_cur;
        return L[i - 1].h;
    }

    // G (rows of done chunks) or Gs (snapshot rows, rebuilt once per epoch)
    void remask(uint32_t i, const float* src, uint32_t r0, uint32_t r1, const DropKey& key, bool snapshot = false) {
        auto& d = L[i];
        RemaskParams p{r0, r1, d.din, src, src_stride(i), snapshot ? d.Gs : d.G, d.sin, orig, key};
        const uint32_t rows = r1 - r0;
        launch(GP_K_REMASK, double(rows) * d.din * 8.0, 0, 0,
               [&]() { k_remask<<<row_grid(rows, (const void*)k_remask, 0), kBlock, 0, cs>>>(p); });
    }

    void forward_layer(uint32_t i, uint32_t r0, uint32_t r1, uint32_t t, uint64_t done) {
        auto& d = L[i];
        const uint32_t rows = r1 - r0;
        if (rows == 0) return;
        const float* h0src = needs_h0 ? (first ? L[0].h : h0) : nullptr;
        const uint32_t h0stride = pad8(H);
        float* gnext = nullptr;
        uint32_t gnstride = 0;
        DropKey nk;
        if (i + 1 < len && L[i + 1].agg) {
            gnext = L[i + 1].G;
            gnstride = L[i + 1].sin;
            nk = drop_key(t, d.l + 1, L[i + 1].din);
        }
        const float alpha = float(d.spec.alpha), beta = float(d.spec.beta);
        auto gather_done = [&]() {
            if (on_gather_done && d.agg) on_gather_done(i);
        };
        auto write_wait = [&]() {
            if (before_g_write && gnext) before_g_write(i + 1);
        };
        if (d.din <= kMaxWidth) {
            FwdParams p{};
            p.r0 = r0;
            p.r1 = r1;
            p.ticket = take_ticket();
            p.rowptr = rowptr;
            p.edges = edges;
            p.gsrc = d.G;
            // one table (merged, synchronous, or stage 0's features): plain gather, no per-entry choice
            p.gsnap = d.agg && d.Gs != d.G ? d.Gs : nullptr;
            p.done = done;
            p.gstride = d.sin;
            p.zrow = n;
            p.xsrc = cur_src(i);
            p.xstride = src_stride(i);
            p.in_mask = drop_key(t, d.l, d.din);
            p.orig = orig;
            p.h0 = h0src;
            p.h0stride = h0stride;
            p.alpha = alpha;
            p.oma = 1.f - alpha;  // (T{1} - a) in float, nn.hpp:184-187
            p.beta = beta;
            p.omb = 1.f - beta;
            p.W = d.W;
            p.bias = d.b;
            p.din = d.din;
            p.dout = d.dout;
            p.relu = d.spec.relu;
            p.pre = d.pre;
            p.prestride = d.sin;
            p.out = d.h;
            p.outstride = d.sout;
            p.gnext = gnext;
            p.gnstride = gnstride;
            p.next_mask = nk;
            p.rowptr_m = rowptr_m;
            p.edges_m = edges_m;
            p.sgap = d.sgap;
            p.prestride = d.skw;
            const size_t smem = row_smem_bytes(d.din, d.dout, 2);
            const double e = d.agg ? double(rowptr_nnz(r0, r1)) : 0.0;
            const double bytes = (d.agg ? e * 8.0 + double(rows + 1) * 8.0 + double(n) * d.din * 4.0
                                        : double(rows) * d.din * 4.0) +
                                 double(rows) * (d.din + d.dout) * 4.0 +
                                 (d.spec.kind == GP_GCN2CONV ? double(rows) * d.din * 4.0 : 0.0) +
                                 (gnext ? double(rows) * d.dout * 4.0 : 0.0);
            const double flops = 2.0 * e * d.din + 2.0 * double(rows) * d.din * d.dout;
            const double gather = e * double(d.sin) * 4.0;
            const int cls = d.agg ? GP_K_FWD_AGG : GP_K_FWD_DENSE;
            if (d.sage) {
                // pre = [own row | mean of neighbours] (gapped), then b + pre.W + ReLU + epilogue
                const double eb = e * 8.0 + double(rows + 1) * 8.0 + double(n) * d.din * 4.0 + double(rows) * d.kw * 4.0;
                const double db = double(rows) * (d.kw + d.dout + (gnext ? d.dout : 0)) * 4.0 +
                                  double(d.kw) * d.dout * 4.0;
                launch(GP_K_FWD_AGG, eb, 2.0 * e * d.din, gather, [&]() { fwd_nb<FWD_SAGE, true>(rows, kEdgeSlotBytes, p); });
                gather_done();
                write_wait();
                FwdParams q = p;
                q.W = d.Wg;
                q.din = d.kw;
                launch(GP_K_FWD_DENSE, db, 2.0 * double(rows) * d.kin * d.dout, 0,
                       [&]() { fwd_dense_go<false>(rows, q); });
                return;
            }
            if (!d.agg && d.tc && split_rows) {
                // Dense on tcgen05: pre = drop(x) (the reference's dropped input row), then b + pre.W'
                RemaskParams rp{r0, r1, d.din, cur_src(i), src_stride(i), d.pre, d.skw, orig, drop_key(t, d.l, d.din)};
                launch(GP_K_FWD_DENSE, double(rows) * d.din * 8.0, 0, 0,
                       [&]() { k_remask<<<row_grid(rows, (const void*)k_remask, 0), kBlock, 0, cs>>>(rp); });
                write_wait();
                if (dual_snap && d.hs) dual_done[i] = 1;
                const double db = double(rows) * (d.din + d.dout + (gnext ? d.dout : 0)) * 4.0 + double(d.din) * d.dout * 4.0;
                launch(GP_K_FWD_DENSE, db, 2.0 * double(rows) * d.din * d.dout, 0,
                       [&]() { tc_xform_go<false>(tc_fwd_params(d, p)); });
                return;
            }
            if (d.agg && split_rows) {
                // gather + initial-residual mix -> pre, then b + pre.W + epilogue
                const bool g2 = d.spec.kind == GP_GCN2CONV;
                const double eb = e * 8.0 + double(rows + 1) * 8.0 + double(n) * d.din * 4.0 +
                                  double(rows) * d.din * 4.0 * (g2 ? 2.0 : 1.0);
                const double db = double(rows) * (d.din + d.dout + (gnext ? d.dout : 0)) * 4.0 +
                                  double(d.din) * d.dout * 4.0;
                launch(GP_K_FWD_AGG, eb, 2.0 * e * d.din, gather, [&]() {
                    if (g2) fwd_nb<FWD_GCN2, true>(rows, kEdgeSlotBytes, p);
                    else fwd_nb<FWD_GCN, true>(rows, kEdgeSlotBytes, p);
                });
                gather_done();
                write_wait();
                if (d.tc && dual_snap && d.hs) dual_done[i] = 1;
                launch(GP_K_FWD_DENSE, db, 2.0 * double(rows) * d.din * d.dout, 0, [&]() {
                    if (d.tc) tc_xform_go<false>(tc_fwd_params(d, p));
                    else if (g2) fwd_dense_go<true>(rows, p);
                    else fwd_dense_go<false>(rows, p);
                });
                return;
            }
            write_wait();
            if (d.spec.kind == GP_DENSE)
                launch(cls, bytes, flops, 0, [&]() { fwd_nb<FWD_DENSE>(rows, smem, p); });
            else if (d.spec.kind == GP_GCNCONV)
                launch(cls, bytes, flops, gather, [&]() { fwd_nb<FWD_GCN>(rows, smem, p); });
            else
                launch(cls, bytes, flops, gather, [&]() { fwd_nb<FWD_GCN2>(rows, smem, p); });
            gather_done();
            return;
        }
        // wide input (layer 0 with F > 128): pre first, then the tiled transform. SageConv:
        // mean aggregate into the gapped second half, the dropped own row into the first
        if (d.spec.kind == GP_GCN2CONV) throw Error(GP_EINVAL, "Gcn2Conv wider than 128");
        if (d.agg) {
            SpmmParams sp{r0, r1, d.din, n, d.sage ? rowptr_m : rowptr, d.sage ? edges_m : edges, d.G, d.sin,
                          d.pre + d.sgap, d.skw};
            const double e = double(rowptr_nnz(r0, r1));
            launch(GP_K_FWD_AGG, e * 8.0 + double(n) * d.din * 4.0 + double(rows) * d.din * 4.0,
                   2.0 * e * d.din, e * d.sin * 4.0,
                   [&]() { k_spmm_pre<<<row_grid(rows, (const void*)k_spmm_pre, 0), kBlock, 0, cs>>>(sp); });
            gather_done();
            if (d.sage) {
                RemaskParams rp{r0, r1, d.din, cur_src(i), src_stride(i), d.pre, d.skw, orig, drop_key(t, d.l, d.din)};
                launch(GP_K_FWD_DENSE, double(rows) * d.din * 8.0, 0, 0,
                       [&]() { k_remask<<<row_grid(rows, (const void*)k_remask, 0), kBlock, 0, cs>>>(rp); });
            }
        } else {
            RemaskParams rp{r0, r1, d.din, cur_src(i), src_stride(i), d.pre, d.sin, orig,
                            drop_key(t, d.l, d.din)};
            launch(GP_K_FWD_DENSE, double(rows) * d.din * 8.0, 0, 0,
                   [&]() { k_remask<<<row_grid(rows, (const void*)k_remask, 0), kBlock, 0, cs>>>(rp); });
        }
        GemmParams g{};
        g.r0 = r0;
        g.r1 = r1;
        g.A = d.pre;
        g.astride = d.skw;
        g.W = d.sage ? d.Wg : d.W;
        g.bias = d.b;
        g.din = d.kw;
        g.dout = d.dout;
        g.relu = d.spec.relu;
        g.out = d.h;
        g.outstride = d.sout;
        g.gnext = gnext;
        g.gnstride = gnstride;
        g.next_mask = nk;
        g.orig = orig;
        write_wait();
        launch(GP_K_FWD_DENSE,
               double(rows) * (d.din + d.dout + (gnext ? d.dout : 0)) * 4.0 + double(d.din) * d.dout * 4.0,
               2.0 * double(rows) * d.din * d.dout, 0,
               [&]() { k_dense_gemm<<<(rows + 63) / 64, kBlock, 0, cs>>>(g); });
    }

    // CSR entries of rows [r0, r1) whose column chunk is in `done` (what a done-filtered
    // gather fetches); the whole count when [r0, r1) is not one (rank, chunk) block
    double done_nnz(uint32_t r0, uint32_t r1, uint64_t done) {
        if (done == all_chunks() || !hg || hg->blk_nnz.empty()) return double(rowptr_nnz(r0, r1));
        for (uint32_t k = 0; k < K; ++k)
            if (row_begin(k) == r0 && row_end(k) == r1) {
                const size_t blk = (size_t(grank) * K + k) * K;
                uint64_t e = 0;
                for (uint32_t c = 0; c < K; ++c)
                    if ((done >> c) & 1ull) e += hg->blk_nnz[blk + c];
                return double(e);
            }
        return double(rowptr_nnz(r0, r1));
    }
    std::vector<uint64_t> h_rowptr;  // host copy for byte accounting
    uint64_t rowptr_nnz(uint32_t r0, uint32_t r1) {
        if (h_rowptr.empty()) {
            h_rowptr.resize(size_t(n) + 1);
            GP_CUDA(cudaMemcpy(h_rowptr.data(), rowptr, h_rowptr.size() * 8, cudaMemcpyDeviceToHost));
        }
        return h_rowptr[r1] - h_rowptr[r0];
    }

    // backward kernel for local layer i over rows [r0, r1)
    void backward_layer(uint32_t i, uint32_t r0, uint32_t r1, uint32_t t, uint64_t done) {
        auto& d = L[i];
        const uint32_t rows = r1 - r0;
        if (rows == 0) return;
        BwdParams p{};
        p.r0 = r0;
        p.r1 = r1;
        p.ticket = take_ticket();
        p.rowptr = rowptr;
        p.edges = edges;
        p.done = done;
        p.orig = orig;
        p.dh_width = d.dout;
        int prev = PREV_TOP;
        double e = 0;
        if (i + 1 == len) {
            p.dtop = dtop;
            p.dtopstride = d.sout;
        } else {
            auto& nx = L[i + 1];
            p.bgn = nx.bg;
            p.bgn_snap = nx.bgs;
            p.bgnstride = nx.skw;
            p.zrow = n;
            p.prev_mask = drop_key(t, nx.l, nx.din);
            if (nx.sage) {
                prev = hist ? PREV_SAGE_HIST : PREV_SAGE;
                p.rowptr_m = rowptr_m;
                p.edges_m = edges_mt;
                p.sgap = nx.sgap;
                e = double(rowptr_nnz(r0, r1));
            } else if (nx.agg) {
                prev = hist ? PREV_AGG_HIST : (done == all_chunks() ? PREV_AGG_ALL : PREV_AGG);
                e = hist ? double(rowptr_nnz(r0, r1)) : done_nnz(r0, r1, done);  // entries gathered
                if (prev == PREV_AGG && bwd_csr_ready) {  // the same entries, pre-filtered
                    p.rowptr = rowptr_f;
                    p.edges = edges_f;
                    prev = PREV_AGG_ALL;
                }
            } else {
                prev = PREV_OWN;
            }
        }
        p.dh0stride = pad8(H);
        if (d.l == 0 && needs_h0) p.dh0_add = dh0;
        p.h = d.h;
        p.hstride = d.sout;
        p.relu = d.spec.relu;
        p.dz = d.dz;
        p.dzstride = d.sout;
        p.W = d.W;
        p.WT = d.sage ? d.WTg : d.WT;
        p.din = d.kw;  // dagg width: the gapped [own | mean] layout for SageConv
        p.dout = d.dout;
        p.need_dagg = d.l > 0;
        p.gcn2 = d.spec.kind == GP_GCN2CONV;
        const float alpha = float(d.spec.alpha), beta = float(d.spec.beta);
        p.alpha = alpha;
        p.oma = 1.f - alpha;
        p.beta = beta;
        p.omb = 1.f - beta;
        p.dh0 = dh0;
        p.bg = d.bg;
        p.bgstride = d.skw;
        const size_t smem = p.need_dagg ? row_smem_bytes(d.dout, d.din, 2) : kEdgeSlotBytes;
        const double bytes = e * 8.0 + (e > 0 ? double(n) * d.dout * 4.0 : double(rows) * d.dout * 4.0) +
                             double(rows) * d.dout * 8.0 + (p.need_dagg ? double(rows) * d.din * 4.0 : 0.0) +
                             (p.gcn2 ? double(rows) * d.din * 8.0 : 0.0);
        const double flops = 2.0 * e * d.dout + (p.need_dagg ? 2.0 * double(rows) * d.din * d.dout : 0.0);
        const double gather = e * double(pad8(d.dout)) * 4.0;
        const int cls = prev == PREV_AGG || prev == PREV_AGG_ALL || prev == PREV_AGG_HIST || prev == PREV_SAGE ||
                                prev == PREV_SAGE_HIST
                            ? GP_K_BWD_AGG
                            : GP_K_BWD_DENSE;
        // SageConv layers (2*din-wide dagg) and SageConv neighbours always run split; so do
        // tcgen05 layers whatever feeds their gradient (a stage's last layer, PREV_TOP, too),
        // so a layer's arithmetic never depends on where the stage boundaries fall
        if ((split_rows && (cls == GP_K_BWD_AGG || (d.tc && p.need_dagg))) || d.sage || prev == PREV_SAGE ||
            prev == PREV_SAGE_HIST) {
            // gather (+ mask, dh0 term, ReLU) -> dz, then dz.W^T + mixes -> bg, dh0
            const double ab = e * 8.0 + double(n) * d.dout * 4.0 + double(rows) * d.dout * 8.0;
            launch(cls, ab, 2.0 * e * d.dout, gather, [&]() {
                switch (prev) {
                    case PREV_TOP: bwd_nb<PREV_TOP, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    case PREV_AGG: bwd_nb<PREV_AGG, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    case PREV_AGG_ALL: bwd_nb<PREV_AGG_ALL, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    case PREV_AGG_HIST: bwd_nb<PREV_AGG_HIST, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    case PREV_SAGE: bwd_nb<PREV_SAGE, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    case PREV_SAGE_HIST: bwd_nb<PREV_SAGE_HIST, OUT_LAYER, true>(rows, kEdgeSlotBytes, p); break;
                    default: bwd_nb<PREV_OWN, OUT_LAYER, true>(rows, kEdgeSlotBytes, p);
                }
            });
            if (p.need_dagg) {
                const double db = double(rows) * (d.dout + d.din) * 4.0 + (p.gcn2 ? double(rows) * d.din * 8.0 : 0.0) +
                                  double(d.din) * d.dout * 4.0;
                launch(GP_K_BWD_DENSE, db, 2.0 * double(rows) * d.din * d.dout, 0, [&]() {
                    if (d.tc) tc_xform_go<true>(tc_bwd_params(d, p));
                    else bwd_dense_go(rows, p);
                });
            }
            return;
        }
        switch (prev) {
            case PREV_TOP:
                launch(cls, bytes, flops, 0, [&]() { bwd_nb<PREV_TOP, OUT_LAYER>(rows, smem, p); });
                break;
            case PREV_AGG:
                launch(cls, bytes, flops, gather, [&]() { bwd_nb<PREV_AGG, OUT_LAYER>(rows, smem, p); });
                break;
            case PREV_AGG_ALL:
                launch(cls, bytes, flops, gather, [&]() { bwd_nb<PREV_AGG_ALL, OUT_LAYER>(rows, smem, p); });
                break;
            case PREV_AGG_HIST:
                launch(cls, bytes, flops, gather,
                       [&]() { bwd_nb<PREV_AGG_HIST, OUT_LAYER>(rows, smem, p); });
                break;
            default:
                launch(cls, bytes, flops, 0, [&]() { bwd_nb<PREV_OWN, OUT_LAYER>(rows, smem, p); });
        }
    }

    // backward_prev of local layer 0 on a non-first stage -> dh_in
    void backward_dhin(uint32_t r0, uint32_t r1, uint32_t t, uint64_t done) {
        auto& d = L[0];
        const uint32_t rows = r1 - r0;
        if (rows == 0) return;
        BwdParams p{};
        p.r0 = r0;
        p.r1 = r1;
        p.ticket = take_ticket();
        p.rowptr = rowptr;
        p.edges = edges;
        p.done = done;
        p.orig = orig;
        p.dh_width = d.din;
        p.bgn = d.bg;
        p.bgn_snap = d.bgs;
        p.bgnstride = d.skw;
        p.zrow = n;
        p.prev_mask = drop_key(t, d.l, d.din);
        p.dh_in = dh_in;
        p.dhinstride = sin0;
        p.rowptr_m = rowptr_m;
        p.edges_m = edges_mt;
        p.sgap = d.sgap;
        const double e = d.agg ? (hist ? double(rowptr_nnz(r0, r1)) : done_nnz(r0, r1, done)) : 0.0;
        const double bytes = e * 8.0 + (d.agg ? double(n) : double(rows)) * d.din * 4.0 + double(rows) * d.din * 4.0;
        if (d.sage)
            launch(GP_K_BWD_AGG, bytes, 2.0 * e * d.din, e * d.sin * 4.0, [&]() {
                if (hist) bwd_nb<PREV_SAGE_HIST, OUT_DHIN>(rows, kEdgeSlotBytes, p);
                else bwd_nb<PREV_SAGE, OUT_DHIN>(rows, kEdgeSlotBytes, p);
            });
        else if (!d.agg)
            launch(GP_K_BWD_DENSE, bytes, 0, 0, [&]() { bwd_nb<PREV_OWN, OUT_DHIN>(rows, kEdgeSlotBytes, p); });
        else if (hist)
            launch(GP_K_BWD_AGG, bytes, 2.0 * e * d.din, e * d.sin * 4.0,
                   [&]() { bwd_nb<PREV_AGG_HIST, OUT_DHIN>(rows, kEdgeSlotBytes, p); });
        else if (done == all_chunks() || bwd_csr_ready) {
            if (done != all_chunks()) {  // the same entries, pre-filtered
                p.rowptr = rowptr_f;
                p.edges = edges_f;
            }
            launch(GP_K_BWD_AGG, bytes, 2.0 * e * d.din, e * d.sin * 4.0,
                   [&]() { bwd_nb<PREV_AGG_ALL, OUT_DHIN>(rows, kEdgeSlotBytes, p); });
        }
        else
            launch(GP_K_BWD_AGG, bytes, 2.0 * e * d.din, e * d.sin * 4.0,
                   [&]() { bwd_nb<PREV_AGG, OUT_DHIN>(rows, kEdgeSlotBytes, p); });
    }

    uint64_t all_chunks() const { return K == 64 ? ~0ull : ((1ull << K) - 1); }

    XentParams xent_params(uint32_t r0, uint32_t r1) {
        auto& d = L[len - 1];
        XentParams p{};
        p.r0 = r0;
        p.r1 = r1;
        p.classes = d.dout;
        p.logits = d.h;
        p.lstride = d.sout;
        p.labels = labels;
        p.split = split;
        p.inv_count = inv_train;
        p.grad = dtop;
        p.gstride = d.sout;
        p.part_loss = part_loss;
        p.part_correct = part_correct;
        return p;
    }

    // Parameter gradients over this rank's own rows (param_grads_for_rows over
    // inner_sets[r], engines_impl.hpp:873-876), group sync (:877), optimizer (:878).
    void param_step() {
        ++step;  // Optimizer::step (nn.hpp:456-467): one update per epoch per stage
        const double c1d = 1.0 - std::pow(cfg.beta1, double(step));
        const double c2d = 1.0 - std::pow(cfg.beta2, double(step));
        const uint32_t rb = own_begin(), re = own_end(), nown = re - rb;
        for (uint32_t i = 0; i < len; ++i) {
            auto& d = L[i];
            // SageConv: dW rows [0, din) from pre's own half, [din, 2 din) from its mean half
            for (uint32_t half = 0; half < (d.sage ? 2u : 1u); ++half)
                pgrad_half(d, half, rb, re, nown);
        }
        if (G > 1) group_sync_grads();
        adam_all(c1d, c2d);
    }

    void pgrad_half(LayerDev& d, uint32_t half, uint32_t rb, uint32_t re, uint32_t nown) {
        {
            const float* pre = d.pre + (half ? d.sgap : 0);
            float* gW = d.gW + (half ? size_t(d.din) * d.dout : 0);
            float* gb = half ? nullptr : d.gb;
            const uint32_t ti = (d.din + 127) / 128, tj = 1;
            const double pg_bytes = double(nown) * (d.din * tj + d.dout * ti) * 4.0 + double(splits) * d.din * d.dout * 4.0;
            const double pg_flops = 2.0 * double(nown) * d.din * d.dout;
            uint32_t used_splits = splits;
            if (use_tc_pgrad) {
                // tcgen05 (3xTF32) split-K GEMM, one CTA per SM (TMEM accumulator, ~120 KB smem)
                used_splits = std::min<uint32_t>(splits, uint32_t(num_sms));
                TcPgradParams tp{nown, (nown + used_splits - 1) / used_splits, 0, pre, d.skw, d.dz, d.sout, d.din,
                                 d.dout, (d.dout + 15) / 16 * 16, ws, gb ? wsb : nullptr, id_rows};
                const size_t smem = tc_pgrad_smem(tp.npad);
                dim3 grid(used_splits, ti, 1);
                launch(GP_K_PGRAD, pg_bytes, pg_flops, 0, [&]() { k_pgrad_tc<<<grid, kTcThreads, smem, cs>>>(tp); });
            } else {
                const uint32_t rps = (nown + splits - 1) / splits;
                PgradParams pp{nown, rps, 0, pre, d.skw, d.dz, d.sout, d.din, d.dout, ws, gb ? wsb : nullptr, id_rows};
                dim3 grid(splits, ti, 1);
                launch(GP_K_PGRAD, pg_bytes, pg_flops, 0, [&]() { k_pgrad_partial<<<grid, 256, 0, cs>>>(pp); });
            }
            const uint32_t tot = d.din * d.dout + d.dout;
            const bool gcn2 = d.spec.kind == GP_GCN2CONV;
            launch(GP_K_PGRAD, double(splits) * tot * 4.0 + tot * 4.0, 0, 0, [&]() {
                k_pgrad_fold<<<(tot + 255) / 256, 256, 0, cs>>>(ws, gb ? wsb : nullptr, used_splits, d.din, d.dout,
                                                                float(d.spec.beta), gcn2, gW, gb);
            });
        }
    }

    // GP_FUSED_STEP=1 (default): the optimizer step and the derived weight copies of all
    // non-SageConv layers in one k_param_step launch (was 4-5 launches per layer)
    bool fused_step = true;
    StepLayer* step_table = nullptr;
    uint32_t step_max = 0;
    // the per-layer descriptor table of k_param_step, built at engine setup (gp_create), not
    // inside an epoch
    void build_step_table() {
        if (step_table || len == 0) return;
        std::vector<StepLayer> t(len);
        for (uint32_t i = 0; i < len; ++i) {
            auto& d = L[i];
            const bool g2 = d.spec.kind == GP_GCN2CONV && !tc_mix_epi;
            t[i] = StepLayer{d.W, d.gW, d.mW, d.vW, d.WT, d.b, d.gb, d.mb, d.vb, d.tc ? d.xf_fwd : nullptr,
                             d.tc ? d.xf_bwd : nullptr, d.din, d.dout, g2 ? 1u : 0u, float(d.spec.beta),
                             1.f - float(d.spec.beta)};
            step_max = std::max(step_max, d.din * d.dout + (d.b ? d.dout : 0u));
        }
        step_table = dalloc<StepLayer>(len, false);
        GP_CUDA(cudaMemcpyAsync(step_table, t.data(), t.size() * sizeof(StepLayer), cudaMemcpyHostToDevice, cs));
        GP_CUDA(cudaStreamSynchronize(cs));  // t is a host temporary
    }
    void adam_all(double c1d, double c2d) {
        bool any_sage = false;
        for (auto& d : L) any_sage |= d.sage;
        if (fused_step && !any_sage && len > 0 && len <= 65535) {
            if (!step_table) build_step_table();
            AdamParams a{};
            a.sgd = cfg.optimizer == 1;
            a.lr = float(cfg.lr);
            a.b1 = float(cfg.beta1);
            a.b2 = float(cfg.beta2);
            a.omb1 = 1.f - a.b1;
            a.omb2 = 1.f - a.b2;
            a.eps = float(cfg.eps);
            a.c1 = float(c1d);
            a.c2 = float(c2d);
            double elems = 0;
            for (auto& d : L) elems += double(d.din) * d.dout + (d.b ? d.dout : 0);
            const dim3 grid(std::min<uint32_t>((step_max + 255) / 256, 1024u), len);
            launch(GP_K_OPTIM, elems * 36.0, 0, 0, [&]() { k_param_step<<<grid, 256, 0, cs>>>(step_table, a); });
            return;
        }
        for (uint32_t i = 0; i < len; ++i) {
            auto& d = L[i];
            AdamParams a{};
            a.sgd = cfg.optimizer == 1;
            a.lr = float(cfg.lr);
            a.b1 = float(cfg.beta1);
            a.b2 = float(cfg.beta2);
            a.omb1 = 1.f - a.b1;
            a.omb2 = 1.f - a.b2;
            a.eps = float(cfg.eps);
            a.c1 = float(c1d);
            a.c2 = float(c2d);
            a.p = d.W;
            a.g = d.gW;
            a.m = d.mW;
            a.v = d.vW;
            a.n = d.kin * d.dout;
            launch(GP_K_OPTIM, a.n * 20.0, 0, 0, [&]() { k_adam<<<(a.n + 255) / 256, 256, 0, cs>>>(a); });
            transpose_w(d);
            if (d.b) {
                a.p = d.b;
                a.g = d.gb;
                a.m = d.mb;
                a.v = d.vb;
                a.n = d.dout;
                launch(GP_K_OPTIM, a.n * 20.0, 0, 0, [&]() { k_adam<<<1, 256, 0, cs>>>(a); });
            }
        }
    }

    // ---- transport ------------------------------------------------------------
    uint64_t bytes_sent[6] = {0, 0, 0, 0, 0, 0};
    uint64_t msgs_sent[6] = {0, 0, 0, 0, 0, 0};

    std::vector<Piece> fwd_pieces(uint32_t k, bool as_sender) {
        const uint32_t r0 = row_begin(k), rows = row_end(k) - row_begin(k);
        std::vector<Piece> v;
        if (as_sender) {
            auto& d = L[len - 1];
            v.push_back({d.h + size_t(r0) * d.sout, size_t(rows) * d.sout});
            if (needs_h0) v.push_back({(first ? L[0].h : h0) + size_t(r0) * pad8(H), size_t(rows) * pad8(H)});
        } else {
            v.push_back({in_cur + size_t(r0) * sin0, size_t(rows) * sin0});
            if (needs_h0) v.push_back({h0 + size_t(r0) * pad8(H), size_t(rows) * pad8(H)});
        }
        return v;
    }
    std::vector<Piece> bwd_pieces(uint32_t k, bool as_sender) {
        const uint32_t r0 = row_begin(k), rows = row_end(k) - row_begin(k);
        std::vector<Piece> v;
        if (as_sender) {
            v.push_back({dh_in + size_t(r0) * sin0, size_t(rows) * sin0});
        } else {
            auto& d = L[len - 1];
            v.push_back({dtop + size_t(r0) * d.sout, size_t(rows) * d.sout});
        }
        if (needs_h0) v.push_back({dh0 + size_t(r0) * pad8(H), size_t(rows) * pad8(H)});
        return v;
    }

    cudaEvent_t pool_event() {
        auto& tr_ = tr;
        if (tr_.ev_next == tr_.ev_pool.size()) {
            cudaEvent_t e;
            GP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            tr_.ev_pool.push_back(e);
        }
        return tr_.ev_pool[tr_.ev_next++];
    }

    void account(int tag, uint32_t k, uint32_t width) {
        const uint64_t rows = row_end(k) - row_begin(k);
        bytes_sent[tag] += rows * (uint64_t(width) + (needs_h0 ? H : 0)) * 4;  // 4 B/value (fabric.hpp:59)
        ++msgs_sent[tag];
    }

    void wait_local(LocalQueue& q, uint32_t k, LocalQueue::Msg& out) {
        std::unique_lock<std::mutex> lk(q.mu);
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(600);
        while (q.q.empty()) {
            if (q.aborted || aborted) throw Error(GP_EFABRIC, "transport aborted");
            if (q.cv.wait_until(lk, deadline) == std::cv_status::timeout && q.q.empty())
                throw Error(GP_EFABRIC, "watchdog: stage " + std::to_string(s) + " blocked on recv of chunk " +
                                            std::to_string(k));
        }
        out = std::move(q.q.front());
        q.q.pop_front();
        if (out.chunk != k)
            throw Error(GP_EFABRIC, "transport: expected chunk " + std::to_string(k) + ", got " +
                                        std::to_string(out.chunk));
    }

    void post_local(LocalQueue& q, uint32_t k, std::vector<Piece> src) {
        cudaEvent_t ev = pool_event();
        GP_CUDA(cudaEventRecord(ev, cs));
        std::lock_guard<std::mutex> lk(q.mu);
        if (q.aborted) throw Error(GP_EFABRIC, "transport aborted");
        q.q.push_back({k, ev, std::move(src), device});
        q.cv.notify_all();
    }

    void copy_in(const LocalQueue::Msg& m, const std::vector<Piece>& dst) {
        GP_CUDA(cudaStreamWaitEvent(cs, m.ready, 0));
        for (size_t i = 0; i < dst.size(); ++i) {
            if (m.device == device)
                GP_CUDA(cudaMemcpyAsync(dst[i].ptr, m.src[i].ptr, dst[i].floats * 4, cudaMemcpyDeviceToDevice, cs));
            else
                GP_CUDA(cudaMemcpyPeerAsync(dst[i].ptr, device, m.src[i].ptr, m.device, dst[i].floats * 4, cs));
        }
    }

    void nccl_xfer(void* comm, cudaStream_t st, int peer, const std::vector<Piece>& pcs, bool send) {
        cudaEvent_t ev = pool_event();
        GP_CUDA(cudaEventRecord(ev, cs));
        GP_CUDA(cudaStreamWaitEvent(st, ev, 0));
        nccl_check(g_nccl.group_start(), "ncclGroupStart");
        for (const auto& p : pcs) {
            if (send)
                nccl_check(g_nccl.send(p.ptr, p.floats, kNcclFloat, peer, comm, st), "ncclSend");
            else
                nccl_check(((NcclRecvFn)g_nccl.recv)(p.ptr, p.floats, kNcclFloat, peer, comm, st), "ncclRecv");
        }
        nccl_check(g_nccl.group_end(), "ncclGroupEnd");
        nccl_wait(comm, send ? "ncclSend" : "ncclRecv");  // non-blocking comm: enqueued
        cudaEvent_t done = pool_event();
        GP_CUDA(cudaEventRecord(done, st));
        GP_CUDA(cudaStreamWaitEvent(cs, done, 0));
    }

    // ---- CUDA-IPC rings (gp_link_ipc) --------------------------------------------
    // Host-side wait with a watchdog: an in-stream wait on a dead peer never
    // completes, so the epoch fails with GP_EFABRIC instead of hanging.
    void sync_watchdog(cudaStream_t st, double seconds) {
        cudaEvent_t e;
        GP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        GP_CUDA(cudaEventRecord(e, st));
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(seconds);
        for (;;) {
            const cudaError_t q = cudaEventQuery(e);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) {
                cudaEventDestroy(e);
                GP_CUDA(q);
            }
            if (aborted || std::chrono::steady_clock::now() > deadline) {
                // the event stays recorded on a stuck stream: leak it
                throw Error(GP_EFABRIC, "watchdog: stage " + std::to_string(s) +
                                            (aborted ? " aborted" : " blocked on a peer stage (IPC transport)"));
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
        cudaEventDestroy(e);
    }

    // Receive-ring slot sizes: the largest message of any chunk in that direction.
    uint64_t ipc_slot_floats(bool up_side) {
        uint64_t m = 0;
        for (uint32_t k = 0; k < K; ++k) {
            uint64_t t = 0;
            for (const auto& p : up_side ? fwd_pieces(k, false) : bwd_pieces(k, false)) t += p.floats;
            m = std::max(m, t);
        }
        return m;
    }

    void ipc_export(uint8_t* up_blob, uint8_t* down_blob) {
        GP_CUDA(cudaSetDevice(device));
        if (!graph_ready) throw Error(GP_EINVAL, "gp_ipc_export: upload the graph first");
        g_memops.load();
        for (int side = 0; side < 2; ++side) {
            uint8_t* out = side == 0 ? up_blob : down_blob;
            if (!out) continue;
            const bool present = side == 0 ? !first : !last;
            if (!present) throw Error(GP_EINVAL, side == 0 ? "gp_ipc_export: stage 0 has no upstream boundary"
                                                           : "gp_ipc_export: last stage has no downstream boundary");
            IpcSide& x = side == 0 ? tr.ipc_up : tr.ipc_down;
            if (!x.own) {
                x.own_R = std::min<uint32_t>(K, 3);
                x.own_slot = (ipc_slot_floats(side == 0) + 63) & ~uint64_t(63);
                x.own_bytes = kIpcRing + x.own_slot * 4 * x.own_R;
                x.own = dalloc<char>(x.own_bytes);  // zeroed: counters start at 0
                GP_CUDA(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking));
                GP_CUDA(cudaStreamCreateWithFlags(&x.rstream, cudaStreamNonBlocking));
            }
            IpcBlob b{};
            b.magic = kIpcMagic;
            b.version = GP_ABI_VERSION;
            b.stage = s;
            b.role = uint32_t(side);
            b.n = n;
            b.K = K;
            b.R = x.own_R;
            b.pad0 = grank;  // a stage link joins the same partition rank of adjacent stages
            b.slot_floats = x.own_slot;
            b.bytes = x.own_bytes;
            b.ptr = uint64_t(reinterpret_cast<uintptr_t>(x.own));
            b.pid = int32_t(getpid());
            b.device = device;
            GP_CUDA(cudaIpcGetMemHandle(&b.handle, x.own));
            std::memset(out, 0, GP_IPC_BLOB_BYTES);
            std::memcpy(out, &b, sizeof(b));
        }
    }

    void ipc_link(const uint8_t* up_peer, const uint8_t* down_peer) {
        GP_CUDA(cudaSetDevice(device));
        for (int side = 0; side < 2; ++side) {
            const uint8_t* in = side == 0 ? up_peer : down_peer;
            if (!in) continue;
            IpcSide& x = side == 0 ? tr.ipc_up : tr.ipc_down;
            if (!x.own) throw Error(GP_EINVAL, "gp_link_ipc: call gp_ipc_export for this side first");
            if (x.peer) throw Error(GP_EINVAL, "gp_link_ipc: side already linked");
            IpcBlob b;
            std::memcpy(&b, in, sizeof(b));
            // up side pairs with the upstream stage's down region and vice versa
            const uint32_t want_stage = side == 0 ? s - 1 : s + 1, want_role = side == 0 ? 1u : 0u;
            if (b.magic != kIpcMagic || b.version != GP_ABI_VERSION) throw Error(GP_EINVAL, "gp_link_ipc: not an IPC blob");
            if (b.stage != want_stage || b.role != want_role)
                throw Error(GP_EINVAL, "gp_link_ipc: blob of stage " + std::to_string(b.stage) + " role " +
                                           std::to_string(b.role) + " does not face this boundary");
            if (b.n != n || b.K != K) throw Error(GP_EINVAL, "gp_link_ipc: N/K mismatch");
            if (b.pad0 != grank) throw Error(GP_EINVAL, "gp_link_ipc: peer is another partition rank");
            // Two stages in one CUDA context must not wait on each other in-stream: any
            // implicit context synchronisation (module loading, frees, ...) on one stage's
            // host thread then waits for the other stage's pending wait, whose value that
            // thread has yet to enqueue. Same-process peers on one device link locally.
            if (b.pid == int32_t(getpid()) && b.device == device)
                throw Error(GP_EINVAL,
                            "gp_link_ipc: the peer stage shares this process's CUDA context (same device); "
                            "use gp_link_local");
            if (b.pid == int32_t(getpid())) {
                x.peer = reinterpret_cast<char*>(uintptr_t(b.ptr));  // same process: plain UVA pointer
                if (b.device != device) {
                    cudaDeviceEnablePeerAccess(b.device, 0);
                    cudaGetLastError();
                }
            } else {
                void* p = nullptr;
                GP_CUDA(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess));
                x.peer = static_cast<char*>(p);
                x.peer_opened = true;
            }
            x.peer_slot = b.slot_floats;
            x.peer_R = b.R;
        }
    }

    CUdeviceptr dptr(char* base, size_t off) { return CUdeviceptr(reinterpret_cast<uintptr_t>(base + off)); }

    bool ipc_smcopy = false;  // GP_IPC_SMCOPY=1: message copies as kernels instead of copy-engine memcpy
    void ipc_copy(float* dst, const float* src, size_t floats, cudaStream_t st) {
        if (!floats) return;
        if (ipc_smcopy) {
            const uint32_t blocks = uint32_t(std::min<size_t>(size_t(num_sms) * 2, (floats / 4 + 255) / 256 + 1));
            k_copy<<<blocks, 256, 0, st>>>(dst, src, floats);
            GP_CUDA(cudaGetLastError());
        } else {
            GP_CUDA(cudaMemcpyAsync(dst, src, floats * 4, cudaMemcpyDefault, st));
        }
    }

    void ipc_send(IpcSide& x, uint32_t k, const std::vector<Piece>& pcs) {
        uint64_t tot = 0;
        for (const auto& p : pcs) tot += p.floats;
        if (tot > x.peer_slot)
            throw Error(GP_EFABRIC, "IPC send of chunk " + std::to_string(k) + " exceeds the peer's slot");
        const uint32_t seq = ++x.send_seq, slot = (seq - 1) % x.peer_R;
        cudaEvent_t ev = pool_event();
        GP_CUDA(cudaEventRecord(ev, cs));
        GP_CUDA(cudaStreamWaitEvent(x.stream, ev, 0));
        if (seq > x.peer_R)  // slot reuse: the receiver has unpacked message seq - R
            cu_check(g_memops.wait(x.stream, dptr(x.own, kIpcAck), seq - x.peer_R, CU_STREAM_WAIT_VALUE_GEQ),
                     "cuStreamWaitValue32(ack)");
        float* dst = reinterpret_cast<float*>(x.peer + kIpcRing) + size_t(slot) * x.peer_slot;
        for (const auto& p : pcs) {
            ipc_copy(dst, p.ptr, p.floats, x.stream);
            dst += p.floats;
        }
        cu_check(g_memops.write(x.stream, dptr(x.peer, kIpcReady), seq, CU_STREAM_WRITE_VALUE_DEFAULT),
                 "cuStreamWriteValue32(ready)");
    }

    // Receive on the side's own stream, in message order (the ack counter stays
    // monotone whichever compute stream consumes the chunk); compute waits on it.
    void ipc_recv(IpcSide& x, const std::vector<Piece>& pcs) {
        const uint32_t seq = ++x.recv_seq, slot = (seq - 1) % x.own_R;
        cudaStream_t rs = x.rstream;
        cudaEvent_t go = pool_event();
        GP_CUDA(cudaEventRecord(go, cs));  // destination rows are free once cs got here
        GP_CUDA(cudaStreamWaitEvent(rs, go, 0));
        cu_check(g_memops.wait(rs, dptr(x.own, kIpcReady), seq, CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32(ready)");
        const float* src = reinterpret_cast<const float*>(x.own + kIpcRing) + size_t(slot) * x.own_slot;
        for (const auto& p : pcs) {
            ipc_copy(p.ptr, src, p.floats, rs);
            src += p.floats;
        }
        cu_check(g_memops.write(rs, dptr(x.peer, kIpcAck), seq, CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32(ack)");
        cudaEvent_t done = pool_event();
        GP_CUDA(cudaEventRecord(done, rs));
        GP_CUDA(cudaStreamWaitEvent(cs, done, 0));
    }

    void send_fwd(uint32_t k) {
        account(0, k, L[len - 1].dout);
        if (tr.ipc_down.linked()) ipc_send(tr.ipc_down, k, fwd_pieces(k, true));
        else if (tr.down_local) post_local(tr.down_local->fwd, k, fwd_pieces(k, true));
        else if (tr.down_comm) nccl_xfer(tr.down_comm, tr.down_stream, 1, fwd_pieces(k, true), true);
        else throw Error(GP_EFABRIC, "no downstream link");
    }
    void recv_fwd(uint32_t k) {
        if (tr.ipc_up.linked()) {
            ipc_recv(tr.ipc_up, fwd_pieces(k, false));
        } else if (tr.up_local) {
            LocalQueue::Msg m;
            wait_local(tr.up_local->fwd, k, m);
            copy_in(m, fwd_pieces(k, false));
        } else if (tr.up_comm) {
            nccl_xfer(tr.up_comm, tr.up_stream, 0, fwd_pieces(k, false), false);
        } else {
            throw Error(GP_EFABRIC, "no upstream link");
        }
    }
    void send_bwd(uint32_t k) {
        account(1, k, in0);
        if (tr.ipc_up.linked()) ipc_send(tr.ipc_up, k, bwd_pieces(k, true));
        else if (tr.up_local) post_local(tr.up_local->bwd, k, bwd_pieces(k, true));
        else if (tr.up_comm) nccl_xfer(tr.up_comm, tr.up_stream, 0, bwd_pieces(k, true), true);
        else throw Error(GP_EFABRIC, "no upstream link");
    }
    void recv_bwd(uint32_t k) {
        if (tr.ipc_down.linked()) {
            ipc_recv(tr.ipc_down, bwd_pieces(k, false));
        } else if (tr.down_local) {
            LocalQueue::Msg m;
            wait_local(tr.down_local->bwd, k, m);
            copy_in(m, bwd_pieces(k, false));
        } else if (tr.down_comm) {
            nccl_xfer(tr.down_comm, tr.down_stream, 1, bwd_pieces(k, false), false);
        } else {
            throw Error(GP_EFABRIC, "no downstream link");
        }
    }

    // ---- hybrid group across processes ------------------------------------------
    std::vector<char*> group_buffers() const {
        std::vector<char*> v;
        auto add = [&](const void* p) {
            if (p) v.push_back(static_cast<char*>(const_cast<void*>(p)));
        };
        for (const auto& d : L) {
            add(d.h);
            add(d.hs);
            add(d.bg);
            add(d.bgs);
            add(d.gW);
            add(d.gb);
        }
        add(in_cur);
        add(in_snap);
        return v;
    }

    struct GroupBlobHead {
        uint32_t magic, version, stage, G, grank, nbufs, n, K;
        int32_t pid, device;
        uint64_t flags_ptr;
        cudaIpcMemHandle_t flags;
    };
    struct GroupBlobBuf {
        uint64_t ptr;
        cudaIpcMemHandle_t h;
    };

    size_t group_export(uint8_t* out, size_t cap) {
        GP_CUDA(cudaSetDevice(device));
        if (G < 2) throw Error(GP_EINVAL, "gp_group_export: not a hybrid worker (group_size < 2)");
        if (G > kGroupMaxRanks) throw Error(GP_EINVAL, "gp_group_export: group_size > 8");
        if (!graph_ready) throw Error(GP_EINVAL, "gp_group_export: upload the graph first");
        if (last_epoch != 0) throw Error(GP_EINVAL, "gp_group_export: link before the first epoch");
        g_memops.load();
        auto& ig = tr.ipcg;
        if (!ig.own_flags) {
            ig.own_flags = dalloc<char>(size_t(kGroupKinds) * kGroupMaxRanks * 4);
            ig.own_bufs = group_buffers();
        }
        const size_t need = sizeof(GroupBlobHead) + ig.own_bufs.size() * sizeof(GroupBlobBuf);
        if (!out) return need;
        if (cap < need) throw Error(GP_EINVAL, "gp_group_export: blob buffer too small");
        GroupBlobHead h{};
        h.magic = kGroupMagic;
        h.version = GP_ABI_VERSION;
        h.stage = s;
        h.G = G;
        h.grank = grank;
        h.nbufs = uint32_t(ig.own_bufs.size());
        h.n = n;
        h.K = K;
        h.pid = int32_t(getpid());
        h.device = device;
        h.flags_ptr = uint64_t(reinterpret_cast<uintptr_t>(ig.own_flags));
        GP_CUDA(cudaIpcGetMemHandle(&h.flags, ig.own_flags));
        std::memcpy(out, &h, sizeof(h));
        for (size_t j = 0; j < ig.own_bufs.size(); ++j) {
            GroupBlobBuf b{};
            b.ptr = uint64_t(reinterpret_cast<uintptr_t>(ig.own_bufs[j]));
            GP_CUDA(cudaIpcGetMemHandle(&b.h, ig.own_bufs[j]));
            std::memcpy(out + sizeof(h) + j * sizeof(b), &b, sizeof(b));
        }
        return need;
    }

    void group_link_ipc(const uint8_t* const* blobs, const uint64_t* lens) {
        GP_CUDA(cudaSetDevice(device));
        auto& ig = tr.ipcg;
        if (!ig.own_flags) throw Error(GP_EINVAL, "gp_link_group_ipc: call gp_group_export first");
        if (ig.linked || tr.group) throw Error(GP_EINVAL, "gp_link_group_ipc: group already linked");
        ig.peer_bufs.assign(G, {});
        ig.peer_flags.assign(G, nullptr);
        const int32_t me = int32_t(getpid());
        auto open = [&](const cudaIpcMemHandle_t& h, uint64_t ptr, int32_t pid) -> char* {
            if (pid == me) return reinterpret_cast<char*>(uintptr_t(ptr));
            void* p = nullptr;
            GP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            ig.opened.push_back(static_cast<char*>(p));
            return static_cast<char*>(p);
        };
        for (uint32_t r = 0; r < G; ++r) {
            if (r == grank) continue;
            if (!blobs || !blobs[r] || lens[r] < sizeof(GroupBlobHead))
                throw Error(GP_EINVAL, "gp_link_group_ipc: missing blob of rank " + std::to_string(r));
            GroupBlobHead h;
            std::memcpy(&h, blobs[r], sizeof(h));
            if (h.magic != kGroupMagic || h.version != GP_ABI_VERSION)
                throw Error(GP_EINVAL, "gp_link_group_ipc: not a group blob");
            if (h.stage != s || h.G != G || h.grank != r || h.n != n || h.K != K ||
                h.nbufs != ig.own_bufs.size() || lens[r] < sizeof(h) + size_t(h.nbufs) * sizeof(GroupBlobBuf))
                throw Error(GP_EINVAL, "gp_link_group_ipc: blob of rank " + std::to_string(r) +
                                           " does not match this group member");
            ig.peer_flags[r] = open(h.flags, h.flags_ptr, h.pid);
            for (uint32_t j = 0; j < h.nbufs; ++j) {
                GroupBlobBuf b;
                std::memcpy(&b, blobs[r] + sizeof(h) + size_t(j) * sizeof(b), sizeof(b));
                ig.peer_bufs[r].push_back(open(b.h, b.ptr, h.pid));
            }
        }
        ig.linked = true;
    }

    // Peer r's buffer that plays the role of my buffer `mine` (same export index).
    const float* peer_of(uint32_t r, const void* mine) const {
        const auto& ig = tr.ipcg;
        for (size_t j = 0; j < ig.own_bufs.size(); ++j)
            if (ig.own_bufs[j] == mine) return reinterpret_cast<const float*>(ig.peer_bufs[r][j]);
        throw Error(GP_ERUNTIME, "group transport: buffer not exported");
    }

    void ipcg_signal(uint32_t dst, uint32_t kind, uint32_t value) {
        cu_check(g_memops.write(cs, dptr(tr.ipcg.peer_flags[dst], IpcGroup::off(kind, grank)), value,
                                CU_STREAM_WRITE_VALUE_DEFAULT),
                 "cuStreamWriteValue32(group)");
    }
    void ipcg_wait(uint32_t src, uint32_t kind, uint32_t value) {
        cu_check(g_memops.wait(cs, dptr(tr.ipcg.own_flags, IpcGroup::off(kind, src)), value, CU_STREAM_WAIT_VALUE_GEQ),
                 "cuStreamWaitValue32(group)");
    }

    // ---- hybrid group operations (G > 1) ----------------------------------------
    // FIFO tags: (kind-specific id) so every pull checks it got the expected message.
    static uint32_t halo_tag(uint32_t layer, uint32_t k) { return (layer << 8) | (k & 0xff); }

    void group_post(uint32_t kind, uint32_t tag, std::vector<Piece> src) {
        if (tr.ipcg.linked) {  // rows are final once cs gets here: bump every peer's counter
            const uint32_t seq = ++tr.ipcg.post_seq[kind];
            for (uint32_t r2 = 0; r2 < G; ++r2)
                if (r2 != grank) ipcg_signal(r2, kind, seq);
            return;
        }
        if (!tr.group) throw Error(GP_EFABRIC, "hybrid worker without a group link");
        auto& gl = *tr.group;
        cudaEvent_t ev = pool_event();
        GP_CUDA(cudaEventRecord(ev, cs));
        for (uint32_t r2 = 0; r2 < G; ++r2) {
            if (r2 == grank) continue;
            auto& q = gl.at(grank, r2, kind);
            std::lock_guard<std::mutex> lk(q.mu);
            if (q.aborted) throw Error(GP_EFABRIC, "transport aborted");
            q.q.push_back({tag, ev, src, device});
            q.cv.notify_all();
        }
    }

    // Pull the halo rows of chunks [k_lo, k_hi) from every peer's buffer.
    // dst = base + col0 (col0: SageConv's aggregated half of bg); peers' rows are read
    // from the matching column of their own buffer
    void halo_pull(uint32_t kind, uint32_t tag, uint32_t k_lo, uint32_t k_hi, float* dst, uint32_t stride,
                   float* dstG, uint32_t gstride, uint32_t width, const DropKey& key, uint32_t col0 = 0) {
        for (uint32_t r2 = 0; r2 < G; ++r2) {
            if (r2 == grank) continue;
            const float* src = nullptr;
            if (tr.ipcg.linked) {
                ipcg_wait(r2, kind, ++tr.ipcg.recv_seq[kind][r2]);
                src = peer_of(r2, dst - col0) + col0;
            } else {
                if (!tr.group) throw Error(GP_EFABRIC, "hybrid worker without a group link");
                LocalQueue::Msg m;
                wait_local(tr.group->at(r2, grank, kind), tag, m);
                GP_CUDA(cudaStreamWaitEvent(cs, m.ready, 0));
                src = m.src[0].ptr + col0;
            }
            const uint32_t a = pull_off[size_t(r2) * (K + 1) + k_lo], b = pull_off[size_t(r2) * (K + 1) + k_hi];
            if (b == a) continue;
            PullParams p{pull_idx + a, b - a, src, dst, stride, dstG, gstride, width, orig, key};
            launch(GP_K_XFER, double(b - a) * width * (dstG ? 12.0 : 8.0), 0, 0,
                   [&]() { k_pull_rows<<<row_grid(b - a, (const void*)k_pull_rows, 0), kBlock, 0, cs>>>(p); });
        }
    }

    // Ledger of one halo exchange (sender side, 4 B/value): rows this rank pushes.
    void count_halo(int tag, uint32_t k_lo, uint32_t k_hi, uint32_t width) {
        for (uint32_t r2 = 0; r2 < G; ++r2) {
            if (r2 == grank) continue;
            uint64_t rows = 0;
            for (uint32_t k = k_lo; k < k_hi; ++k) rows += push_cnt[size_t(k) * G + r2];
            bytes_sent[tag] += rows * width * 4;
            if (rows) ++msgs_sent[tag];
        }
    }

    // Forward halo of local layer i for chunks [k_lo, k_hi): before layer i reads
    // neighbours, pull peers' current input rows (and their dropped copies).
    void halo_fwd(uint32_t i, uint32_t k_lo, uint32_t k_hi, uint32_t t) {
        auto& d = L[i];
        count_halo(2, k_lo, k_hi, d.din);
        if (i == 0 && first) return;  // stage-0 features are replicated: identical rows
        float* cur = const_cast<float*>(cur_src(i));
        const uint32_t tag = halo_tag(d.l, k_hi - k_lo == K ? 0xff : k_lo);
        group_post(0, tag, {Piece{cur, 0}});
        halo_pull(0, tag, k_lo, k_hi, cur, src_stride(i), d.G, d.sin, d.din, drop_key(t, d.l, d.din));
    }

    // Backward halo of local layer i: after backward_out_row wrote this layer's
    // dagg rows, pull the peers' boundary rows before backward_prev_row reads them.
    void halo_bwd(uint32_t i, uint32_t k_lo, uint32_t k_hi) {
        auto& d = L[i];
        count_halo(3, k_lo, k_hi, d.din);
        if (d.l == 0) return;  // global layer 0 never propagates further (no dagg kept)
        const uint32_t tag = halo_tag(d.l, k_hi - k_lo == K ? 0xff : k_lo);
        group_post(1, tag, {Piece{d.bg, 0}});
        // SageConv: neighbours read the aggregated half of dagg (exchange_rows offset in, :838-844)
        halo_pull(1, tag, k_lo, k_hi, d.bg + d.sgap, d.skw, nullptr, 0, d.din, DropKey{}, d.sgap);
    }

    // group_weight_sync: rank 0 folds in rank order and everyone takes its result.
    void group_sync_grads() {
        std::vector<Piece> mine;
        uint64_t values = 0;
        for (auto& d : L) {
            mine.push_back({d.gW, size_t(d.kin) * d.dout});
            values += uint64_t(d.kin) * d.dout;
            if (d.gb) {
                mine.push_back({d.gb, d.dout});
                values += d.dout;
            }
        }
        if (tr.ipcg.linked) {
            // counters: 2 grads ready (-> rank 0), 3 fold done (-> rank r), 4 copied (-> rank 0)
            const uint32_t seq = ++tr.ipcg.sync_seq;
            if (grank != 0) {
                ipcg_signal(0, 2, seq);
                ipcg_wait(0, 3, seq);
                for (auto& m : mine)
                    GP_CUDA(cudaMemcpyAsync(m.ptr, peer_of(0, m.ptr), m.floats * 4, cudaMemcpyDefault, cs));
                ipcg_signal(0, 4, seq);
                bytes_sent[4] += values * 4;
                ++msgs_sent[4];
                return;
            }
            for (uint32_t r2 = 1; r2 < G; ++r2) ipcg_wait(r2, 2, seq);
            for (auto& m : mine) {
                FoldParams f{};
                f.src[0] = m.ptr;
                for (uint32_t r2 = 1; r2 < G; ++r2) f.src[r2] = peer_of(r2, m.ptr);
                f.dst = m.ptr;
                f.G = G;
                f.n = uint32_t(m.floats);
                launch(GP_K_XFER, double(f.n) * 4.0 * (G + 1), 0, 0,
                       [&]() { k_group_fold<<<(f.n + 255) / 256, 256, 0, cs>>>(f); });
            }
            for (uint32_t r2 = 1; r2 < G; ++r2) ipcg_signal(r2, 3, seq);
            // the folded result lives in this rank's gradient buffers, which the next
            // epoch overwrites: wait until every peer has copied it
            for (uint32_t r2 = 1; r2 < G; ++r2) ipcg_wait(r2, 4, seq);
            bytes_sent[4] += uint64_t(G - 1) * values * 4;
            msgs_sent[4] += G - 1;
            return;
        }
        if (!tr.group) throw Error(GP_EFABRIC, "hybrid worker without a group link");
        auto& gl = *tr.group;
        if (grank != 0) {
            cudaEvent_t ev = pool_event();
            GP_CUDA(cudaEventRecord(ev, cs));
            {
                auto& q = gl.at(grank, 0, 2);
                std::lock_guard<std::mutex> lk(q.mu);
                if (q.aborted) throw Error(GP_EFABRIC, "transport aborted");
                q.q.push_back({0u, ev, mine, device});
                q.cv.notify_all();
            }
            bytes_sent[4] += values * 4;
            ++msgs_sent[4];
            LocalQueue::Msg m;
            wait_local(gl.at(0, grank, 2), 1u, m);
            GP_CUDA(cudaStreamWaitEvent(cs, m.ready, 0));
            for (size_t j = 0; j < mine.size(); ++j)
                GP_CUDA(cudaMemcpyAsync(mine[j].ptr, m.src[j].ptr, mine[j].floats * 4, cudaMemcpyDeviceToDevice, cs));
            return;
        }
        std::vector<LocalQueue::Msg> peers(G);
        for (uint32_t r2 = 1; r2 < G; ++r2) {
            wait_local(gl.at(r2, 0, 2), 0u, peers[r2]);
            GP_CUDA(cudaStreamWaitEvent(cs, peers[r2].ready, 0));
        }
        for (size_t j = 0; j < mine.size(); ++j) {
            FoldParams f{};
            f.src[0] = mine[j].ptr;
            for (uint32_t r2 = 1; r2 < G; ++r2) f.src[r2] = peers[r2].src[j].ptr;
            f.dst = mine[j].ptr;
            f.G = G;
            f.n = uint32_t(mine[j].floats);
            launch(GP_K_XFER, double(f.n) * 4.0 * (G + 1), 0, 0,
                   [&]() { k_group_fold<<<(f.n + 255) / 256, 256, 0, cs>>>(f); });
        }
        group_post(2, 1u, mine);
        bytes_sent[4] += uint64_t(G - 1) * values * 4;
        msgs_sent[4] += G - 1;
    }

    // ---- trace helpers ----------------------------------------------------------
    cudaEvent_t trace_mark() {
        if (!tracing) return nullptr;
        cudaEvent_t e = take_event();
        GP_CUDA(cudaEventRecord(e, cs));
        return e;
    }
    void trace_add(uint32_t kind, int32_t chunk, cudaEvent_t a, cudaEvent_t b) {
        if (!tracing) return;
        trace_pending.push_back({trace_epoch, kind, chunk, int32_t(lb), int32_t(le) - 1, a, b});
    }
    // Idle span while blocked on the message of chunk k, then the Recv instant
    // (fabric.cpp:350-357).
    template <class F>
    void traced_recv(uint32_t k, F&& recv) {
        cudaEvent_t a = trace_mark();
        recv();
        cudaEvent_t b = trace_mark();
        trace_add(GP_TRACE_IDLE, int32_t(k), a, b);
        trace_add(GP_TRACE_RECV, int32_t(k), b, b);
    }
    template <class F>
    void traced_send(uint32_t k, F&& send) {
        cudaEvent_t a = trace_mark();
        trace_add(GP_TRACE_SEND, int32_t(k), a, a);  // instant at send time (fabric.cpp:293-295)
        send();
    }
    void trace_begin_epoch(uint32_t t) {
        if (!tracing) return;
        if (!trace_origin) GP_CUDA(cudaEventCreate(&trace_origin));
        if (!trace_stamp) GP_CUDA(cudaHostAlloc(&trace_stamp, 8, cudaHostAllocMapped));
        trace_epoch = t;
        GP_CUDA(cudaEventRecord(trace_origin, cs));
        unsigned long long* dptr = nullptr;
        GP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), trace_stamp, 0));
        k_stamp<<<1, 1, 0, cs>>>(dptr);
        GP_CUDA(cudaGetLastError());
    }
    // after the epoch's stream synchronize
    void trace_resolve() {
        if (trace_pending.empty()) return;
        const double base = double(*trace_stamp);
        auto at = [&](cudaEvent_t e) {
            float ms = 0.f;
            GP_CUDA(cudaEventElapsedTime(&ms, trace_origin, e));
            return base + double(ms) * 1e6;
        };
        for (const auto& r : trace_pending) {
            gp_trace_event e{};
            e.epoch = r.epoch;
            e.kind = r.kind;
            e.chunk = r.chunk;
            e.layer_lo = r.llo;
            e.layer_hi = r.lhi;
            e.t_start_ns = at(r.a);
            e.t_end_ns = r.b == r.a ? e.t_start_ns : at(r.b);
            trace_done.push_back(e);
        }
        // an event can close one record and open the next (idle -> recv): recycle once
        std::vector<cudaEvent_t> used;
        for (const auto& r : trace_pending) used.insert(used.end(), {r.a, r.b});
        std::sort(used.begin(), used.end());
        used.erase(std::unique(used.begin(), used.end()), used.end());
        ev_free.insert(ev_free.end(), used.begin(), used.end());
        trace_pending.clear();
    }

    // ---- one epoch ---------------------------------------------------------------
    // ---- chunk wavefront helpers ------------------------------------------------
    // W compute streams; chunk j runs on stream j % W. Off for hybrid groups (halo
    // exchange is ordered on one stream), K = 1, and in profiling mode (clean
    // per-kernel times). Merged gather tables rely on the one-stream order for hybrid
    // groups: a halo pull overwrites chunk k's boundary rows of G_i, which earlier chunks
    // gather as snapshot rows; on one stream those gathers are complete by then (with W > 1
    // the pull would need the before_g_write ordering the producer epilogues get).
    int wave_width() const { return G == 1 && K > 1 && !profiling && !tracing ? wave_w : 1; }
    cudaStream_t wave_stream(uint32_t j, int W, cudaStream_t main) const { return j % W ? cs_side[j % W] : main; }
    cudaEvent_t record_event() {
        cudaEvent_t e = pool_event();
        GP_CUDA(cudaEventRecord(e, cs));
        return e;
    }
    void wave_fork(int W) {
        if (W < 2) return;
        cudaEvent_t e = record_event();
        for (int w = 1; w < W; ++w) GP_CUDA(cudaStreamWaitEvent(cs_side[w], e, 0));
    }
    void wave_join(int W, cudaStream_t main) {
        for (int w = 1; w < W; ++w) {
            cudaEvent_t e = pool_event();
            GP_CUDA(cudaEventRecord(e, cs_side[w]));
            GP_CUDA(cudaStreamWaitEvent(main, e, 0));
        }
    }

    // Lean layout: snap := cur for every stash the next epoch reads stale rows from
    // (all n rows: hybrid halo rows pulled into cur are part of the snapshot, like the
    // reference's whole-matrix copy). backward = true: the historical dagg tables.
    void copy_snapshots(bool backward) {
        auto copy = [&](float* dst, const float* src, size_t floats) {  // SM copy at HBM rate
            if (!dst || !src || dst == src) return;
            const uint32_t blocks = uint32_t(std::min<size_t>(size_t(num_sms) * 8, (floats / 4 + 255) / 256 + 1));
            launch(GP_K_REMASK, double(floats) * 8.0, 0, 0, [&]() { k_copy<<<blocks, 256, 0, cs>>>(dst, src, floats); });
        };
        if (backward) {
            for (auto& d : L) copy(d.bgs, d.bg, size_t(n) * d.skw);
            return;
        }
        copy(in_snap, in_cur, size_t(n) * sin0);
        for (uint32_t i = 0; i < len; ++i)
            if (!(i < dual_done.size() && dual_done[i])) copy(L[i].hs, L[i].h, size_t(n) * L[i].sout);
    }

    void run_epoch(uint32_t t, const uint32_t* order, gp_epoch_stats* out) {
        GP_CUDA(cudaSetDevice(device));
        if (!graph_ready) throw Error(GP_EINVAL, "graph not uploaded");
        if (first && !x_ready) throw Error(GP_EINVAL, "features not uploaded");
        if (last && !labels_ready) throw Error(GP_EINVAL, "labels not uploaded");
        if (t == 0) throw Error(GP_EINVAL, "epochs are 1-based");
        std::vector<uint32_t> ord(order, order + K);
        {
            std::vector<uint8_t> seen(K, 0);
            for (uint32_t k : ord) {
                if (k >= K || seen[k]) throw Error(GP_EINVAL, "order is not a permutation of 0..K-1");
                seen[k] = 1;
            }
        }
        const auto h_start = std::chrono::steady_clock::now();
        std::fill(bytes_sent, bytes_sent + 6, 0);
        std::fill(msgs_sent, msgs_sent + 6, 0);
        launches = 0;
        tr.ev_next = 0;
        zero_words(tickets, kTickets);
        ticket_next = 0;
        GP_CUDA(cudaEventRecord(ev_start, cs));
        trace_begin_epoch(t);

        // Snapshot (engines_impl.hpp:671-679): snap := cur. Every cur row is
        // rewritten before it is read again, so a pointer swap is exact.
        const uint32_t fix_alpha = std::max<uint32_t>(1, cfg.fix_alpha);
        if (!sync && (t - 1) % fix_alpha == 0) {
            if (!lean) {
                if (in_snap) std::swap(in_snap, in_cur);
                for (auto& d : L) {
                    if (d.hs) std::swap(d.hs, d.h);
                    if (d.bgs) std::swap(d.bgs, d.bg);
                }
            } else if (!(t == 1 && last_epoch == 0) && last_epoch != t - 1 && !state_restored) {
                // lean snapshots are copied at the end of epoch t-1 (copy_snapshots)
                throw Error(GP_EINVAL, "lean stash layout: epoch " + std::to_string(t) +
                                           " refreshes the snapshot but epoch " + std::to_string(t - 1) +
                                           " did not run here (restore it with gp_set_history, or GP_LEAN=0)");
            }
        }
        state_restored = false;
        dual_snap = lean && !sync && G == 1 && t % fix_alpha == 0;
        dual_done.assign(len, 0);
        // Masked gather sources start from the snapshot rows (stale reads). With
        // remask_overlap, layers >= 1 are remasked on cs_prep; rm_ev[i] orders every chunk's
        // first write of G_i (the layer i-1 epilogue) and read of it after the remask.
        std::vector<cudaEvent_t> rm_ev(len, nullptr);
        const bool ovl = remask_overlap && cs_prep && !sync && !profiling;  // profiling: one launch at a time
        if (ovl) GP_CUDA(cudaStreamWaitEvent(cs_prep, record_event(), 0));
        for (uint32_t i = 0; i < len; ++i) {
            if (!L[i].agg) continue;
            if (i == 0 && first) {
                remask(0, x0, 0, n, drop_key(t, L[0].l, L[0].din));  // cur == snap == x0
            } else if (!sync) {
                if (ovl && i > 0) {
                    cudaStream_t main = cs;
                    cs = cs_prep;
                    remask(i, snap_src(i), 0, n, drop_key(t, L[i].l, L[i].din), true);
                    rm_ev[i] = record_event();
                    cs = main;
                } else {
                    remask(i, snap_src(i), 0, n, drop_key(t, L[i].l, L[i].din), true);
                }
            }
        }
        auto wait_remask = [&](uint32_t i) {  // before a kernel that writes or reads G_i
            if (i < len && rm_ev[i]) GP_CUDA(cudaStreamWaitEvent(cs, rm_ev[i], 0));
        };

        // ---- forward -----------------------------------------------------------
        const uint64_t all_done = K == 64 ? ~0ull : ((1ull << K) - 1);
        if (!sync) {
            // Multi-stream wavefront (SURVEY §8(a')9): chunk j+1 runs layer i while chunk
            // j runs layer i+1. Legal because gathers read done chunks from G (rows
            // written this epoch) and not-done chunks from the separate snapshot table
            // Gs, so a chunk never reads rows the concurrent chunk is writing; the one
            // cross-chunk dependency ("layer i of chunk j+1 reads G_i rows of chunk j,
            // written by chunk j's layer i-1 / input remask") is one event.
            const int W = wave_width();
            cudaStream_t main = cs;
            struct Restore {
                cudaStream_t& ref;
                cudaStream_t v;
                ~Restore() { ref = v; }
            } restore{cs, main};
            // ev[j % W][i]: chunk j's input (i = 0) / layer i-1 output (i >= 1) is written
            std::vector<std::vector<cudaEvent_t>> ev(W, std::vector<cudaEvent_t>(len + 1, nullptr));
            // merged_g: rd[j % W][i]: chunk j's gather from G_i has finished; chunk j+w
            // overwrites its own (snapshot) rows of G_i only after that
            std::vector<std::vector<cudaEvent_t>> rd(W, std::vector<cudaEvent_t>(len, nullptr));
            uint32_t kk = 0;
            struct Unhook {
                Stage* st;
                ~Unhook() { st->on_gather_done = nullptr, st->before_g_write = nullptr; }
            } unhook{this};
            if (merged_g && W > 1) {
                on_gather_done = [&](uint32_t i) { rd[kk % W][i] = record_event(); };
                before_g_write = [&](uint32_t i) {
                    for (uint32_t w = 1; w < uint32_t(W) && w <= kk; ++w)
                        if (cudaEvent_t e = rd[(kk - w) % W][i]) GP_CUDA(cudaStreamWaitEvent(cs, e, 0));
                };
            }
            wave_fork(W);
            uint64_t done = 0;
            for (; kk < K; ++kk) {
                const uint32_t k = ord[kk];
                const uint32_t r0 = row_begin(k), r1 = row_end(k);
                done |= 1ull << k;  // "processed" includes the current chunk (:789)
                cs = wave_stream(kk, W, main);
                auto& mine = ev[kk % W];
                if (!first) traced_recv(k, [&]() { recv_fwd(k); });
                cudaEvent_t c0 = trace_mark();
                if (!first && L[0].agg) {
                    if (before_g_write) before_g_write(0);
                    remask(0, in_cur, r0, r1, drop_key(t, L[0].l, L[0].din));
                }
                if (W > 1) mine[0] = record_event();
                for (uint32_t i = 0; i < len; ++i) {
                    if (G > 1 && L[i].agg) halo_fwd(i, k, k + 1, t);  // exchange_rows (:792-794)
                    if (L[i].agg)  // G_i rows of the W-1 previous chunks (other streams)
                        for (uint32_t w = 1; w < uint32_t(W) && w <= kk; ++w)
                            GP_CUDA(cudaStreamWaitEvent(cs, ev[(kk - w) % W][i], 0));
                    if (kk == 0) wait_remask(i);  // chunk 0 reads G_i (later chunks follow it)
                    wait_remask(i + 1);           // the epilogue writes this chunk's rows of G_{i+1}
                    forward_layer(i, r0, r1, t, done);
                    if (W > 1) mine[i + 1] = record_event();
                }
                trace_add(GP_TRACE_COMPUTE, int32_t(k), c0, trace_mark());
                if (!last) traced_send(k, [&]() { send_fwd(k); });
            }
            wave_join(W, main);
            for (uint32_t i = 0; i < len; ++i) wait_remask(i);
        } else {
            if (!first)
                for (uint32_t kk = 0; kk < K; ++kk) traced_recv(ord[kk], [&]() { recv_fwd(ord[kk]); });
            cudaEvent_t c0 = trace_mark();
            if (!first && L[0].agg) remask(0, in_cur, own_begin(), own_end(), drop_key(t, L[0].l, L[0].din));
            for (uint32_t i = 0; i < len; ++i) {
                if (G > 1 && L[i].agg) halo_fwd(i, 0, K, t);  // exchange_rows_full (:806-808)
                forward_layer(i, own_begin(), own_end(), t, all_done);
            }
            trace_add(GP_TRACE_COMPUTE, -1, c0, trace_mark());  // whole partition (:811)
            if (!last)
                for (uint32_t kk = 0; kk < K; ++kk) traced_send(ord[kk], [&]() { send_fwd(ord[kk]); });
        }

        // lean layout: the next epoch's snapshot (snap := cur at t+1) is taken now, before
        // the backward overwrites h with dz
        if (lean && !sync && t % fix_alpha == 0) copy_snapshots(false);

        // ---- metrics (last stage) ---------------------------------------------------
        if (last) {
            XentParams p = xent_params(0, own_end() - own_begin());
            p.rows = id_rows;
            launch(GP_K_XENT, double(own_end() - own_begin()) * L[len - 1].dout * 4.0, 0, 0,
                   [&]() { k_xent_stats<<<xent_blocks, kBlock, 0, cs>>>(p); });
            launch(GP_K_XENT, 0, 0, 0, [&]() {
                k_xent_fold<<<1, 32, 0, cs>>>(part_loss, part_correct, xent_blocks, red_loss, red_correct);
            });
            if (needs_h0)
                zero_words(reinterpret_cast<uint32_t*>(dh0 + size_t(own_begin()) * pad8(H)),
                           size_t(own_end() - own_begin()) * pad8(H));
        }

        // ---- backward ---------------------------------------------------------------
        if (!sync) build_bwd_csr(ord);
        if (!sync) {
            // Wavefront over W streams (SURVEY §8(a')9): chunk j+1 of the backward order
            // runs layer i+1 while chunk j runs layer i. Legal because a chunk only
            // gathers from chunks already done (the others are filtered out), so the only
            // cross-chunk dependency is "layer i of chunk j+1 reads bg_{i+1} of chunk j",
            // one event per (chunk, layer).
            const int W = wave_width();
            cudaStream_t main = cs;
            struct Restore {
                cudaStream_t& ref;
                cudaStream_t v;
                ~Restore() { ref = v; }
            } restore{cs, main};
            // ev[j % W][i]: bg_i rows of the j-th chunk (backward order) are written
            std::vector<std::vector<cudaEvent_t>> ev(W, std::vector<cudaEvent_t>(len + 1, nullptr));
            wave_fork(W);
            uint64_t done = 0;
            uint32_t j = 0;
            for (uint32_t kk = K; kk-- > 0; ++j) {
                const uint32_t k = ord[kk];
                const uint32_t r0 = row_begin(k), r1 = row_end(k);
                done |= 1ull << k;
                cs = wave_stream(j, W, main);
                auto& mine = ev[j % W];
                auto wait_prev = [&](uint32_t i) {
                    for (uint32_t w = 1; w < uint32_t(W) && w <= j; ++w)
                        GP_CUDA(cudaStreamWaitEvent(cs, ev[(j - w) % W][i], 0));
                };
                if (!last) traced_recv(k, [&]() { recv_bwd(k); });
                cudaEvent_t c0 = trace_mark();
                if (last) {
                    XentParams p = xent_params(r0, r1);
                    launch(GP_K_XENT, double(r1 - r0) * L[len - 1].dout * 8.0, 0, 0,
                           [&]() { k_xent_grad<<<row_grid(r1 - r0, (const void*)k_xent_grad, 0), kBlock, 0, cs>>>(p); });
                }
                for (uint32_t i = len; i-- > 0;) {
                    if (G > 1 && i + 1 < len && L[i + 1].agg) halo_bwd(i + 1, k, k + 1);  // (:838-844)
                    if (i + 1 < len && L[i + 1].agg) wait_prev(i + 1);
                    backward_layer(i, r0, r1, t, done);
                    if (W > 1) mine[i] = record_event();
                }
                if (G > 1 && L[0].agg) halo_bwd(0, k, k + 1);
                if (!first) {
                    if (L[0].agg) wait_prev(0);
                    backward_dhin(r0, r1, t, done);
                }
                trace_add(GP_TRACE_COMPUTE, int32_t(k), c0, trace_mark());
                if (!first) traced_send(k, [&]() { send_bwd(k); });
            }
            wave_join(W, main);
        } else {
            const uint64_t done = K == 64 ? ~0ull : ((1ull << K) - 1);
            const uint32_t ob = own_begin(), oe = own_end();
            if (!last)
                for (uint32_t kk = K; kk-- > 0;) traced_recv(ord[kk], [&]() { recv_bwd(ord[kk]); });
            cudaEvent_t c0 = trace_mark();
            if (last) {
                XentParams p = xent_params(ob, oe);
                launch(GP_K_XENT, double(oe - ob) * L[len - 1].dout * 8.0, 0, 0,
                       [&]() { k_xent_grad<<<row_grid(oe - ob, (const void*)k_xent_grad, 0), kBlock, 0, cs>>>(p); });
            }
            for (uint32_t i = len; i-- > 0;) {
                if (G > 1 && i + 1 < len && L[i + 1].agg) halo_bwd(i + 1, 0, K);
                backward_layer(i, ob, oe, t, done);
            }
            if (G > 1 && L[0].agg) halo_bwd(0, 0, K);
            if (!first) backward_dhin(ob, oe, t, done);
            trace_add(GP_TRACE_COMPUTE, -1, c0, trace_mark());  // whole partition (:867)
            if (!first)
                for (uint32_t kk = K; kk-- > 0;) traced_send(ord[kk], [&]() { send_bwd(ord[kk]); });
        }

        bwd_csr_ready = false;
        if (lean && hist && t % fix_alpha == 0) copy_snapshots(true);
        {
            cudaEvent_t c0 = trace_mark();
            param_step();
            trace_add(GP_TRACE_COMPUTE, -1, c0, trace_mark());  // epoch-close parameter step
        }
        GP_CUDA(cudaEventRecord(ev_end, cs));
        const double enqueue_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h_start).count();
        if (tr.ipc_up.linked() || tr.ipc_down.linked() || tr.ipcg.linked) {
            sync_watchdog(cs, 600.0);
            for (cudaStream_t st : {tr.ipc_up.stream, tr.ipc_down.stream, tr.ipc_up.rstream, tr.ipc_down.rstream})
                if (st) sync_watchdog(st, 600.0);
        }
        GP_CUDA(cudaStreamSynchronize(cs));
        if (tr.up_stream) GP_CUDA(cudaStreamSynchronize(tr.up_stream));
        if (tr.down_stream) GP_CUDA(cudaStreamSynchronize(tr.down_stream));
        last_epoch = t;

        gp_epoch_stats st{};
        st.epoch = t;
        if (last) {
            st.has_quality = 1;
            GP_CUDA(cudaMemcpy(&st.loss_sum, red_loss, 8, cudaMemcpyDeviceToHost));
            unsigned long long c[3];
            GP_CUDA(cudaMemcpy(c, red_correct, 24, cudaMemcpyDeviceToHost));
            for (int i = 0; i < 3; ++i) st.correct[i] = c[i];
        }
        for (int i = 0; i < 6; ++i) {
            st.bytes_sent[i] = bytes_sent[i];
            st.msgs_sent[i] = msgs_sent[i];
        }
        GP_CUDA(cudaEventElapsedTime(&st.epoch_ms, ev_start, ev_end));
        if (host_timing)  // host-side enqueue time of the epoch next to its device time
            std::fprintf(stderr, "[gp epoch] stage %u t=%u enqueue %.1f ms device %.1f ms launches %llu\n", s, t,
                         enqueue_ms, double(st.epoch_ms), (unsigned long long)launches);
        st.kernel_launches = launches;
        float busy = 0.f;
        std::vector<std::pair<float, float>> iv[GP_K_NUM];  // launch intervals since ev_start
        for (auto& tm : timed) {
            float ms = 0.f, t0 = 0.f;
            GP_CUDA(cudaEventElapsedTime(&ms, tm.a, tm.b));
            GP_CUDA(cudaEventElapsedTime(&t0, ev_start, tm.a));
            iv[tm.cls].emplace_back(t0, t0 + ms);
            busy += ms;
            prof.ms[tm.cls] += ms;
            prof.launches[tm.cls] += 1;
            prof.alg_bytes[tm.cls] += tm.bytes;
            prof.flops[tm.cls] += tm.flops;
            prof.gather_bytes[tm.cls] += tm.gather;
            ev_free.push_back(tm.a);
            ev_free.push_back(tm.b);
        }
        timed.clear();
        for (int c = 0; c < GP_K_NUM; ++c) {
            auto& v = iv[c];
            std::sort(v.begin(), v.end());
            double span = 0, lo = 0, hi = -1;
            for (auto& x : v) {
                if (x.first > hi) {
                    if (hi > lo) span += hi - lo;
                    lo = x.first;
                    hi = x.second;
                } else {
                    hi = std::max<double>(hi, x.second);
                }
            }
            if (hi > lo) span += hi - lo;
            prof.span_ms[c] += span;
        }
        st.busy_ms = busy;
        trace_resolve();
        if (out) *out = st;
    }

    // ---- historical-embedding state (resume) -------------------------------------
    // The rows the next epoch reads stale values from: h_snap / in_snap / dagg_snap
    // after epoch last_epoch's snapshot rule (engines_impl.hpp:671-679). Lean layout:
    // the snapshot buffer itself (copies are taken at the end of the epoch). Swap
    // layout: the current buffer when the next epoch refreshes, else the snapshot.
    struct HistBuf {
        float *next, *snap, *cur;
        uint32_t width, stride;
    };
    HistBuf history(uint32_t which, uint32_t i) {
        if (sync) throw Error(GP_EINVAL, "synchronous mode keeps no historical embeddings");
        const uint32_t fix_alpha = std::max<uint32_t>(1, cfg.fix_alpha);
        const bool refresh_next = last_epoch % fix_alpha == 0;
        HistBuf b{};
        if (which == GP_BUF_HIST_IN) {
            b = {nullptr, in_snap, in_cur, in0, sin0};
        } else {
            if (i >= len) throw Error(GP_EINVAL, "local layer out of range");
            auto& d = L[i];
            if (which == GP_BUF_HIST_H) b = {nullptr, d.hs, d.h, d.dout, d.sout};
            else b = {nullptr, d.bgs, d.bg, d.kw, d.skw};  // SageConv: both (gapped) halves
        }
        if (!b.snap) throw Error(GP_EINVAL, "no historical rows for this buffer on this stage");
        b.next = lean || !refresh_next ? b.snap : b.cur;
        return b;
    }

    // Restore the historical rows (original vertex order, N x width) before resuming
    // at epoch last_epoch + 1 = t: the next run_epoch reads them as the snapshot.
    void upload_history(uint32_t which, uint32_t i, const float* in, uint64_t count, uint32_t resume_epoch) {
        GP_CUDA(cudaSetDevice(device));
        if (!graph_ready) throw Error(GP_EINVAL, "graph not uploaded");
        if (which != GP_BUF_HIST_H && which != GP_BUF_HIST_IN && which != GP_BUF_HIST_DAGG)
            throw Error(GP_EINVAL, "gp_upload_history: not a history buffer");
        last_epoch = resume_epoch;
        const HistBuf hb = history(which, i);
        if (count != uint64_t(n) * hb.width) throw Error(GP_EINVAL, "count != N * width");
        std::vector<float> tmp(size_t(n) * hb.stride, 0.f);
        for (uint32_t r = 0; r < n; ++r) std::memcpy(&tmp[size_t(r) * hb.stride], in + size_t(inv[r]) * hb.width, size_t(hb.width) * 4);
        // swap layout: both halves, so whichever the next epoch's rule picks holds them
        for (float* dst : {hb.snap, lean ? nullptr : hb.cur})
            if (dst) GP_CUDA(cudaMemcpy(dst, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice));
        settle_uploads();
        state_restored = true;
    }

    void download(uint32_t which, uint32_t i, float* out, uint64_t count) {
        GP_CUDA(cudaSetDevice(device));
        GP_CUDA(cudaStreamSynchronize(cs));
        if (!graph_ready) throw Error(GP_EINVAL, "graph not uploaded");
        const float* src = nullptr;
        uint32_t width = 0, stride = 0, gap = 0;
        auto need_layer = [&]() -> LayerDev& {
            if (i >= len) throw Error(GP_EINVAL, "local layer out of range");
            return L[i];
        };
        switch (which) {
            case GP_BUF_H: {
                auto& d = need_layer();
                if (lean && last_epoch) throw Error(GP_EINVAL, "lean stash layout: h holds dz after the backward (GP_LEAN=0 keeps activations)");
                src = d.h; width = d.dout; stride = d.sout; break;
            }
            case GP_BUF_PRE: { auto& d = need_layer(); src = d.pre; width = d.din; stride = d.skw; gap = d.sgap; break; }
            case GP_BUF_DZ: { auto& d = need_layer(); src = d.dz; width = d.dout; stride = d.sout; break; }
            case GP_BUF_DAGG: { auto& d = need_layer(); src = d.bg; width = d.din; stride = d.skw; gap = d.sgap; break; }
            case GP_BUF_HSNAP: { auto& d = need_layer(); src = d.hs; width = d.dout; stride = d.sout; break; }
            case GP_BUF_GATHER: {
                auto& d = need_layer();
                if (lean && last_epoch && d.bg == d.G) throw Error(GP_EINVAL, "lean stash layout: the gather table holds dagg after the backward (GP_LEAN=0)");
                src = d.G; width = d.din; stride = d.sin; break;
            }
            case GP_BUF_DH0: src = dh0; width = H; stride = pad8(H); break;
            case GP_BUF_IN: src = in_cur; width = in0; stride = sin0; break;
            case GP_BUF_DH_IN: src = dh_in; width = in0; stride = sin0; break;
            case GP_BUF_HIST_H:
            case GP_BUF_HIST_IN:
            case GP_BUF_HIST_DAGG: {
                const HistBuf hb = history(which, i);
                src = hb.next;
                width = hb.width;
                stride = hb.stride;
                break;
            }
            default: throw Error(GP_EINVAL, "unknown buffer");
        }
        if (!src) throw Error(GP_EINVAL, "buffer not allocated on this stage");
        // SageConv pre / dagg: k_in = 2 din columns, halves at 0 and gap
        const uint32_t ow = gap ? 2 * width : width;
        if (count != uint64_t(n) * ow) throw Error(GP_EINVAL, "count != N * width");
        std::vector<float> tmp(size_t(n) * stride, 0.f);
        if (own_only(src))  // a hybrid worker's owner-row buffer: other rows read as zero
            GP_CUDA(cudaMemcpy(tmp.data() + size_t(own_begin()) * stride, src + size_t(own_begin()) * stride,
                               size_t(own_end() - own_begin()) * stride * 4, cudaMemcpyDeviceToHost));
        else
            GP_CUDA(cudaMemcpy(tmp.data(), src, tmp.size() * 4, cudaMemcpyDeviceToHost));
        for (uint32_t r = 0; r < n; ++r) {
            std::memcpy(out + size_t(inv[r]) * ow, &tmp[size_t(r) * stride], size_t(width) * 4);
            if (gap) std::memcpy(out + size_t(inv[r]) * ow + width, &tmp[size_t(r) * stride + gap], size_t(width) * 4);
        }
    }
};

gp_status fail(Stage* st, const std::exception& e) {
    gp_status code = GP_ERUNTIME;
    if (auto* ge = dynamic_cast<const Error*>(&e)) code = ge->code;
    else if (dynamic_cast<const std::invalid_argument*>(&e)) code = GP_EINVAL;
    if (st) st->err = e.what();
    g_tls_error = e.what();
    return code;
}

template <typename F>
gp_status guard(Stage* st, F&& f) {
    try {
        f();
        return GP_OK;
    } catch (const std::exception& e) {
        return fail(st, e);
    }
}

}  // namespace
}  // namespace gp

struct gp_ctx {
    gp::Stage st;
};

extern "C" {

uint32_t gp_abi_version(void) { return GP_ABI_VERSION; }

gp_status gp_device_count(int* out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    if (out) *out = n;
    return GP_OK;
}

gp_status gp_create(const gp_stage_config* cfg, gp_ctx** out) {
    if (!cfg || !out) {
        gp::g_tls_error = "gp_create: null argument";
        return GP_EINVAL;
    }
    *out = nullptr;
    gp_ctx* c = new gp_ctx();
    const gp_status s = gp::guard(&c->st, [&]() { c->st.init(*cfg); });
    if (s != GP_OK) {
        gp::g_tls_error = c->st.err;
        delete c;
        return s;
    }
    *out = c;
    return GP_OK;
}

void gp_destroy(gp_ctx* ctx) { delete ctx; }

const char* gp_last_error(const gp_ctx* ctx) {
    if (ctx && !ctx->st.err.empty()) return ctx->st.err.c_str();
    return gp::g_tls_error.c_str();
}

gp_status gp_upload_graph(gp_ctx* ctx, const uint64_t* offsets, const uint32_t* cols, const float* vals,
                          uint64_t nnz, const uint32_t* chunk_of) {
    return gp::guard(&ctx->st, [&]() { ctx->st.upload_graph(offsets, cols, vals, nnz, chunk_of); });
}

gp_status gp_upload_graph_raw(gp_ctx* ctx, const uint64_t* offsets, const uint32_t* neighbors,
                              uint64_t num_neighbors, int self_loops, const uint32_t* chunk_of) {
    return gp::guard(&ctx->st, [&]() {
        ctx->st.upload_graph_raw(offsets, neighbors, num_neighbors, self_loops != 0, chunk_of);
    });
}

gp_status gp_upload_partition(gp_ctx* ctx, const uint32_t* part_of) {
    return gp::guard(&ctx->st, [&]() { ctx->st.upload_partition(part_of); });
}

gp_status gp_link_group(gp_ctx** members, uint32_t G) {
    if (!members || G == 0) {
        gp::g_tls_error = "gp_link_group: no members";
        return GP_EINVAL;
    }
    return gp::guard(&members[0]->st, [&]() {
        auto link = std::make_shared<gp::GroupLink>(G);
        for (uint32_t r = 0; r < G; ++r) {
            auto& st = members[r]->st;
            if (st.G != G || st.grank != r) throw gp::Error(GP_EINVAL, "gp_link_group: member order must be rank order");
            if (st.s != members[0]->st.s) throw gp::Error(GP_EINVAL, "gp_link_group: members must share a stage");
            link->members.push_back(&st);
        }
        for (uint32_t r = 0; r < G; ++r) members[r]->st.tr.group = link;
    });
}

gp_status gp_share_graph(gp_ctx* ctx, const gp_ctx* owner) {
    return gp::guard(&ctx->st, [&]() { ctx->st.share_graph(owner->st); });
}

gp_status gp_upload_features(gp_ctx* ctx, const float* x, uint32_t F) {
    return gp::guard(&ctx->st, [&]() { ctx->st.upload_features(x, F); });
}

gp_status gp_upload_labels(gp_ctx* ctx, const uint32_t* labels, const uint8_t* split) {
    return gp::guard(&ctx->st, [&]() { ctx->st.upload_labels(labels, split); });
}

gp_status gp_set_layer_params(gp_ctx* ctx, uint32_t layer, const float* W, const float* b) {
    return gp::guard(&ctx->st, [&]() { ctx->st.set_params(layer, W, b); });
}

gp_status gp_get_layer_params(gp_ctx* ctx, uint32_t layer, float* W, float* b) {
    return gp::guard(&ctx->st, [&]() { ctx->st.get_params(layer, W, b); });
}

gp_status gp_get_layer_grads(gp_ctx* ctx, uint32_t layer, float* W, float* b) {
    return gp::guard(&ctx->st, [&]() { ctx->st.get_grads(layer, W, b); });
}

gp_status gp_get_optimizer_state(gp_ctx* ctx, uint32_t layer, float* mW, float* vW, float* mb, float* vb,
                                 uint64_t* step) {
    return gp::guard(&ctx->st, [&]() { ctx->st.get_opt_state(layer, mW, vW, mb, vb, step); });
}

gp_status gp_set_optimizer_state(gp_ctx* ctx, uint32_t layer, const float* mW, const float* vW, const float* mb,
                                 const float* vb, uint64_t step) {
    return gp::guard(&ctx->st, [&]() { ctx->st.set_opt_state(layer, mW, vW, mb, vb, step); });
}

gp_status gp_link_local(gp_ctx* up, gp_ctx* down) {
    return gp::guard(&down->st, [&]() {
        if (up->st.s + 1 != down->st.s) throw gp::Error(GP_EINVAL, "gp_link_local: stages not adjacent");
        if (up->st.n != down->st.n || up->st.K != down->st.K)
            throw gp::Error(GP_EINVAL, "gp_link_local: N/K mismatch");
        auto link = std::make_shared<gp::LocalLink>();
        up->st.tr.down_local = link;
        down->st.tr.up_local = link;
        if (up->st.device != down->st.device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, down->st.device, up->st.device);
            if (can) {
                cudaSetDevice(down->st.device);
                cudaDeviceEnablePeerAccess(up->st.device, 0);
                cudaGetLastError();
                cudaSetDevice(up->st.device);
                cudaDeviceEnablePeerAccess(down->st.device, 0);
                cudaGetLastError();
            }
        }
    });
}

gp_status gp_nccl_unique_id(uint8_t out[128]) {
    if (!gp::g_nccl.load()) {
        gp::g_tls_error = "libnccl.so.2 not loadable";
        return GP_ECUDA;
    }
    const int r = gp::g_nccl.get_unique_id(out);
    if (r != 0) {
        gp::g_tls_error = "ncclGetUniqueId failed";
        return GP_ECUDA;
    }
    return GP_OK;
}

gp_status gp_link_nccl(gp_ctx* ctx, const uint8_t* up_id, const uint8_t* down_id) {
    return gp::guard(&ctx->st, [&]() {
        auto& st = ctx->st;
        if (!gp::g_nccl.load()) throw gp::Error(GP_ECUDA, "libnccl.so.2 not loadable");
        GP_CUDA(cudaSetDevice(st.device));
        if (st.S < 2) throw gp::Error(GP_EINVAL, "gp_link_nccl: a single-stage pipeline has no boundary");
        if (up_id && !st.first) {
            st.tr.up_comm = gp::nccl_comm_init(up_id, 1, "ncclCommInitRankConfig(up)");
            GP_CUDA(cudaStreamCreateWithFlags(&st.tr.up_stream, cudaStreamNonBlocking));
        }
        if (down_id && !st.last) {
            st.tr.down_comm = gp::nccl_comm_init(down_id, 0, "ncclCommInitRankConfig(down)");
            GP_CUDA(cudaStreamCreateWithFlags(&st.tr.down_stream, cudaStreamNonBlocking));
        }
    });
}

gp_status gp_ipc_export(gp_ctx* ctx, uint8_t* up_blob, uint8_t* down_blob) {
    return gp::guard(&ctx->st, [&]() { ctx->st.ipc_export(up_blob, down_blob); });
}

gp_status gp_link_ipc(gp_ctx* ctx, const uint8_t* up_peer_blob, const uint8_t* down_peer_blob) {
    return gp::guard(&ctx->st, [&]() { ctx->st.ipc_link(up_peer_blob, down_peer_blob); });
}

gp_status gp_group_export(gp_ctx* ctx, uint8_t* blob, uint64_t capacity, uint64_t* length) {
    return gp::guard(&ctx->st, [&]() {
        const size_t need = ctx->st.group_export(blob, capacity);
        if (length) *length = need;
    });
}

gp_status gp_link_group_ipc(gp_ctx* ctx, const uint8_t* const* blobs, const uint64_t* lengths) {
    return gp::guard(&ctx->st, [&]() { ctx->st.group_link_ipc(blobs, lengths); });
}

void gp_abort(gp_ctx* ctx) {
    if (!ctx) return;
    auto& st = ctx->st;
    st.aborted = true;
    if (st.tr.group)
        for (auto& q : st.tr.group->q) {
            std::lock_guard<std::mutex> lk(q.mu);
            q.aborted = true;
            q.cv.notify_all();
        }
    for (auto* l : {st.tr.up_local.get(), st.tr.down_local.get()}) {
        if (!l) continue;
        for (auto* q : {&l->fwd, &l->bwd}) {
            std::lock_guard<std::mutex> lk(q->mu);
            q->aborted = true;
            q->cv.notify_all();
        }
    }
}

gp_status gp_run_epoch(gp_ctx* ctx, uint32_t t, const uint32_t* order, gp_epoch_stats* out) {
    return gp::guard(&ctx->st, [&]() { ctx->st.run_epoch(t, order, out); });
}

gp_status gp_download(gp_ctx* ctx, uint32_t which, uint32_t local_layer, float* out, uint64_t count) {
    return gp::guard(&ctx->st, [&]() { ctx->st.download(which, local_layer, out, count); });
}

gp_status gp_stage_footprint(const gp_stage_config* cfg, uint64_t nnz_norm, uint32_t num_features, uint64_t* bytes) {
    if (!cfg || !bytes) return GP_EINVAL;
    gp::Stage st;
    return gp::guard(nullptr, [&]() { *bytes = st.plan_bytes(*cfg, nnz_norm, num_features); });
}

gp_status gp_upload_history(gp_ctx* ctx, uint32_t which, uint32_t local_layer, const float* rows, uint64_t count,
                            uint32_t resume_epoch) {
    if (!ctx || !rows) return GP_EINVAL;
    return gp::guard(&ctx->st, [&]() { ctx->st.upload_history(which, local_layer, rows, count, resume_epoch); });
}

gp_status gp_set_live_timing(gp_ctx* ctx, int kernel_class) {
    if (!ctx || kernel_class < -1 || kernel_class > GP_K_NUM) return GP_EINVAL;
    ctx->st.live_cls = kernel_class;
    return GP_OK;
}

gp_status gp_set_profiling(gp_ctx* ctx, int enable) {
    ctx->st.profiling = enable != 0;
    return GP_OK;
}

gp_status gp_set_trace(gp_ctx* ctx, int enable) {
    ctx->st.tracing = enable != 0;
    return GP_OK;
}

gp_status gp_get_trace(gp_ctx* ctx, gp_trace_event* out, uint64_t cap, uint64_t* count) {
    const auto& v = ctx->st.trace_done;
    if (count) *count = v.size();
    if (out) std::copy_n(v.begin(), std::min<uint64_t>(cap, v.size()), out);
    return GP_OK;
}

gp_status gp_clear_trace(gp_ctx* ctx) {
    ctx->st.trace_done.clear();
    return GP_OK;
}

gp_status gp_get_profile(gp_ctx* ctx, gp_profile* out) {
    if (out) *out = ctx->st.prof;
    return GP_OK;
}

gp_status gp_reset_profile(gp_ctx* ctx) {
    ctx->st.prof = gp_profile{};
    return GP_OK;
}

gp_status gp_mark(gp_ctx* ctx, uint32_t slot) {
    return gp::guard(&ctx->st, [&]() {
        auto& st = ctx->st;
        if (slot >= 16) throw gp::Error(GP_EINVAL, "mark slot must be < 16");
        GP_CUDA(cudaSetDevice(st.device));
        if (!st.marks[slot]) GP_CUDA(cudaEventCreate(&st.marks[slot]));
        GP_CUDA(cudaEventRecord(st.marks[slot], st.cs));
    });
}

gp_status gp_elapsed(gp_ctx* ctx, uint32_t a, uint32_t b, float* ms) {
    return gp::guard(&ctx->st, [&]() {
        auto& st = ctx->st;
        if (a >= 16 || b >= 16 || !st.marks[a] || !st.marks[b]) throw gp::Error(GP_EINVAL, "unrecorded mark");
        GP_CUDA(cudaSetDevice(st.device));
        GP_CUDA(cudaEventSynchronize(st.marks[b]));
        GP_CUDA(cudaEventElapsedTime(ms, st.marks[a], st.marks[b]));
    });
}

gp_status gp_synchronize(gp_ctx* ctx) {
    return gp::guard(&ctx->st, [&]() {
        GP_CUDA(cudaSetDevice(ctx->st.device));
        GP_CUDA(cudaStreamSynchronize(ctx->st.cs));
    });
}

gp_status gp_device_bytes(gp_ctx* ctx, uint64_t* out) {
    if (out) *out = ctx->st.dev_bytes;
    return GP_OK;
}

}  // extern "C"

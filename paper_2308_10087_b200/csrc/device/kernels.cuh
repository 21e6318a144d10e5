// sm_100a kernels of the stage engine. Every kernel is a restatement of a
// reference per-row routine; arithmetic that the reference performs in a fixed
// scalar order (ascending neighbour, ascending inner index, mul then add) is
// performed in the same order with explicitly rounded IEEE operations, so the
// forward pass is bit-identical to the CPU reference for the same parameters.
//
// Layout: vertices are renumbered chunk-contiguously; every
// N x d activation is row-major with a row stride padded to a multiple of 8
// floats (32-byte sectors); the normalised adjacency is CSR with one packed
// 8-byte entry per non-zero: {col | chunk << 26, float weight}. One warp owns
// one row; lane l owns columns 4l..4l+3 (d <= 128), so every neighbour gather is
// one 16-byte load per lane and one contiguous sector run per warp.
#pragma once

#include "common.cuh"

namespace gp {

constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = kWarpsPerBlock * 32;
constexpr unsigned kFull = 0xffffffffu;

enum FwdKind { FWD_DENSE = 0, FWD_GCN = 1, FWD_GCN2 = 2, FWD_SAGE = 3 };
// PREV_AGG_ALL: PREV_AGG when every chunk is done (the last chunk of a backward pass,
// synchronous mode): no done filter, so no per-batch compaction.
enum PrevKind { PREV_TOP = 0, PREV_AGG = 1, PREV_AGG_HIST = 2, PREV_OWN = 3, PREV_SAGE = 4, PREV_SAGE_HIST = 5,
                PREV_AGG_ALL = 6 };
enum OutKind { OUT_LAYER = 0, OUT_DHIN = 1 };

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4_rw(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// ---------------------------------------------------------------------------
// CSR row gather: acc[c] = sum over the row's entries in ascending column order
// of w * src[col][c]  (kernel::spmv_row, nn.hpp:143-154, one mul and one add per
// term). FILTER skips entries whose chunk is not in `done` (backward_prev_row's
// nullptr getter, nn.hpp:249-250, engines_impl.hpp:771-778); HIST reads those
// from `src_snap` instead (historical-gradient ablation, :773-776).
// The 32 entries of a batch are loaded once, coalesced, and broadcast by
// shuffle; 8 gathers are kept in flight per lane.
// ---------------------------------------------------------------------------
// Streaming (evict-first) load of the CSR entries so they do not displace the
// gather table from L2; gathers use the read-only path with default policy.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint2 ld_edge(const uint2* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(evict_first_policy()));
    return r;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// Gather-table reads: kept in L2 (evict_last) — the table (N x d, ~97 MB at
// Reddit shape) is re-read ~deg times per row and must survive the streams.
__device__ __forceinline__ float4 ld_gather(const float* p, uint64_t pol) {
    float4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
        : "l"(p), "l"(pol));
    return r;
}
// Row-local streams (pre, h, dz, h0, ...): evict_first so they never displace
// the gather table.
__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 r;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(evict_first_policy()));
    return r;
}
__device__ __forceinline__ void st_stream(float* p, float4 v) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(evict_first_policy())
                 : "memory");
}

// Gathers of one batch are issued back to back, without branches or selects
// on the loaded values (a select after a load forces a scoreboard wait):
//  * padding entries past the end of a batch re-read the batch's first row with
//    weight 0; acc starts at +0 and a sum of products never becomes -0, so
//    acc + 0*x == acc bit-for-bit — padding is indistinguishable from skipping;
//  * lanes beyond the row width alias lane 0's address (no extra sectors); their
//    values are never stored.
template <int NB, bool HIST>
__device__ __forceinline__ void gather_batch(float4& acc, uint2 my, int t, int cnt, uint64_t pol, const float* lsrc,
                                             const float* lsnap, uint32_t stride, uint64_t done) {
    const uint32_t first = __shfl_sync(kFull, my.x, 0) & kColMask;
    float4 x[NB];
    float w[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int tt = (t + i) & 31;
        const uint32_t packed = __shfl_sync(kFull, my.x, tt);
        const float wv = __uint_as_float(__shfl_sync(kFull, my.y, tt));
        const bool valid = t + i < cnt;
        const float* s = lsrc;
        if (HIST && valid && !((done >> (packed >> kColBits)) & 1ull)) s = lsnap;
        w[i] = valid ? wv : 0.f;
        x[i] = ld_gather(s + size_t(valid ? (packed & kColMask) : first) * stride, pol);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        acc.x = mul_add(acc.x, w[i], x[i].x);
        acc.y = mul_add(acc.y, w[i], x[i].y);
        acc.z = mul_add(acc.z, w[i], x[i].z);
        acc.w = mul_add(acc.w, w[i], x[i].w);
    }
}

// FILTER (backward, zeroed historical gradients): entries whose chunk is not in
// `done` are dropped from each 32-entry batch by a warp ballot and a stable
// compaction (ascending order kept), so they cost neither loads nor FMAs.
template <bool FILTER, bool HIST>
__device__ __forceinline__ float4 gather_row(const uint64_t* __restrict__ rowptr,
                                             const uint2* __restrict__ edges, uint32_t v,
                                             const float* __restrict__ src,
                                             const float* __restrict__ src_snap, uint32_t stride,
                                             uint64_t done, int lane, bool active) {
    float4 acc = f4_zero();
    const uint64_t e0 = rowptr[v], e1 = rowptr[v + 1];
    const uint32_t loff = active ? 4u * lane : 0u;
    const float* lsrc = src + loff;
    const float* lsnap = HIST ? src_snap + loff : nullptr;
    const uint64_t pol = evict_last_policy();
    for (uint64_t base = e0; base < e1; base += 32) {
        int cnt = int(e1 - base < 32 ? e1 - base : 32);
        uint2 my = lane < cnt ? ld_edge(edges + base + lane) : make_uint2(0u, 0u);
        if (FILTER && !HIST) {
            const bool ok = lane < cnt && ((done >> (my.x >> kColBits)) & 1ull);
            const unsigned m = __ballot_sync(kFull, ok);
            cnt = __popc(m);
            if (cnt == 0) continue;
            const int from = lane < cnt ? int(__fns(m, 0, lane + 1)) : 0;
            my.x = __shfl_sync(kFull, my.x, from);
            my.y = __shfl_sync(kFull, my.y, from);
        }
        int t = 0;
        for (; t + 8 <= cnt; t += 8) gather_batch<8, HIST>(acc, my, t, cnt, pol, lsrc, lsnap, stride, done);
        if (cnt - t > 4)
            gather_batch<8, HIST>(acc, my, t, cnt, pol, lsrc, lsnap, stride, done);
        else if (cnt > t)
            gather_batch<4, HIST>(acc, my, t, cnt, pol, lsrc, lsnap, stride, done);
    }
    return acc;
}

__device__ __forceinline__ float4 drop4(const DropKey& m, uint32_t vo, uint32_t c0, uint32_t width,
                                        float4 x) {
    float4 r;
    r.x = c0 + 0 < width ? drop_apply(m, vo, c0 + 0, x.x) : 0.f;
    r.y = c0 + 1 < width ? drop_apply(m, vo, c0 + 1, x.y) : 0.f;
    r.z = c0 + 2 < width ? drop_apply(m, vo, c0 + 2, x.z) : 0.f;
    r.w = c0 + 3 < width ? drop_apply(m, vo, c0 + 3, x.w) : 0.f;
    return r;
}

// ---------------------------------------------------------------------------
// Masked gather source: dst[v] = DropMask::apply(src[v]) for rows [r0, r1)
// (the dropout the reference applies on every read of a layer input,
// nn.hpp:152, :167). Used once per epoch per layer over the snapshot rows and
// once per chunk over freshly received stage-input rows.
// ---------------------------------------------------------------------------
struct RemaskParams {
    uint32_t r0, r1, width;
    const float* src;
    uint32_t sstride;
    float* dst;
    uint32_t dstride;
    const uint32_t* orig;
    DropKey mask;
};

// Rows up to 128 wide: each warp handles kRemaskRows rows per step with all their loads
// issued before the stores (4.35 vs 4.5-4.6 ms per Reddit epoch; the per-element dropout
// hash, not the copy, bounds this kernel).
constexpr uint32_t kRemaskRows = 4;
__global__ void __launch_bounds__(kBlock) k_remask(RemaskParams p) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    if (p.width <= 128) {
        const uint32_t c0 = 4 * lane;
        const bool act = c0 < p.width;
        for (uint32_t v0 = p.r0 + (blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5)) * kRemaskRows; v0 < p.r1;
             v0 += nw * kRemaskRows) {
            float4 x[kRemaskRows];
            uint32_t vo[kRemaskRows];
#pragma unroll
            for (uint32_t q = 0; q < kRemaskRows; ++q) {
                const uint32_t v = v0 + q;
                const bool in = act && v < p.r1;
                vo[q] = v < p.r1 ? p.orig[v] : 0u;
                x[q] = in ? ld4_rw(p.src + size_t(v) * p.sstride + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (uint32_t q = 0; q < kRemaskRows; ++q)
                if (act && v0 + q < p.r1)
                    st4(p.dst + size_t(v0 + q) * p.dstride + c0, drop4(p.mask, vo[q], c0, p.width, x[q]));
        }
        return;
    }
    for (uint32_t v = p.r0 + blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); v < p.r1; v += nw) {
        const uint32_t vo = p.orig[v];
        for (uint32_t c0 = 4 * lane; c0 < p.width; c0 += 128) {
            const float4 x = ld4_rw(p.src + size_t(v) * p.sstride + c0);
            st4(p.dst + size_t(v) * p.dstride + c0, drop4(p.mask, vo, c0, p.width, x));
        }
    }
}

// ---------------------------------------------------------------------------
// Fused forward of one layer over the rows of one chunk (kernel::forward_row,
// nn.hpp:159-197), d_in, d_out <= 128:
//   Dense   : pre = drop(x_v)
//   GcnConv : pre = sum_u w_vu * G[u]          (G = dropped layer input)
//   Gcn2Conv: pre = (1-a) * sum_u w_vu G[u] + a * h0[v]
//   out = b + pre . W   (ascending inner index, exact-zero skip, matrix.hpp:63-74)
//   Gcn2Conv: out = (1-beta) pre + beta out;  ReLU
// and, in the epilogue, the next layer's gather source gnext[v] = drop'(out).
// W is staged in shared memory (<= 64 KB).
// ---------------------------------------------------------------------------
struct FwdParams {
    uint32_t r0, r1;
    uint32_t* ticket;  // zeroed work counter (row pairs handed out)
    const uint64_t* rowptr;
    const uint2* edges;
    const float* gsrc;   // gather table rows of done chunks (cur)
    const float* gsnap;  // gather table rows of not-done chunks (snapshot); may equal gsrc
    uint64_t done;       // chunks processed so far this epoch, including the current one
    uint32_t gstride;
    uint32_t zrow;
    const float* xsrc;
    uint32_t xstride;
    DropKey in_mask;
    const uint32_t* orig;
    const float* h0;
    uint32_t h0stride;
    float alpha, oma, beta, omb;
    const float* W;
    const float* bias;
    uint32_t din, dout;
    uint32_t relu;
    float* pre;
    uint32_t prestride;
    float* out;
    uint32_t outstride;
    float* gnext;
    uint32_t gnstride;
    DropKey next_mask;
    // SageConv (FWD_SAGE): mean adjacency (graph neighbours, weight 1/deg(v)) and the
    // column of pre where the aggregated half starts (pad8(din); own half at 0)
    const uint64_t* rowptr_m;
    const uint2* edges_m;
    uint32_t sgap;
};

// GcnConv aggregation for d_in > 128 (column blocks of 128): pre = A_hat . G.
struct SpmmParams {
    uint32_t r0, r1, width, zrow;
    const uint64_t* rowptr;
    const uint2* edges;
    const float* gsrc;
    uint32_t gstride;
    float* pre;
    uint32_t prestride;
};

__global__ void __launch_bounds__(kBlock) k_spmm_pre(SpmmParams p) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    for (uint32_t v = p.r0 + blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); v < p.r1; v += nw)
        for (uint32_t c0 = 0; c0 < p.width; c0 += 128) {
            const bool act = c0 + 4 * lane < p.width;
            const float4 z = gather_row<false, false>(p.rowptr, p.edges, v, p.gsrc + c0, nullptr,
                                                      p.gstride, 0ull, lane, act);
            if (act) st4(p.pre + size_t(v) * p.prestride + c0 + 4 * lane, z);
        }
}

// ---------------------------------------------------------------------------
// Dense transform for d_in > 128 (GCNII's Dense F->H input layer): out = b + pre.W
// with the same ascending-k, mul-then-add, zero-skip order as dense_rows
// (matrix.hpp:63-74), followed by the bias/ReLU/next-mask epilogue.
// CTA tile: 64 rows x 128 output columns; thread: 8 rows x 4 columns.
// ---------------------------------------------------------------------------
struct GemmParams {
    uint32_t r0, r1;
    const float* A;
    uint32_t astride;
    const float* W;
    const float* bias;
    uint32_t din, dout;
    uint32_t relu;
    float* out;
    uint32_t outstride;
    float* gnext;
    uint32_t gnstride;
    DropKey next_mask;
    const uint32_t* orig;
};

__global__ void __launch_bounds__(kBlock) k_dense_gemm(GemmParams p) {
    __shared__ float As[64][33];
    __shared__ float4 Bs[32][32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const uint32_t row0 = p.r0 + blockIdx.x * 64;
    const bool col_act = uint32_t(4 * tx) < p.dout;
    float4 acc[8];
    const float4 b0 = make_float4(
        (p.bias && 4 * tx + 0 < p.dout) ? p.bias[4 * tx + 0] : 0.f,
        (p.bias && 4 * tx + 1 < p.dout) ? p.bias[4 * tx + 1] : 0.f,
        (p.bias && 4 * tx + 2 < p.dout) ? p.bias[4 * tx + 2] : 0.f,
        (p.bias && 4 * tx + 3 < p.dout) ? p.bias[4 * tx + 3] : 0.f);
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = b0;
    for (uint32_t k0 = 0; k0 < p.din; k0 += 32) {
        for (int idx = threadIdx.x; idx < 64 * 32; idx += kBlock) {
            const int r = idx / 32, kk = idx % 32;
            const uint32_t row = row0 + r, k = k0 + kk;
            As[r][kk] = (row < p.r1 && k < p.din) ? p.A[size_t(row) * p.astride + k] : 0.f;
        }
        for (int idx = threadIdx.x; idx < 32 * 32; idx += kBlock) {
            const int kk = idx / 32, c4 = idx % 32;
            const uint32_t k = k0 + kk;
            float4 w = f4_zero();
            if (k < p.din) {
                const float* wr = p.W + size_t(k) * p.dout;
                const uint32_t c = 4 * c4;
                w.x = c + 0 < p.dout ? wr[c + 0] : 0.f;
                w.y = c + 1 < p.dout ? wr[c + 1] : 0.f;
                w.z = c + 2 < p.dout ? wr[c + 2] : 0.f;
                w.w = c + 3 < p.dout ? wr[c + 3] : 0.f;
            }
            Bs[kk][c4] = w;
        }
        __syncthreads();
        const uint32_t kmax = p.din - k0 < 32 ? p.din - k0 : 32;
        for (uint32_t kk = 0; kk < kmax; ++kk) {
            const float4 b = Bs[kk][tx];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float a = As[ty * 8 + r][kk];
                if (a != 0.f) {
                    acc[r].x = mul_add(acc[r].x, a, b.x);
                    acc[r].y = mul_add(acc[r].y, a, b.y);
                    acc[r].z = mul_add(acc[r].z, a, b.z);
                    acc[r].w = mul_add(acc[r].w, a, b.w);
                }
            }
        }
        __syncthreads();
    }
    if (!col_act) return;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t row = row0 + ty * 8 + r;
        if (row >= p.r1) continue;
        float4 o = acc[r];
        if (p.relu) {
            if (o.x < 0.f) o.x = 0.f;
            if (o.y < 0.f) o.y = 0.f;
            if (o.z < 0.f) o.z = 0.f;
            if (o.w < 0.f) o.w = 0.f;
        }
        if (4 * tx + 3 >= p.dout) {  // keep padding columns zero
            if (4 * tx + 0 >= p.dout) o.x = 0.f;
            if (4 * tx + 1 >= p.dout) o.y = 0.f;
            if (4 * tx + 2 >= p.dout) o.z = 0.f;
            if (4 * tx + 3 >= p.dout) o.w = 0.f;
        }
        st4(p.out + size_t(row) * p.outstride + 4 * tx, o);
        if (p.gnext)
            st4(p.gnext + size_t(row) * p.gnstride + 4 * tx,
                drop4(p.next_mask, p.orig[row], 4 * tx, p.dout, o));
    }
}

// ---------------------------------------------------------------------------
// Fused backward step for the rows of one chunk:
//   (1) incoming gradient dh of layer i =
//         PREV_TOP : dtop[u]  (received from the next stage, or logits grad)
//         PREV_AGG : drop_{i+1}( sum_v w_uv * bg_{i+1}[v] over done chunks )
//                    (backward_prev_row of layer i+1, nn.hpp:222-257; bg holds
//                     (1-a)*dagg for Gcn2Conv and dagg for GcnConv)
//         PREV_OWN : drop_{i+1}( bg_{i+1}[u] )     (Dense layer i+1)
//       (+ dh0_run[u] when layer i is global layer 0 of a GCNII, :753-758)
//   (2) OUT_LAYER: backward_out_row of layer i (nn.hpp:202-218):
//         dz = relu ? (h>0 ? dh : 0) : dh ; dagg = dz . W^T (ascending j)
//         Gcn2Conv: dagg = (1-beta) dz + beta dagg ; dh0 += a dagg
//       and stores dz and bg_i (the gather source of layer i's backward_prev);
//       OUT_DHIN : stores dh into dh_in (gradient sent to the previous stage).
// ---------------------------------------------------------------------------
struct BwdParams {
    uint32_t r0, r1;
    uint32_t* ticket;
    const uint64_t* rowptr;
    const uint2* edges;
    const float* bgn;
    const float* bgn_snap;
    uint32_t bgnstride;
    uint32_t zrow;
    uint64_t done;
    DropKey prev_mask;
    const float* dtop;
    uint32_t dtopstride;
    const uint32_t* orig;
    uint32_t dh_width;
    const float* dh0_add;
    uint32_t dh0stride;
    const float* h;
    uint32_t hstride;
    uint32_t relu;
    float* dz;
    uint32_t dzstride;
    const float* W;
    const float* WT;  // W^T (dout x din), staged by the split path's k_bwd_tile
    uint32_t din, dout;
    uint32_t need_dagg;
    uint32_t gcn2;
    float alpha, oma, beta, omb;
    float* dh0;
    float* bg;
    uint32_t bgstride;
    float* dh_in;
    uint32_t dhinstride;
    // next layer SageConv (PREV_SAGE*): transposed mean adjacency (weight 1/deg(col))
    // and the column of its bg where the aggregated half's gradient starts
    const uint64_t* rowptr_m;
    const uint2* edges_m;
    uint32_t sgap;
};

// ---------------------------------------------------------------------------
// Softmax cross-entropy head (nn.hpp:373-403, engines_impl.hpp:39-51, :725-734).
// Warp per row, C <= 128. Loss is summed in double; per-block partials are
// folded in a fixed order so a run is reproducible.
// ---------------------------------------------------------------------------
struct XentParams {
    uint32_t r0, r1, classes;
    const float* logits;
    uint32_t lstride;
    const uint32_t* labels;
    const uint8_t* split;
    float inv_count;
    float* grad;
    uint32_t gstride;
    double* part_loss;
    unsigned long long* part_correct;  // 3 per block
    // k_xent_stats: row i of [r0, r1) is stash row rows[i] (ascending original id), so
    // the loss partials do not depend on the chunking; null: row i
    const uint32_t* rows;
};

struct RowSoftmax {
    float mx, sum;
    uint32_t argmax;
};

__device__ __forceinline__ RowSoftmax row_softmax(const float4 l, uint32_t classes, int lane) {
    const uint32_t c0 = 4 * lane;
    float best = -INFINITY;
    uint32_t bi = 0xffffffffu;
    const float vals[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (c0 + q < classes && (bi == 0xffffffffu || vals[q] > best)) {
            best = vals[q];
            bi = c0 + q;
        }
    for (int off = 16; off > 0; off >>= 1) {
        const float ob = __shfl_xor_sync(kFull, best, off);
        const uint32_t oi = __shfl_xor_sync(kFull, bi, off);
        if (oi != 0xffffffffu && (bi == 0xffffffffu || ob > best || (ob == best && oi < bi))) {
            best = ob;
            bi = oi;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (c0 + q < classes) s += expf(vals[q] - best);
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
    return {best, s, bi};
}

__global__ void __launch_bounds__(kBlock) k_xent_stats(XentParams p) {
    __shared__ double sl[kWarpsPerBlock];
    __shared__ unsigned long long sc[kWarpsPerBlock][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double loss = 0.0;
    unsigned long long corr[3] = {0, 0, 0};
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    for (uint32_t i = p.r0 + blockIdx.x * kWarpsPerBlock + warp; i < p.r1; i += nw) {
        const uint32_t v = p.rows ? p.rows[i] : i;
        const uint8_t s = p.split[v];
        if (s == 0 || s > 3) continue;
        const float4 l = uint32_t(4 * lane) < p.classes
                             ? ld4_rw(p.logits + size_t(v) * p.lstride + 4 * lane)
                             : f4_zero();
        const RowSoftmax r = row_softmax(l, p.classes, lane);
        const uint32_t label = p.labels[v];
        if (lane == 0) {
            corr[s - 1] += r.argmax == label;
            if (s == 1) {
                const float ll = p.logits[size_t(v) * p.lstride + label];
                loss += double(logf(r.sum)) - double(ll - r.mx);
            }
        }
    }
    if (lane == 0) {
        sl[warp] = loss;
        sc[warp][0] = corr[0];
        sc[warp][1] = corr[1];
        sc[warp][2] = corr[2];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        unsigned long long c[3] = {0, 0, 0};
        for (int w = 0; w < kWarpsPerBlock; ++w) {
            t += sl[w];
            for (int k = 0; k < 3; ++k) c[k] += sc[w][k];
        }
        p.part_loss[blockIdx.x] = t;
        for (int k = 0; k < 3; ++k) p.part_correct[3 * blockIdx.x + k] = c[k];
    }
}

__global__ void k_xent_fold(const double* part_loss, const unsigned long long* part_correct, uint32_t parts,
                            double* out_loss, unsigned long long* out_correct) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t = 0;
    unsigned long long c[3] = {0, 0, 0};
    for (uint32_t b = 0; b < parts; ++b) {
        t += part_loss[b];
        for (int k = 0; k < 3; ++k) c[k] += part_correct[3 * b + k];
    }
    *out_loss = t;
    for (int k = 0; k < 3; ++k) out_correct[k] = c[k];
}

// grad = (softmax - onehot) / n_train on train rows, 0 elsewhere (xent_row_grad).
__global__ void __launch_bounds__(kBlock) k_xent_grad(XentParams p) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    const bool act = uint32_t(4 * lane) < p.classes;
    for (uint32_t v = p.r0 + blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); v < p.r1; v += nw) {
        float4 g = f4_zero();
        if (p.split[v] == 1) {
            const float4 l = act ? ld4_rw(p.logits + size_t(v) * p.lstride + 4 * lane) : f4_zero();
            const RowSoftmax r = row_softmax(l, p.classes, lane);
            const uint32_t label = p.labels[v];
            const float vals[4] = {l.x, l.y, l.z, l.w};
            float outv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t j = 4 * lane + q;
                float e = j < p.classes ? __fmul_rn(__fdiv_rn(expf(vals[q] - r.mx), r.sum), p.inv_count) : 0.f;
                if (j == label) e = __fsub_rn(e, p.inv_count);
                outv[q] = e;
            }
            g = make_float4(outv[0], outv[1], outv[2], outv[3]);
        }
        if (act) st4(p.grad + size_t(v) * p.gstride + 4 * lane, g);
    }
}

// ---------------------------------------------------------------------------
// Parameter gradients (param_grads_for_rows, nn.hpp:269-293): dW = pre^T dz
// (x beta for Gcn2Conv), db = sum dz, over ALL rows, once per epoch
// (engines_impl.hpp:873-876). Split-K over row ranges into a workspace, then a
// fixed-order fold: deterministic run to run (not bitwise equal to the
// reference's single ascending sum; tolerance-level, SURVEY §8a' item 7).
// CTA tile: 64 (k_in) x 64 (out); thread: 4 x 4; rows staged 32 at a time.
// ---------------------------------------------------------------------------
struct PgradParams {
    uint32_t n, rows_per_split;  // n = end row (exclusive); rows start at row0
    uint32_t row0;
    const float* pre;
    uint32_t prestride;
    const float* dz;
    uint32_t dzstride;
    uint32_t din, dout;
    float* ws;   // splits x din x dout
    float* wsb;  // splits x dout
    const uint32_t* rows;  // reduction row i -> stash row rows[i] (ascending original id); null: i
};

// CTA tile 128 (k_in) x 128 (out): each row of pre/dz is read once per CTA.
// Thread (ti, tj) owns i in {4ti..4ti+3, 64+4ti..+3} and j likewise, so the
// shared-memory float4 reads of a warp are contiguous (conflict-free).
// Rows are staged 16 at a time, double-buffered through registers.
constexpr int kPgRows = 16;
__global__ void __launch_bounds__(256, 2) k_pgrad_partial(PgradParams p) {
    __shared__ __align__(16) float Ps[2][kPgRows][128];
    __shared__ __align__(16) float Ds[2][kPgRows][128];
    const uint32_t split = blockIdx.x;
    const uint32_t i0 = blockIdx.y * 128;
    const uint32_t rbeg = p.row0 + split * p.rows_per_split;
    const uint32_t rend = min(p.n, rbeg + p.rows_per_split);
    const int tid = threadIdx.x;
    const int ti = tid / 16, tj = tid % 16;
    float acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
    float bacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // staging: 16 rows x 128 cols x 2 arrays = 4096 floats = 1024 float4; 4 per thread
    const int lr = tid / 16, lc = (tid % 16) * 8;  // thread loads row lr, cols lc..lc+7 of both arrays
    float4 rp[2], rd[2];
    auto fetch = [&](uint32_t r0) {
        const uint32_t row = r0 + lr;
        const bool ok = row < rend;
        const uint32_t srow = ok && p.rows ? p.rows[row] : row;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t ci = i0 + lc + 4 * h, cj = lc + 4 * h;
            rp[h] = (ok && ci < p.din) ? *reinterpret_cast<const float4*>(p.pre + size_t(srow) * p.prestride + ci)
                                       : f4_zero();
            rd[h] = (ok && cj < p.dout) ? *reinterpret_cast<const float4*>(p.dz + size_t(srow) * p.dzstride + cj)
                                        : f4_zero();
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            *reinterpret_cast<float4*>(&Ps[buf][lr][lc + 4 * h]) = rp[h];
            *reinterpret_cast<float4*>(&Ds[buf][lr][lc + 4 * h]) = rd[h];
        }
    };
    int buf = 0;
    if (rbeg < rend) {
        fetch(rbeg);
        stash(0);
    }
    __syncthreads();
    for (uint32_t r0 = rbeg; r0 < rend; r0 += kPgRows) {
        const bool more = r0 + kPgRows < rend;
        if (more) fetch(r0 + kPgRows);
#pragma unroll 4
        for (int r = 0; r < kPgRows; ++r) {
            const float4 a0 = *reinterpret_cast<const float4*>(&Ps[buf][r][4 * ti]);
            const float4 a1 = *reinterpret_cast<const float4*>(&Ps[buf][r][64 + 4 * ti]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Ds[buf][r][4 * tj]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Ds[buf][r][64 + 4 * tj]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
            if (ti == 0)
#pragma unroll
                for (int b = 0; b < 8; ++b) bacc[b] += bv[b];
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    float* w = p.ws + size_t(split) * p.din * p.dout;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const uint32_t i = i0 + (a < 4 ? 4 * ti + a : 64 + 4 * ti + a - 4);
        if (i >= p.din) continue;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t j = b < 4 ? 4 * tj + b : 64 + 4 * tj + b - 4;
            if (j < p.dout) w[size_t(i) * p.dout + j] = acc[a][b];
        }
    }
    if (blockIdx.y == 0 && ti == 0 && p.wsb)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t j = b < 4 ? 4 * tj + b : 64 + 4 * tj + b - 4;
            if (j < p.dout) p.wsb[size_t(split) * p.dout + j] = bacc[b];
        }
}

__global__ void k_pgrad_fold(const float* ws, const float* wsb, uint32_t splits, uint32_t din,
                             uint32_t dout, float scale, uint32_t apply_scale, float* gW, float* gb) {
    const uint32_t total = din * dout;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total + dout;
         idx += gridDim.x * blockDim.x) {
        if (idx < total) {
            float s = 0.f;
            for (uint32_t k = 0; k < splits; ++k) s += ws[size_t(k) * total + idx];
            gW[idx] = apply_scale ? __fmul_rn(s, scale) : s;
        } else if (wsb && gb) {
            const uint32_t j = idx - total;
            float s = 0.f;
            for (uint32_t k = 0; k < splits; ++k) s += wsb[size_t(k) * dout + j];
            gb[j] = s;
        }
    }
}

// ---------------------------------------------------------------------------
// Adam / SGD (Optimizer::update, nn.hpp:474-490) with the reference's float
// operation order; c1/c2 are computed on the host in double and rounded.
// ---------------------------------------------------------------------------
struct AdamParams {
    float* p;
    const float* g;
    float* m;
    float* v;
    uint32_t n;
    uint32_t sgd;
    float lr, b1, b2, omb1, omb2, eps, c1, c2;
};

// Stage-message copy on the SMs (16-byte vectors when aligned): used by the IPC
// transport instead of copy-engine memcpy when GP_IPC_SMCOPY=1.
__global__ void k_copy(float* __restrict__ dst, const float* __restrict__ src, size_t n) {
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, step = size_t(gridDim.x) * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const size_t n4 = n / 4;
        for (size_t i = tid; i < n4; i += step)
            reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
        for (size_t i = n4 * 4 + tid; i < n; i += step) dst[i] = src[i];
    } else {
        for (size_t i = tid; i < n; i += step) dst[i] = src[i];
    }
}

// SageConv weights in the gapped layout of pre / bg (own half at rows [0, din),
// aggregated half at rows [sgap, sgap + din), zero rows between): Wg (kw x dout)
// for the forward transform and WTg = Wg^T (dout x kw) for dagg = dz.W^T. The
// zero rows meet pre's zero padding columns (+0 products): bit-exact.
__global__ void k_sage_weights(const float* __restrict__ W, float* __restrict__ Wg, float* __restrict__ WTg,
                               uint32_t din, uint32_t dout, uint32_t sgap) {
    const uint32_t kw = sgap + din;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kw * dout; idx += gridDim.x * blockDim.x) {
        const uint32_t r = idx / dout, c = idx % dout;
        float v = 0.f;
        if (r < din) v = W[size_t(r) * dout + c];
        else if (r >= sgap) v = W[size_t(r - sgap + din) * dout + c];
        Wg[idx] = v;
        WTg[size_t(c) * kw + r] = v;
    }
}

// Zero n 32-bit words (in-epoch resets; a kernel of this module instead of the
// runtime's memset, so nothing is loaded lazily while peers wait in-stream).
__global__ void k_zero(uint32_t* __restrict__ p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = 0u;
}

// Trace anchor: the device's global timer (ns) at this point of the stream, so
// CUDA-event times of different stages (devices, processes) share one timebase.
__global__ void k_stamp(unsigned long long* out) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}

__global__ void k_adam(AdamParams a) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const float g = a.g[i];
        if (a.sgd) {
            a.p[i] = __fsub_rn(a.p[i], __fmul_rn(a.lr, g));
            continue;
        }
        const float m = __fadd_rn(__fmul_rn(a.b1, a.m[i]), __fmul_rn(a.omb1, g));
        const float v = __fadd_rn(__fmul_rn(a.b2, a.v[i]), __fmul_rn(__fmul_rn(a.omb2, g), g));
        a.m[i] = m;
        a.v[i] = v;
        const float mhat = __fdiv_rn(m, a.c1);
        const float vhat = __fdiv_rn(v, a.c2);
        a.p[i] = __fsub_rn(a.p[i], __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
    }
}

}  // namespace gp

namespace gp {

// ---------------------------------------------------------------------------
// Hybrid halo pull (exchange_rows / unpack_rows, engines_impl.hpp:626-643,
// :62-70): copy the listed rows of a peer's buffer into ours; for the forward
// also write the dropped copy into this layer's gather table.
// ---------------------------------------------------------------------------
struct PullParams {
    const uint32_t* rows;
    uint32_t count;
    const float* src;
    float* dst;
    uint32_t stride;
    float* dstG;
    uint32_t gstride;
    uint32_t width;
    const uint32_t* orig;
    DropKey mask;
};

__global__ void __launch_bounds__(kBlock) k_pull_rows(PullParams p) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    for (uint32_t i = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); i < p.count; i += nw) {
        const uint32_t v = p.rows[i];
        for (uint32_t c0 = 4 * lane; c0 < p.width; c0 += 128) {
            const float4 x = ld4_rw(p.src + size_t(v) * p.stride + c0);
            st4(p.dst + size_t(v) * p.stride + c0, x);
            if (p.dstG) st4(p.dstG + size_t(v) * p.gstride + c0, drop4(p.mask, p.orig[v], c0, p.width, x));
        }
    }
}

// Done-filtered CSR of one epoch's backward pass. backward_prev_row (nn.hpp:222-257)
// gathers only the entries of chunks already processed; every layer of chunk k runs with
// the same done set (the chunks at or after k in the forward order, engines_impl.hpp:
// 829-866), so the filter is a per-epoch property of (row, entry), not of the layer. It is
// applied once per epoch here, order-preserving, and the backward gathers of all layers
// then read the compacted rows without a per-batch ballot. Pass 1 (COUNT) writes the kept
// count of row v to rowptr_f[v + 1]; an in-place inclusive scan turns it into row
// pointers (rowptr_f[own_begin] stays 0); pass 2 writes the kept entries.
struct DoneCsrParams {
    const uint64_t* rowptr;
    const uint2* edges;
    uint64_t* rowptr_f;
    uint2* edges_f;
    uint32_t rb[kMaxChunks + 1];  // chunk k owns rows [rb[k], rb[k + 1])
    uint64_t mask[kMaxChunks];    // done set of chunk k's backward step
};

template <bool COUNT>
__global__ void __launch_bounds__(kBlock) k_done_csr(const __grid_constant__ DoneCsrParams p) {
    const uint32_t k = blockIdx.y;
    const uint64_t m = p.mask[k];
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    for (uint32_t v = p.rb[k] + blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); v < p.rb[k + 1]; v += nw) {
        const uint64_t e0 = p.rowptr[v], e1 = p.rowptr[v + 1];
        uint64_t out = COUNT ? 0 : p.rowptr_f[v];
        for (uint64_t e = e0; e < e1; e += 32) {
            const bool in = e + lane < e1;
            const uint2 x = in ? __ldcs(reinterpret_cast<const uint2*>(p.edges) + e + lane) : make_uint2(0u, 0u);
            const bool ok = in && ((m >> (x.x >> kColBits)) & 1ull);
            const unsigned b = __ballot_sync(kFull, ok);
            if (!COUNT && ok) p.edges_f[out + __popc(b & ((1u << lane) - 1u))] = x;
            out += __popc(b);
        }
        if (COUNT && lane == 0) p.rowptr_f[v + 1] = out;
    }
}

// In-place inclusive scan of u64 values (the filtered CSR's row counts -> row pointers):
// k_scan_tiles scans tiles of kScanTile values per CTA and records each tile's total,
// k_scan_totals turns the totals into exclusive tile offsets (one CTA, sequential over
// chunks of 1024), k_scan_add adds them. Integer sums: the result is exact and order-free.
constexpr uint32_t kScanThreads = 1024, kScanPer = 4, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ unsigned long long block_incl_scan(unsigned long long x, unsigned long long* warp_tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long t = lane < int(blockDim.x >> 5) ? warp_tot[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, t, o);
            if (lane >= o) t += y;
        }
        warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const unsigned long long r = x + (w > 0 ? warp_tot[w - 1] : 0ull);
    __syncthreads();  // warp_tot is reused by the caller's next scan
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(unsigned long long* v, uint32_t n,
                                                             unsigned long long* totals) {
    __shared__ unsigned long long wt[32];
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanPer;
    unsigned long long a[kScanPer], sum = 0;
#pragma unroll
    for (int q = 0; q < int(kScanPer); ++q) {
        a[q] = base + q < n ? v[base + q] : 0ull;
        sum += a[q];
    }
    const unsigned long long incl = block_incl_scan(sum, wt);
    unsigned long long run = incl - sum;
#pragma unroll
    for (int q = 0; q < int(kScanPer); ++q) {
        run += a[q];
        if (base + q < n) v[base + q] = run;
    }
    if (threadIdx.x == blockDim.x - 1) totals[blockIdx.x] = incl;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_totals(unsigned long long* totals, uint32_t tiles) {
    __shared__ unsigned long long wt[32];
    unsigned long long carry = 0;
    for (uint32_t c = 0; c < tiles; c += kScanThreads) {
        const uint32_t i = c + threadIdx.x;
        const unsigned long long x = i < tiles ? totals[i] : 0ull;
        const unsigned long long incl = block_incl_scan(x, wt);
        if (i < tiles) totals[i] = carry + incl - x;  // exclusive offset of tile i
        __shared__ unsigned long long last;
        if (threadIdx.x == kScanThreads - 1) last = incl;
        __syncthreads();
        carry += last;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(unsigned long long* v, uint32_t n,
                                                           const unsigned long long* offsets) {
    if (blockIdx.x == 0) return;
    const unsigned long long off = offsets[blockIdx.x];
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanPer;
#pragma unroll
    for (int q = 0; q < int(kScanPer); ++q)
        if (base + q < n) v[base + q] += off;
}

// Normalised adjacency of the renumbered graph built on the device from the raw neighbour
// lists (normalize_adjacency<float> graph.cpp:68-98: w_vu = float(1 / sqrt(d_v d_u)) in double,
// d = degree + 1 with the self loop, which goes before the first neighbour u > v; the
// adjacency bundle nn.hpp:85-98). One warp per renumbered row r (v = inv[r]), 32 entries per
// step: the same entries, order and bits as the host builder (upload_graph_src), which
// remains the path for hybrid groups and precomputed values. Also counts the entries per
// (row chunk, column chunk) for the done-filtered accounting, and flags a neighbour out of
// range or equal to its row.
struct BuildEdgesParams {
    const uint64_t* off;    // raw offsets (original ids)
    const uint32_t* nbr;    // raw neighbours
    const uint32_t* inv;    // renumbered row -> original id
    const uint32_t* perm;   // original id -> renumbered row
    const uint32_t* chunk;  // original id -> chunk
    const uint64_t* rp;     // renumbered row pointers (self loops included)
    uint2* edges;
    unsigned long long* blk;  // K x K entry counts
    uint32_t* bad;
    uint32_t n, K, loops;
};

__global__ void __launch_bounds__(kBlock) k_build_edges(BuildEdgesParams p) {
    extern __shared__ unsigned int hist[];  // K x K per CTA
    for (uint32_t i = threadIdx.x; i < p.K * p.K; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarpsPerBlock;
    const double extra = p.loops ? 1.0 : 0.0;
    for (uint32_t r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); r < p.n; r += nw) {
        const uint32_t v = p.inv[r];
        const uint64_t e0 = p.off[v], e1 = p.off[v + 1];
        const double dv = double(e1 - e0) + extra;
        const uint32_t cr = p.chunk[v];
        const uint64_t base = p.rp[r];
        bool placed = !p.loops;  // warp-uniform: the self loop is written
        const uint2 self = make_uint2(r | (cr << kColBits), __float_as_uint(float(1.0 / sqrt(dv * dv))));
        for (uint64_t b = e0; b < e1; b += 32) {
            const uint64_t i = b + lane;
            const bool in = i < e1;
            const uint32_t u = in ? p.nbr[i] : 0u;
            const bool ok = in && u < p.n && u != v;
            if (__any_sync(kFull, in && !ok) && lane == 0) atomicOr(p.bad, 1u);
            uint32_t shift = placed ? (p.loops ? 1u : 0u) : 0u;
            if (!placed) {
                const unsigned gt = __ballot_sync(kFull, ok && u > v);
                if (gt) {
                    const int first = __ffs(gt) - 1;
                    if (lane == first) p.edges[base + (b - e0) + first] = self;
                    shift = lane >= first ? 1u : 0u;
                    placed = true;
                }
            }
            uint32_t cu = 0xffffffffu;
            if (ok) {
                cu = p.chunk[u];
                const double du = double(p.off[u + 1] - p.off[u]) + extra;
                p.edges[base + (i - e0) + shift] =
                    make_uint2(p.perm[u] | (cu << kColBits), __float_as_uint(float(1.0 / sqrt(dv * du))));
            }
            const unsigned grp = __match_any_sync(kFull, cu);
            if (ok && lane == __ffs(grp) - 1) atomicAdd(&hist[cr * p.K + cu], __popc(grp));
        }
        if (!placed && lane == 0) p.edges[base + (e1 - e0)] = self;
        if (p.loops && lane == 0) atomicAdd(&hist[cr * p.K + cr], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.K * p.K; i += blockDim.x)
        if (hist[i]) atomicAdd(&p.blk[i], (unsigned long long)hist[i]);
}

// group_weight_sync (engines_impl.hpp:102-128): rank 0 folds the group's
// gradients in rank order, g = ((g0 + g1) + g2) + ..., one rounding per add.
struct FoldParams {
    const float* src[8];
    float* dst;
    uint32_t G;
    uint32_t n;
};

__global__ void k_group_fold(FoldParams p) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x) {
        float s = p.src[0][i];
        for (uint32_t r = 1; r < p.G; ++r) s = __fadd_rn(s, p.src[r][i]);
        p.dst[i] = s;
    }
}

}  // namespace gp

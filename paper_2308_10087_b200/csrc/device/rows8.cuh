// Half-warp row kernels with 256-bit gathers (sm_100a `ld.global.v8.f32`).
//
// A half-warp (16 lanes) owns one row; lane h of the half owns columns
// 8h..8h+7, so one LDG.256 per lane fetches a whole 416-byte row (13 lanes,
// 13 sectors) and a warp advances two rows at once. Each row is still reduced
// by its own lanes in ascending neighbour order with one rounded multiply and
// one rounded add per term, so results stay bit-identical to the reference's
// scalar loops (kernel::spmv_row nn.hpp:143-154, dense_rows matrix.hpp:63-74,
// dense_rows_wt matrix.hpp:77-86). Compared with one float4 per lane this
// halves shuffles, address arithmetic and load instructions per gathered edge,
// and the L2 eviction hint is encoded in the instruction (no policy register).
#pragma once

#include "kernels.cuh"

namespace gp {

struct F8 {
    float v[8];
};

__device__ __forceinline__ F8 f8_zero() {
    F8 r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = 0.f;
    return r;
}

// Gather-table read, kept in L2 (evict_last), not allocated in L1. Always
// issued on a valid address (padding slots re-read a row with weight 0), so
// there is neither predication nor a select waiting on the loaded value.
__device__ __forceinline__ F8 ld8_gather(const float* p) {
    F8 x;
    asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(x.v[0]), "=f"(x.v[1]), "=f"(x.v[2]), "=f"(x.v[3]), "=f"(x.v[4]), "=f"(x.v[5]), "=f"(x.v[6]),
          "=f"(x.v[7])
        : "l"(p));
    return x;
}

// Row-local streams: evict_first so they never displace the gather table.
__device__ __forceinline__ F8 ld8_stream(const float* p) {
    F8 x;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(x.v[0]), "=f"(x.v[1]), "=f"(x.v[2]), "=f"(x.v[3]), "=f"(x.v[4]), "=f"(x.v[5]),
                   "=f"(x.v[6]), "=f"(x.v[7])
                 : "l"(p));
    return x;
}
__device__ __forceinline__ void st8_stream(float* p, const F8& x) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(x.v[0]), "f"(x.v[1]), "f"(x.v[2]), "f"(x.v[3]), "f"(x.v[4]), "f"(x.v[5]), "f"(x.v[6]),
                 "f"(x.v[7])
                 : "memory");
}

__device__ __forceinline__ F8 drop8(const DropKey& m, uint32_t vo, uint32_t c0, uint32_t width, const F8& x) {
    F8 r;
#pragma unroll
    for (int q = 0; q < 8; ++q) r.v[q] = c0 + q < width ? drop_apply(m, vo, c0 + q, x.v[q]) : 0.f;
    return r;
}

__device__ __forceinline__ F8 shfl8(const F8& x, int src) {
    F8 r;
#pragma unroll
    for (int q = 0; q < 8; ++q) r.v[q] = __shfl_sync(kFull, x.v[q], src);
    return r;
}

// Sum over the CSR row of w * src[col] (8 columns per lane), in ascending entry
// order with one rounded multiply and add per term.
//
// Entries are consumed in full batches of 16 per half-warp whose 16 gathers are
// fully unrolled (NB issued per group), so the compiler can keep loads of later
// groups in flight under the arithmetic of earlier ones; the CSR batch after the
// current one is prefetched. Unused slots are padding: the half's own row with
// weight 0 (acc starts at +0 and never becomes -0, so acc + 0*x == acc, and the
// address is always valid, so there is no predication on the loads).
//
// FILTER keeps only entries of done chunks: each CSR batch is compacted (ballot +
// __fns, order-preserving) and appended to a per-half queue of up to 15 carried
// entries; a batch of 16 is gathered as soon as either half's queue is full, so
// sparse done-sets do not pay for padded slots. HIST (historical-gradient
// ablation) keeps every entry and reads not-done chunks from `snap`.
// GP_TAIL_SKIP: the last (partial) batch of a row pair gathers only the groups of NB slots
// that hold an entry in either half (padding slots past both halves' ends are not loaded)
#ifndef GP_TAIL_SKIP
#define GP_TAIL_SKIP 1
#endif
#ifndef GP_SMEM_EDGES
#define GP_SMEM_EDGES 1
#endif
// CSR entries of the current batch are broadcast to the half-warp through a
// 16-entry shared-memory slot (one LDS.64 per entry for both halves) instead of
// two shuffles per entry: fewer L1TEX data-pipe wavefronts, which the gather
// saturates first.
constexpr bool kSmemEdges = GP_SMEM_EDGES != 0;
constexpr uint32_t kEdgeSlotBytes = kWarpsPerBlock * 32 * 8;  // per CTA: 16 entries x 2 halves x 8 warps

template <bool FILTER, bool HIST, int NB>
__device__ __forceinline__ F8 gather_row8(const uint64_t* __restrict__ rowptr, const uint2* __restrict__ edges,
                                          uint32_t v, bool has_row, const float* __restrict__ src,
                                          const float* __restrict__ snap, uint32_t stride, uint64_t done,
                                          int lane, bool active, uint2* eslot, const F8& init) {
    const int hl = lane & 15, hb = lane & 16;
    uint64_t e0 = 0, e1 = 0;
    if (has_row) {
        e0 = rowptr[v];
        e1 = rowptr[v + 1];
    }
    const uint32_t n_my = uint32_t(e1 - e0);
    const uint32_t n_max = max(n_my, __shfl_xor_sync(kFull, n_my, 16));
    const uint32_t loff = active ? 8u * hl : 0u;
    const float* ls = src + loff;
    const float* lsn = HIST ? snap + loff : nullptr;
    // padding entry: this half's own row (distinct per half-warp, so padding never
    // concentrates on one L2 line), weight 0, chunk bits 0
    const uint2 pad = make_uint2(has_row ? v : 0u, 0u);
    F8 acc = init;  // +0 (SpMM) or the own-row term SageConv's backward starts from (nn.hpp:234-243)
    uint2* es = eslot + (hb ? 16 : 0);
    // lim: slots [lim, 16) are padding in both halves (warp-uniform), so their groups are skipped
    auto batch16 = [&](const uint2 my, const uint32_t lim) {
        if (kSmemEdges) {
            __syncwarp();
            es[hl] = my;
            __syncwarp();
        }
#pragma unroll
        for (int t = 0; t < 16; t += NB) {
            if (GP_TAIL_SKIP && uint32_t(t) >= lim) break;
            float w[NB];
            F8 x[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                uint32_t packed;
                if (kSmemEdges) {
                    const uint2 e = es[t + i];
                    packed = e.x;
                    w[i] = __uint_as_float(e.y);
                } else {
                    packed = __shfl_sync(kFull, my.x, hb + t + i);
                    w[i] = __uint_as_float(__shfl_sync(kFull, my.y, hb + t + i));
                }
                const float* s = ls;
                if (HIST && !((done >> (packed >> kColBits)) & 1ull)) s = lsn;
                x[i] = ld8_gather(s + size_t(packed & kColMask) * stride);
            }
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc.v[c] = mul_add(acc.v[c], w[i], x[i].v[c]);
        }
    };
    uint2 nxt = hl < int(n_my) ? ld_edge(edges + e0 + hl) : pad;
    if (!FILTER || HIST) {
        for (uint32_t off = 0; off < n_max; off += 16) {
            const uint2 my = nxt;
            nxt = off + 16 + hl < n_my ? ld_edge(edges + e0 + off + 16 + hl) : pad;
            if (off + 16 <= n_max)
                batch16(my, 16u);  // full batch: no group test in the hot loop
            else
                batch16(my, n_max - off);
        }
        return acc;
    }
    uint2 carry = pad;  // queued (compacted) entries in lanes [0, nq)
    int nq = 0;
    for (uint32_t off = 0; off < n_max; off += 16) {
        uint2 e = nxt;
        const bool ok = off + hl < n_my && ((done >> (e.x >> kColBits)) & 1ull);
        nxt = off + 16 + hl < n_my ? ld_edge(edges + e0 + off + 16 + hl) : pad;
        const unsigned m = (__ballot_sync(kFull, ok) >> hb) & 0xffffu;
        const int cnt = __popc(m);
        // compact the batch, then append it behind the queue: lane hl takes
        // queue[hl] if hl < nq, else new[hl - nq]
        const int from = hl < cnt ? int(__fns(m, 0, hl + 1)) : hl;
        e.x = __shfl_sync(kFull, e.x, hb + from);
        e.y = __shfl_sync(kFull, e.y, hb + from);
        const int j = hl - nq;
        const uint32_t ax = __shfl_sync(kFull, e.x, hb + (j < 0 ? 0 : j));
        const uint32_t ay = __shfl_sync(kFull, e.y, hb + (j < 0 ? 0 : j));
        const int tot = nq + cnt;
        const uint2 cur = j < 0 ? carry : (j < cnt ? make_uint2(ax, ay) : pad);
        const int tmax = max(tot, __shfl_xor_sync(kFull, tot, 16));
        if (tmax >= 16) {
            batch16(cur, 16u);
            // entries of the new batch beyond this 16-slot batch stay queued
            const int k = 16 - nq + hl;
            const uint32_t rx = __shfl_sync(kFull, e.x, hb + (k < 16 ? k : 15));
            const uint32_t ry = __shfl_sync(kFull, e.y, hb + (k < 16 ? k : 15));
            nq = tot > 16 ? tot - 16 : 0;
            carry = hl < nq ? make_uint2(rx, ry) : pad;
        } else {
            carry = cur;
            nq = tot;
        }
    }
    const int nq_max = max(nq, __shfl_xor_sync(kFull, nq, 16));
    if (nq_max > 0) batch16(carry, uint32_t(nq_max));
    return acc;
}

// ---------------------------------------------------------------------------
// Row transforms (dense_rows matrix.hpp:63-74, dense_rows_wt :77-86) as warp
// GEMVs over R rows at once: lane L owns output columns L, L+32, L+64, L+96 of
// all R rows. Per input index i the warp reads the staged matrix row i once
// (consecutive lanes, consecutive words: conflict-free, ~4 wavefronts per row
// instead of the 13-15 of a half-warp-per-row layout) and x[.][i] of the R rows by
// broadcast from a [i][R] staging area. Each output still accumulates one rounded
// product per i in ascending i, so results are bit-identical to the reference.
// ---------------------------------------------------------------------------
// Matrix staging: rows x cols, row stride ms = pad8(cols) words, + 32 words of
// tail padding (lanes whose 4th column is past `cols` read padding or the next row
// and discard it). transpose: Ms[r][c] = W[c][r] (W has leading dimension ld).
__host__ __device__ constexpr uint32_t mat_stride(uint32_t cols) { return (cols + 7u) & ~7u; }
__host__ __device__ constexpr size_t row_smem_bytes(uint32_t mrows, uint32_t mcols, uint32_t R) {
    // matrix + tail pad + bias (128) + x staging (8 warps x 128 x R)
    return (size_t(mrows) * mat_stride(mcols) + 32 + 128 + size_t(kWarpsPerBlock) * 128 * R) * 4 + kEdgeSlotBytes;
}

__device__ __forceinline__ void stage_mat(float* Ms, const float* W, uint32_t rows, uint32_t cols, bool transpose,
                                          uint32_t ld) {
    const uint32_t ms = mat_stride(cols);
    for (uint32_t idx = threadIdx.x; idx < rows * ms + 32; idx += blockDim.x) {
        const uint32_t r = idx / ms, c = idx % ms;
        float val = 0.f;
        if (r < rows && c < cols) val = transpose ? W[size_t(c) * ld + r] : W[size_t(r) * ld + c];
        Ms[idx] = val;
    }
}

template <int R>
__device__ __forceinline__ void gemv_w(float (&o)[R][4], const float* __restrict__ xs, const float* __restrict__ Ms,
                                       uint32_t rows, uint32_t ms, int lane) {
    const float* mcol = Ms + lane;
#pragma unroll 2
    for (uint32_t i = 0; i < rows; ++i) {
        float x[R];
        if (R == 2) {
            const float2 t = *reinterpret_cast<const float2*>(xs + 2 * i);
            x[0] = t.x;
            x[1] = t.y;
        } else {
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                const float4 t = *reinterpret_cast<const float4*>(xs + R * i + 4 * q);
                x[4 * q] = t.x, x[4 * q + 1] = t.y, x[4 * q + 2] = t.z, x[4 * q + 3] = t.w;
            }
        }
        const float* mrow = mcol + size_t(i) * ms;
        const float w0 = mrow[0], w1 = mrow[32], w2 = mrow[64], w3 = mrow[96];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            o[r][0] = mul_add(o[r][0], x[r], w0);
            o[r][1] = mul_add(o[r][1], x[r], w1);
            o[r][2] = mul_add(o[r][2], x[r], w2);
            o[r][3] = mul_add(o[r][3], x[r], w3);
        }
    }
}

// Stage the warp's two half-warp rows (8 values per lane) as xs[i][2].
__device__ __forceinline__ void stage_x2(float* xs, const F8& x, int hl, int hb, bool active) {
    if (active) {
#pragma unroll
        for (int c = 0; c < 8; ++c) xs[(8 * hl + c) * 2 + (hb ? 1 : 0)] = x.v[c];
    }
    __syncwarp();
}

__device__ __forceinline__ void st1_stream(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ float ld1_stream(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// Forward epilogue of row v for the lane's columns: (Gcn2Conv) identity mix with
// pre, ReLU, h, and the next layer's dropped gather source (nn.hpp:188-196).
template <int R, bool GCN2>
__device__ __forceinline__ void fwd_epilogue(const FwdParams& p, float (&o)[R][4], const float* xs, uint32_t v0,
                                             int lane, uint64_t pol) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t v = v0 + r;
        if (v >= p.r1) break;
        const uint32_t vo = p.gnext ? p.orig[v] : 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t c = lane + 32 * k;
            if (c >= p.dout) break;
            float val = o[r][k];
            if (GCN2) val = __fadd_rn(__fmul_rn(p.omb, xs[c * R + r]), __fmul_rn(p.beta, val));
            if (p.relu && val < 0.f) val = 0.f;
            st1_stream(p.out + size_t(v) * p.outstride + c, val, pol);
            if (p.gnext) st1_stream(p.gnext + size_t(v) * p.gnstride + c, drop_apply(p.next_mask, vo, c, val), pol);
        }
    }
}

// Backward transform of row u: dagg = dz.W^T (R rows in o), Gcn2Conv mixes,
// dh0 += a*dagg, bg = (1-a)*dagg or dagg (nn.hpp:202-218).
template <int R>
__device__ __forceinline__ void bwd_epilogue(const BwdParams& p, float (&g)[R][4], const float* xs, uint32_t u0,
                                             int lane, uint64_t pol) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t u = u0 + r;
        if (u >= p.r1) break;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t c = lane + 32 * k;
            if (c >= p.din) break;
            float val = g[r][k];
            if (p.gcn2) {
                float* d0 = p.dh0 + size_t(u) * p.dh0stride + c;
                val = __fadd_rn(__fmul_rn(p.omb, xs[c * R + r]), __fmul_rn(p.beta, val));
                st1_stream(d0, __fadd_rn(ld1_stream(d0, pol), __fmul_rn(p.alpha, val)), pol);
                val = __fmul_rn(p.oma, val);
            }
            st1_stream(p.bg + size_t(u) * p.bgstride + c, val, pol);
        }
    }
}

// ---------------------------------------------------------------------------
// Forward of one layer over rows [r0, r1) (kernel::forward_row nn.hpp:159-197):
// gather (or dropped own row for Dense) -> GCNII initial-residual mix -> pre ->
// b + pre.W (the reference's exact-zero skip is an identity here: pre is never
// -0 and x*W = +-0 leaves a non -0 accumulator unchanged) -> identity mix ->
// ReLU -> h, and the next layer's dropped gather source. SPLIT: stop at pre
// (k_fwd_tile in dense_tile.cuh does the transform).
// ---------------------------------------------------------------------------
// Resident CTAs per SM the split (gather-only) kernels are compiled for: no
// staged matrix, so registers alone bound their occupancy.
#ifndef GP_SPLIT_MINB
#define GP_SPLIT_MINB 4
#endif
// MINB > 0 overrides the resident-CTA target of the launch bounds (the split
// kernels are also built for 5 CTAs / 48 registers: better for large launches).
template <int KIND, int NB, bool SPLIT = false, int MINB = 0>
__global__ void __launch_bounds__(kBlock, MINB ? MINB : (SPLIT && NB == 2 ? GP_SPLIT_MINB : (NB == 2 ? 4 : (NB == 4 ? 3 : 2))))
    k_fwd8(FwdParams p) {
    extern __shared__ float4 smem4[];
    const uint32_t ms = mat_stride(p.dout);
    float* Ms = reinterpret_cast<float*>(reinterpret_cast<char*>(smem4) + kEdgeSlotBytes);
    float* bs = Ms + size_t(p.din) * ms + 32;
    float* xs = bs + 128 + (threadIdx.x / 32) * 256;
    if (!SPLIT) {
        stage_mat(Ms, p.W, p.din, p.dout, false, p.dout);
        for (uint32_t c = threadIdx.x; c < 128; c += blockDim.x) bs[c] = (p.bias && c < p.dout) ? p.bias[c] : 0.f;
        __syncthreads();
    }
    const uint64_t pol = evict_first_policy();
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const bool in_act = uint32_t(8 * hl) < p.din;
    for (;;) {
        // dynamic row-pair scheduling: no static tail across a ~6-pair-per-warp launch
        uint32_t pair = 0;
        if (lane == 0) pair = atomicAdd(p.ticket, 1u);
        pair = __shfl_sync(kFull, pair, 0);
        const uint32_t base = p.r0 + 2 * pair;
        if (base >= p.r1) break;
        const uint32_t v = base + (hb ? 1u : 0u);
        const bool has = v < p.r1;
        F8 pre;
        if (KIND == FWD_DENSE) {
            const F8 x = (has && in_act) ? ld8_stream(p.xsrc + size_t(v) * p.xstride + 8 * hl) : f8_zero();
            pre = drop8(p.in_mask, has ? p.orig[v] : 0u, 8 * hl, p.din, x);
        } else if (KIND == FWD_SAGE) {
            // pre = [drop(x_v) | mean over neighbours of drop(x_u)] (nn.hpp:176-182); the own row
            // is the current gather-table row (v's chunk is done), the mean half starts at sgap
            const F8 own = (has && in_act) ? ld8_stream(p.gsrc + size_t(v) * p.gstride + 8 * hl) : f8_zero();
            uint2* es = reinterpret_cast<uint2*>(smem4) + (threadIdx.x / 32) * 32;
            const F8 z = p.gsnap ? gather_row8<false, true, NB>(p.rowptr_m, p.edges_m, v, has, p.gsrc, p.gsnap,
                                                                p.gstride, p.done, lane, in_act, es, f8_zero())
                                 : gather_row8<false, false, NB>(p.rowptr_m, p.edges_m, v, has, p.gsrc, nullptr,
                                                                 p.gstride, p.done, lane, in_act, es, f8_zero());
            if (has && in_act) {
                st8_stream(p.pre + size_t(v) * p.prestride + 8 * hl, own);
                st8_stream(p.pre + size_t(v) * p.prestride + p.sgap + 8 * hl, z);
            }
            continue;  // SageConv runs split: transform in k_fwd_tile (gapped weights)
        } else {
            // "cur if the neighbour's chunk is done, else snapshot" (engines_impl.hpp:740-744); with
            // one (merged) table, gsnap == null and the per-entry table choice is skipped
            uint2* es = reinterpret_cast<uint2*>(smem4) + (threadIdx.x / 32) * 32;
            const F8 z = p.gsnap ? gather_row8<false, true, NB>(p.rowptr, p.edges, v, has, p.gsrc, p.gsnap, p.gstride,
                                                                p.done, lane, in_act, es, f8_zero())
                                 : gather_row8<false, false, NB>(p.rowptr, p.edges, v, has, p.gsrc, nullptr, p.gstride,
                                                                 p.done, lane, in_act, es, f8_zero());
            if (KIND == FWD_GCN2) {
                const F8 h = (has && in_act) ? ld8_stream(p.h0 + size_t(v) * p.h0stride + 8 * hl) : f8_zero();
#pragma unroll
                for (int c = 0; c < 8; ++c) pre.v[c] = __fadd_rn(__fmul_rn(p.oma, z.v[c]), __fmul_rn(p.alpha, h.v[c]));
            } else {
                pre = z;
            }
        }
        if (has && in_act) st8_stream(p.pre + size_t(v) * p.prestride + 8 * hl, pre);
        if (SPLIT) continue;  // transform + epilogue in k_fwd_tile (dense_tile.cuh)

        stage_x2(xs, pre, hl, hb, in_act);
        float o[2][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[0][k] = o[1][k] = bs[(lane + 32 * k) & 127];
        gemv_w<2>(o, xs, Ms, p.din, ms, lane);
        fwd_epilogue<2, KIND == FWD_GCN2>(p, o, xs, base, lane, pol);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Fused backward step (see k_bwd in kernels.cuh for the semantics): incoming
// gradient of layer i (dtop | drop_{i+1}(A_hat . bg_{i+1}) over done chunks |
// drop_{i+1}(bg_{i+1}[u])) (+ dh0 at global layer 0), then backward_out_row of
// layer i (nn.hpp:202-218): dz, dagg = dz.W^T, GCNII mixes, dh0 += a*dagg, and
// bg_i = (1-a)*dagg (Gcn2Conv) or dagg. SPLIT: stop at dz (k_bwd_tile does the rest).
// ---------------------------------------------------------------------------
template <int PREV, int OUT, int NB, bool SPLIT = false, int MINB = 0>
__global__ void __launch_bounds__(kBlock, MINB ? MINB : (SPLIT && NB == 2 ? GP_SPLIT_MINB : (NB == 2 ? 4 : (NB == 4 ? 3 : 2))))
    k_bwd8(BwdParams p) {
    extern __shared__ float4 smem4[];
    const uint32_t ms = mat_stride(p.din);
    float* Ms = reinterpret_cast<float*>(reinterpret_cast<char*>(smem4) + kEdgeSlotBytes);
    float* xs = Ms + size_t(p.dout) * ms + 32 + 128 + (threadIdx.x / 32) * 256;
    if (!SPLIT && OUT == OUT_LAYER && p.need_dagg) {
        stage_mat(Ms, p.W, p.dout, p.din, true, p.dout);  // Ms[j][c] = W[c][j]
        __syncthreads();
    }
    const uint64_t pol = evict_first_policy();
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const bool dh_act = uint32_t(8 * hl) < p.dh_width;
    for (;;) {
        // dynamic row-pair scheduling: no static tail across a ~6-pair-per-warp launch
        uint32_t pair = 0;
        if (lane == 0) pair = atomicAdd(p.ticket, 1u);
        pair = __shfl_sync(kFull, pair, 0);
        const uint32_t base = p.r0 + 2 * pair;
        if (base >= p.r1) break;
        const uint32_t u = base + (hb ? 1u : 0u);
        const bool has = u < p.r1;
        F8 dh;
        if (PREV == PREV_TOP) {
            dh = (has && dh_act) ? ld8_stream(p.dtop + size_t(u) * p.dtopstride + 8 * hl) : f8_zero();
        } else {
            F8 s;
            if (PREV == PREV_OWN) {
                s = (has && dh_act) ? ld8_stream(p.bgn + size_t(u) * p.bgnstride + 8 * hl) : f8_zero();
            } else if (PREV == PREV_SAGE || PREV == PREV_SAGE_HIST) {
                // SageConv backward_prev_row (nn.hpp:234-243): own half of dagg, then the done
                // neighbours' aggregated halves weighted 1/deg(v), ascending
                const F8 own = (has && dh_act) ? ld8_stream(p.bgn + size_t(u) * p.bgnstride + 8 * hl) : f8_zero();
                s = gather_row8<true, PREV == PREV_SAGE_HIST, NB>(
                    p.rowptr_m, p.edges_m, u, has, p.bgn + p.sgap, p.bgn_snap ? p.bgn_snap + p.sgap : nullptr,
                    p.bgnstride, p.done, lane, dh_act, reinterpret_cast<uint2*>(smem4) + (threadIdx.x / 32) * 32, own);
            } else {
                s = gather_row8<PREV != PREV_AGG_ALL, PREV == PREV_AGG_HIST, NB>(p.rowptr, p.edges, u, has, p.bgn,
                                                                              p.bgn_snap, p.bgnstride,
                                                             p.done, lane, dh_act,
                                                             reinterpret_cast<uint2*>(smem4) + (threadIdx.x / 32) * 32,
                                                             f8_zero());
            }
            dh = drop8(p.prev_mask, has ? p.orig[u] : 0u, 8 * hl, p.dh_width, s);
        }
        if (OUT == OUT_DHIN) {
            if (has && dh_act) st8_stream(p.dh_in + size_t(u) * p.dhinstride + 8 * hl, dh);
            continue;
        }
        if (p.dh0_add && has && dh_act) {
            const F8 a = ld8_stream(p.dh0_add + size_t(u) * p.dh0stride + 8 * hl);
#pragma unroll
            for (int c = 0; c < 8; ++c) dh.v[c] = __fadd_rn(dh.v[c], a.v[c]);
        }
        F8 dz = dh;
        if (p.relu) {
            const F8 h = (has && dh_act) ? ld8_stream(p.h + size_t(u) * p.hstride + 8 * hl) : f8_zero();
#pragma unroll
            for (int c = 0; c < 8; ++c) dz.v[c] = h.v[c] > 0.f ? dh.v[c] : 0.f;
        }
        if (has && dh_act) st8_stream(p.dz + size_t(u) * p.dzstride + 8 * hl, dz);
        if (SPLIT || !p.need_dagg) continue;  // dz.W^T in k_bwd_tile (dense_tile.cuh)
        stage_x2(xs, dz, hl, hb, dh_act);
        float g[2][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[0][k] = g[1][k] = 0.f;
        gemv_w<2>(g, xs, Ms, p.dout, ms, lane);
        bwd_epilogue<2>(p, g, xs, base, lane, pol);
        __syncwarp();
    }
}

}  // namespace gp

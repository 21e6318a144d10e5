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

// NB = gathers in flight per lane (x 2 rows per warp), a template parameter.

// Sum over the CSR row of w * src[col] (8 columns per lane). FILTER drops
// entries of not-yet-done chunks (stable ballot compaction per 16-entry batch);
// HIST reads those from `snap` instead. Padding slots use weight 0 and keep the
// previous registers: acc starts at +0 and never becomes -0, so acc + 0*x == acc.
template <bool FILTER, bool HIST, int NB>
__device__ __forceinline__ F8 gather_row8(const uint64_t* __restrict__ rowptr, const uint2* __restrict__ edges,
                                          uint32_t v, bool has_row, const float* __restrict__ src,
                                          const float* __restrict__ snap, uint32_t stride, uint64_t done,
                                          int lane, bool active) {
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
    // padding slots re-read this half's own row (the self-loop row: distinct per
    // half-warp, so padding never concentrates on one L2 line)
    const float* lpad = ls + size_t(has_row ? v : 0u) * stride;
    F8 acc = f8_zero();
    // CSR batch of the next iteration is loaded one batch ahead
    uint2 nxt = hl < int(min(16u, n_my)) ? ld_edge(edges + e0 + hl) : make_uint2(0u, 0u);
    for (uint32_t off = 0; off < n_max; off += 16) {
        int cnt = n_my > off ? int(min(16u, n_my - off)) : 0;
        uint2 my = nxt;
        {
            const uint32_t noff = off + 16;
            const int ncnt = n_my > noff ? int(min(16u, n_my - noff)) : 0;
            nxt = hl < ncnt ? ld_edge(edges + e0 + noff + hl) : make_uint2(0u, 0u);
        }
        if (FILTER && !HIST) {
            const bool ok = hl < cnt && ((done >> (my.x >> kColBits)) & 1ull);
            const unsigned m = (__ballot_sync(kFull, ok) >> hb) & 0xffffu;
            cnt = __popc(m);
            const int from = hl < cnt ? int(__fns(m, 0, hl + 1)) : 0;
            my.x = __shfl_sync(kFull, my.x, hb + from);
            my.y = __shfl_sync(kFull, my.y, hb + from);
        }
        const int cmax = max(cnt, __shfl_xor_sync(kFull, cnt, 16));
        for (int t = 0; t < cmax; t += NB) {
            float w[NB];
            F8 x[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int tt = t + i;
                const int sl = hb + (tt & 15);
                const uint32_t packed = __shfl_sync(kFull, my.x, sl);
                const float wv = __uint_as_float(__shfl_sync(kFull, my.y, sl));
                const bool valid = tt < cnt;
                const float* s = ls;
                if (HIST && !((done >> (packed >> kColBits)) & 1ull)) s = lsn;
                w[i] = valid ? wv : 0.f;
                x[i] = ld8_gather(valid ? s + size_t(packed & kColMask) * stride : lpad);
            }
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc.v[c] = mul_add(acc.v[c], w[i], x[i].v[c]);
        }
    }
    return acc;
}

// Weight staging: row i of an (rows x cols) matrix is stored as 2*cols8 float4
// slots, slot (part, h) = part * cols8 + h holding columns 8h+4part..8h+4part+3,
// so the two LDS.128 of a half-warp are each 256 contiguous bytes.
__device__ __forceinline__ void stage_w8(float* Ws, const float* W, uint32_t rows, uint32_t cols, bool transpose,
                                         uint32_t ld) {
    const uint32_t c8 = (cols + 7) / 8;
    for (uint32_t idx = threadIdx.x; idx < rows * c8 * 8; idx += blockDim.x) {
        const uint32_t r = idx / (c8 * 8), c = idx % (c8 * 8);
        const uint32_t h = c / 8, part = (c % 8) / 4, q = c % 4;
        float val = 0.f;
        if (c < cols) val = transpose ? W[size_t(c) * ld + r] : W[size_t(r) * ld + c];
        Ws[(size_t(r) * 2 * c8 + part * c8 + h) * 4 + q] = val;
    }
}

__device__ __forceinline__ void w8_row(const float4* Ws4, uint32_t r, uint32_t c8, int hl, float4& a, float4& b) {
    a = Ws4[size_t(r) * 2 * c8 + hl];
    b = Ws4[size_t(r) * 2 * c8 + c8 + hl];
}

// Row-local GEMV: o[c] += sum_i x_i * M[i][c] over i ascending (x held 8 per
// lane across the half-warp), one rounded mul and add per term.
__device__ __forceinline__ void gemv8(F8& o, const F8& x, const float4* Ws4, uint32_t rows, uint32_t c8, int hl,
                                      int hb) {
    const uint32_t r8 = (rows + 7) / 8;
    for (uint32_t ib = 0; ib < r8; ++ib) {
        const F8 xb = shfl8(x, hb + int(ib));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t i = 8 * ib + q;
            if (i < rows) {
                float4 a, b;
                w8_row(Ws4, i, c8, hl, a, b);
                const float xi = xb.v[q];
                o.v[0] = mul_add(o.v[0], xi, a.x);
                o.v[1] = mul_add(o.v[1], xi, a.y);
                o.v[2] = mul_add(o.v[2], xi, a.z);
                o.v[3] = mul_add(o.v[3], xi, a.w);
                o.v[4] = mul_add(o.v[4], xi, b.x);
                o.v[5] = mul_add(o.v[5], xi, b.y);
                o.v[6] = mul_add(o.v[6], xi, b.z);
                o.v[7] = mul_add(o.v[7], xi, b.w);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Forward of one layer over rows [r0, r1) (kernel::forward_row nn.hpp:159-197):
// gather (or dropped own row for Dense) -> GCNII initial-residual mix -> pre ->
// b + pre.W (the reference's exact-zero skip is an identity here: pre is never
// -0 and x*W = +-0 leaves a non -0 accumulator unchanged) -> identity mix ->
// ReLU -> h, and the next layer's dropped gather source.
// ---------------------------------------------------------------------------
template <int KIND, int NB>
__global__ void __launch_bounds__(kBlock, NB == 2 ? 4 : (NB == 4 ? 3 : 2)) k_fwd8(FwdParams p) {
    extern __shared__ float4 smem4[];
    const uint32_t c8 = (p.dout + 7) / 8;
    float* Ws = reinterpret_cast<float*>(smem4);
    stage_w8(Ws, p.W, p.din, p.dout, false, p.dout);
    float* bs = Ws + size_t(p.din) * c8 * 8;
    for (uint32_t c = threadIdx.x; c < c8 * 8; c += blockDim.x) {
        const uint32_t h = c / 8, part = (c % 8) / 4, q = c % 4;
        bs[(part * c8 + h) * 4 + q] = (p.bias && c < p.dout) ? p.bias[c] : 0.f;
    }
    __syncthreads();
    const float4* Ws4 = reinterpret_cast<const float4*>(Ws);
    const float4* bs4 = reinterpret_cast<const float4*>(bs);

    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const bool in_act = uint32_t(8 * hl) < p.din;
    const bool out_act = uint32_t(8 * hl) < p.dout;
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
        } else {
            const F8 z = gather_row8<false, false, NB>(p.rowptr, p.edges, v, has, p.gsrc, nullptr, p.gstride, 0ull, lane,
                                                   in_act);
            if (KIND == FWD_GCN2) {
                const F8 h = (has && in_act) ? ld8_stream(p.h0 + size_t(v) * p.h0stride + 8 * hl) : f8_zero();
#pragma unroll
                for (int c = 0; c < 8; ++c) pre.v[c] = __fadd_rn(__fmul_rn(p.oma, z.v[c]), __fmul_rn(p.alpha, h.v[c]));
            } else {
                pre = z;
            }
        }
        if (has && in_act) st8_stream(p.pre + size_t(v) * p.prestride + 8 * hl, pre);

        F8 o;
        {
            const float4 a = bs4[hl < int(c8) ? hl : 0], b = bs4[c8 + (hl < int(c8) ? hl : 0)];
            o.v[0] = a.x, o.v[1] = a.y, o.v[2] = a.z, o.v[3] = a.w;
            o.v[4] = b.x, o.v[5] = b.y, o.v[6] = b.z, o.v[7] = b.w;
        }
        gemv8(o, pre, Ws4, p.din, c8, hl < int(c8) ? hl : 0, hb);
        if (KIND == FWD_GCN2) {
#pragma unroll
            for (int c = 0; c < 8; ++c) o.v[c] = __fadd_rn(__fmul_rn(p.omb, pre.v[c]), __fmul_rn(p.beta, o.v[c]));
        }
        if (p.relu) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (o.v[c] < 0.f) o.v[c] = 0.f;
        }
        if (has && out_act) {
            st8_stream(p.out + size_t(v) * p.outstride + 8 * hl, o);
            if (p.gnext)
                st8_stream(p.gnext + size_t(v) * p.gnstride + 8 * hl, drop8(p.next_mask, p.orig[v], 8 * hl, p.dout, o));
        }
    }
}

// ---------------------------------------------------------------------------
// Fused backward step (see k_bwd in kernels.cuh for the semantics): incoming
// gradient of layer i (dtop | drop_{i+1}(A_hat . bg_{i+1}) over done chunks |
// drop_{i+1}(bg_{i+1}[u])) (+ dh0 at global layer 0), then backward_out_row of
// layer i (nn.hpp:202-218): dz, dagg = dz.W^T, GCNII mixes, dh0 += a*dagg, and
// bg_i = (1-a)*dagg (Gcn2Conv) or dagg.
// ---------------------------------------------------------------------------
template <int PREV, int OUT, int NB>
__global__ void __launch_bounds__(kBlock, NB == 2 ? 4 : (NB == 4 ? 3 : 2)) k_bwd8(BwdParams p) {
    extern __shared__ float4 smem4[];
    float* Wt = reinterpret_cast<float*>(smem4);
    const uint32_t c8 = (p.din + 7) / 8;
    if (OUT == OUT_LAYER && p.need_dagg) {
        stage_w8(Wt, p.W, p.dout, p.din, true, p.dout);  // Wt[j][c] = W[c][j]
        __syncthreads();
    }
    const float4* Wt4 = reinterpret_cast<const float4*>(Wt);
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const bool dh_act = uint32_t(8 * hl) < p.dh_width;
    const bool in_act = uint32_t(8 * hl) < p.din;
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
            if (PREV == PREV_OWN)
                s = (has && dh_act) ? ld8_stream(p.bgn + size_t(u) * p.bgnstride + 8 * hl) : f8_zero();
            else
                s = gather_row8<true, PREV == PREV_AGG_HIST, NB>(p.rowptr, p.edges, u, has, p.bgn, p.bgn_snap, p.bgnstride,
                                                             p.done, lane, dh_act);
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
        if (!p.need_dagg) continue;
        F8 g = f8_zero();
        gemv8(g, dz, Wt4, p.dout, c8, hl < int(c8) ? hl : 0, hb);
        if (!(has && in_act)) continue;
        if (p.gcn2) {
            float* d0 = p.dh0 + size_t(u) * p.dh0stride + 8 * hl;
            F8 a = ld8_stream(d0);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                g.v[c] = __fadd_rn(__fmul_rn(p.omb, dz.v[c]), __fmul_rn(p.beta, g.v[c]));
                a.v[c] = __fadd_rn(a.v[c], __fmul_rn(p.alpha, g.v[c]));
                g.v[c] = __fmul_rn(p.oma, g.v[c]);
            }
            st8_stream(d0, a);
        }
        st8_stream(p.bg + size_t(u) * p.bgstride + 8 * hl, g);
    }
}

}  // namespace gp

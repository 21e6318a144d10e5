// Register-tiled row transforms for the split row path (gather kernel writes
// pre / dz, these apply the weight matrix and the epilogue).
//
// The transform of a chunk is a skinny GEMM (rows x din) . (din x dout) with
// din, dout <= 128, but it must stay bit-identical to the reference's scalar
// loops: out[v][c] = b[c] + sum_i pre[v][i] * W[i][c] in ascending i with one
// rounded multiply and one rounded add per term (dense_rows matrix.hpp:63-74;
// dense_rows_wt :77-86 for the backward). No tensor-core accumulation can
// reproduce that rounding sequence, so this is an FP32 CUDA-core kernel whose
// floor is 2 FP instructions per MAC (ptxas contracts any packed f32x2
// mul/add pair into FFMA2, so the packed forms are not usable either).
//
// Tiling: a thread owns 4 rows x 8 columns (32 accumulators). Per 4 input
// indices it reads 4 x 4 row values (four LDS.128 from the row tile As[r][i]) and
// 4 x 8 matrix values (eight LDS.128 from Ws[i][c]): 12 shared loads per 256 FP
// instructions, so the kernel is FP-issue bound, not shared-memory bound like the
// 2-rows-per-warp GEMV fused into the gather kernel. A CTA of 256 threads covers
// ceil(dout/8) column groups x floor(256 / groups) row groups (dout = 100: 13 x
// 19 -> 76 rows per tile); tiles are handed out grid-stride and double-buffered
// with cp.async, so the next tile's rows stream in under the current tile's math.
#pragma once

#include "kernels.cuh"

namespace gp {

constexpr int kTileThreads = 256;

struct TileGeom {
    uint32_t ncg;  // column groups of 8
    uint32_t nrg;  // row groups (a thread owns rows rg + r nrg, r < TR)
    uint32_t tm;   // rows per tile = TR * nrg
    uint32_t kp;   // contraction length padded to 4 (zero rows of Ws, zero columns of As)
    uint32_t ams;  // As row stride (floats): kp + 4
    uint32_t ms;   // Ws row stride (floats): 8 * ncg + 4 per 4 column groups (see ws_col)
};

// Column group cg starts at 8 cg + 4 (cg / 4) in a Ws row: the 16-byte slots the
// 13 (dout = 100) groups read in one LDS.128 are then distinct modulo 8 within
// groups 0-7 and 8-15, so a warp's matrix read costs the minimum 2 wavefronts
// instead of the 4 that 8-float-aligned groups (banks repeating every 4 groups)
// would.
__host__ __device__ constexpr uint32_t ws_col(uint32_t cg) { return 8u * cg + 4u * (cg >> 2); }

__host__ __device__ inline TileGeom tile_geom(uint32_t width_in, uint32_t width_out, uint32_t tr) {
    TileGeom g;
    g.ncg = (width_out + 7u) / 8u;
    g.nrg = kTileThreads / g.ncg;
    g.tm = tr * g.nrg;
    g.kp = (width_in + 3u) & ~3u;
    g.ams = g.kp + 4u;
    g.ms = ws_col(g.ncg - 1) + 8u;
    return g;
}

// Ws + bias + two row-tile buffers (double-buffered cp.async)
__host__ __device__ inline size_t tile_smem_bytes(uint32_t width_in, uint32_t width_out, uint32_t tr) {
    const TileGeom g = tile_geom(width_in, width_out, tr);
    return (size_t(g.kp) * g.ms + 128 + 2 * size_t(g.tm) * g.ams) * 4;
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(ok ? 16u : 0u)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(ok ? 4u : 0u)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ float4 ld4_hint(const float* p, uint64_t pol) {
    float4 a;
    asm("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
        : "l"(p), "l"(pol));
    return a;
}

// Asynchronously copy rows [v0, v0+tm) x columns [0, kp) of src (row stride ld,
// a multiple of 8 floats, so every 16-byte piece is aligned) into As[r][k]; rows
// past r1 are zero-filled. Does not commit.
__device__ __forceinline__ void stage_rows_async(float* As, const float* src, uint32_t ld, uint32_t v0, uint32_t r1,
                                                 const TileGeom& g) {
    const uint32_t k4 = g.kp / 4u;
    uint32_t r = threadIdx.x / k4, q = threadIdx.x % k4;
    const uint32_t dr = kTileThreads / k4, dq = kTileThreads % k4;
    for (uint32_t idx = threadIdx.x; idx < g.tm * k4; idx += kTileThreads) {
        const bool ok = v0 + r < r1;
        cp_async16(As + size_t(r) * g.ams + 4 * q, ok ? src + size_t(v0 + r) * ld + 4 * q : src, ok);
        r += dr;
        q += dq;
        if (q >= k4) q -= k4, ++r;
    }
}

// Asynchronously stage the row-major (rows x cols) matrix M (leading dimension
// cols) as Ws[i][ws_col(c / 8) + c % 8] for i < kp, zero padded, all copies in
// flight at once: 16-byte pieces when cols % 4 == 0 (every piece is then either
// inside the matrix or padding), 4-byte copies otherwise. Does not commit.
__device__ __forceinline__ void stage_w_async(float* Ws, const float* M, uint32_t rows, uint32_t cols,
                                              const TileGeom& g) {
    const uint32_t w8 = 8u * g.ncg;
    if ((cols & 3u) == 0) {
        const uint32_t w4 = w8 / 4u;
        for (uint32_t idx = threadIdx.x; idx < g.kp * w4; idx += kTileThreads) {
            const uint32_t i = idx / w4, c = 4u * (idx % w4);
            const bool ok = i < rows && c < cols;
            cp_async16(Ws + size_t(i) * g.ms + ws_col(c >> 3) + (c & 7u), ok ? M + size_t(i) * cols + c : M, ok);
        }
        return;
    }
    for (uint32_t idx = threadIdx.x; idx < g.kp * w8; idx += kTileThreads) {
        const uint32_t i = idx / w8, c = idx % w8;
        const bool ok = i < rows && c < cols;
        cp_async4(Ws + size_t(i) * g.ms + ws_col(c >> 3) + (c & 7u), ok ? M + size_t(i) * cols + c : M, ok);
    }
}

// WT = W^T for the backward transform's staging (W is rows x cols row-major).
__global__ void k_transpose(const float* __restrict__ W, float* __restrict__ WT, uint32_t rows, uint32_t cols) {
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < rows * cols; idx += gridDim.x * blockDim.x) {
        const uint32_t j = idx / rows, c = idx % rows;
        WT[idx] = W[size_t(c) * cols + j];
    }
}

// acc[r][j] (+)= sum_i As[rg + r nrg][i] * Ws[i][8cg + j], ascending i, mul and
// add rounded separately. The zero padding of i up to kp adds +0 products, which
// leave the (never -0) accumulators unchanged. Rows of a thread are nrg apart, so
// the ~3 row groups of a warp read consecutive As rows (ams = 26 slots mod 8:
// conflict-free).
template <int TR>
__device__ __forceinline__ void tile_mac(float (&acc)[TR][8], const float* __restrict__ As,
                                         const float* __restrict__ Ws, const TileGeom& g, uint32_t rg,
                                         uint32_t cg) {
    const float* a = As + size_t(rg) * g.ams;
    const float* w = Ws + ws_col(cg);
    const uint32_t ra = g.nrg * g.ams, ms = g.ms;
#pragma unroll 1
    for (uint32_t i = 0; i < g.kp; i += 4, a += 4, w += 4 * ms) {
        float4 x[TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) x[r] = *reinterpret_cast<const float4*>(a + r * ra);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const float4 w0 = *reinterpret_cast<const float4*>(w + kk * ms);
            const float4 w1 = *reinterpret_cast<const float4*>(w + kk * ms + 4);
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const float xv = f4_get(x[r], kk);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] = mul_add(acc[r][j], xv, wv[j]);
            }
        }
    }
}

// tile_mac with the geometry of a square WIDTH x WIDTH transform fixed at compile
// time (the model widths the engine specialises for: H = 100, 128), so every
// shared-memory offset inside a k-group is an immediate and no index arithmetic
// is issued between the loads and the FP pipe. Same arithmetic order as tile_mac.
template <int TR, int WIDTH>
__device__ __forceinline__ void tile_mac_fixed(float (&acc)[TR][8], const float* __restrict__ As,
                                               const float* __restrict__ Ws, uint32_t rg, uint32_t cg) {
    constexpr uint32_t kNcg = (WIDTH + 7) / 8, kNrg = kTileThreads / kNcg, kKp = (WIDTH + 3) & ~3;
    constexpr uint32_t kAms = kKp + 4, kMs = ws_col(kNcg - 1) + 8, kRa = kNrg * kAms;
    const float* a = As + size_t(rg) * kAms;
    const float* w = Ws + ws_col(cg);
#pragma unroll 1  // unrolling 2 or 5 k-groups measured within 2 %
    for (uint32_t i = 0; i < kKp; i += 4, a += 4, w += 4 * kMs) {
        float4 x[TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) x[r] = *reinterpret_cast<const float4*>(a + r * kRa);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const float4 w0 = *reinterpret_cast<const float4*>(w + kk * kMs);
            const float4 w1 = *reinterpret_cast<const float4*>(w + kk * kMs + 4);
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const float xv = f4_get(x[r], kk);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] = mul_add(acc[r][j], xv, wv[j]);
            }
        }
    }
}

template <int TR, int WIDTH>
__device__ __forceinline__ void tile_mac_any(float (&acc)[TR][8], const float* __restrict__ As,
                                             const float* __restrict__ Ws, const TileGeom& g, uint32_t rg,
                                             uint32_t cg) {
    if constexpr (WIDTH != 0) tile_mac_fixed<TR, WIDTH>(acc, As, Ws, rg, cg);
    else tile_mac<TR>(acc, As, Ws, g, rg, cg);
}

__device__ __forceinline__ void st8_hint(float* p, const float (&x)[8], uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(x[0]),
                 "f"(x[1]), "f"(x[2]), "f"(x[3]), "l"(pol)
                 : "memory");
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p + 4), "f"(x[4]),
                 "f"(x[5]), "f"(x[6]), "f"(x[7]), "l"(pol)
                 : "memory");
}

// Rows per thread for a launch of `rows` rows: 4 (most reuse of each staged
// matrix row) unless that leaves fewer than ~half the SMs with a tile. Measured at
// Reddit shape (tools/fwd_bench.cu): 4 rows per thread is fastest down to 96
// tiles (K = 32 chunks), 1.3x faster than 1 row per thread there.
__host__ inline int tile_rows_per_thread(uint32_t rows, uint32_t width_out, int num_sms) {
    for (int tr = 4; tr > 1; tr /= 2) {
        const uint32_t tm = tile_geom(0, width_out, tr).tm;
        if ((rows + tm - 1) / tm >= uint32_t(num_sms) / 2u) return tr;
    }
    return 1;
}

// ---------------------------------------------------------------------------
// Forward transform + epilogue (kernel::forward_row nn.hpp:185-196) of rows
// [r0, r1) whose pre was written by k_fwd8<KIND, NB, true>: out = b + pre.W,
// Gcn2Conv out = (1-beta) pre + beta out, ReLU, h, and the next layer's dropped
// gather row. Padding columns (c >= dout, up to the 8-float row stride) are
// written as the zeros they already hold.
// ---------------------------------------------------------------------------
// WIDTH != 0: din == dout == WIDTH (host-checked), compile-time geometry.
template <bool GCN2, int TR, int WIDTH = 0>
__global__ void __launch_bounds__(kTileThreads, 2) k_fwd_tile(FwdParams p) {
    extern __shared__ float4 smem4[];
    const TileGeom g = tile_geom(p.din, p.dout, TR);
    float* Ws = reinterpret_cast<float*>(smem4);
    float* bs = Ws + size_t(g.kp) * g.ms;
    float* Ab = bs + 128;
    const uint32_t ntiles = (p.r1 - p.r0 + g.tm - 1) / g.tm;
    uint32_t t = blockIdx.x;
    stage_w_async(Ws, p.W, p.din, p.dout, g);
    if (t < ntiles) stage_rows_async(Ab, p.pre, p.prestride, p.r0 + t * g.tm, p.r1, g);
    cp_async_commit();
    for (uint32_t c = threadIdx.x; c < 128; c += kTileThreads) bs[c] = (p.bias && c < p.dout) ? p.bias[c] : 0.f;
    const uint64_t pol = evict_first_policy();
    const uint32_t cg = threadIdx.x % g.ncg, rg = threadIdx.x / g.ncg;
    const bool act = rg < g.nrg;
    for (uint32_t it = 0; t < ntiles; t += gridDim.x, ++it) {
        const float* As = Ab + size_t(it & 1) * g.tm * g.ams;
        // prefetch the next tile into the other buffer (empty group if none)
        const uint32_t tn = t + gridDim.x;
        if (tn < ntiles) stage_rows_async(Ab + size_t((it + 1) & 1) * g.tm * g.ams, p.pre, p.prestride,
                                          p.r0 + tn * g.tm, p.r1, g);
        cp_async_commit();
        cp_async_wait_1();
        __syncthreads();
        if (act) {
            const uint32_t v0 = p.r0 + t * g.tm;
            uint32_t vo[TR];  // original ids for the next layer's dropout, loaded before the math
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const uint32_t v = v0 + rg + r * g.nrg;
                vo[r] = (p.gnext && v < p.r1) ? p.orig[v] : 0u;
            }
            float acc[TR][8];
#pragma unroll
            for (int r = 0; r < TR; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] = bs[8 * cg + j];
            tile_mac_any<TR, WIDTH>(acc, As, Ws, g, rg, cg);
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const uint32_t lr = rg + r * g.nrg, v = v0 + lr;
                if (v >= p.r1) break;
                float o[8], gn[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t c = 8 * cg + j;
                    float val = 0.f;
                    if (c < p.dout) {
                        val = acc[r][j];
                        if (GCN2) val = __fadd_rn(__fmul_rn(p.omb, As[lr * g.ams + c]), __fmul_rn(p.beta, val));
                        if (p.relu && val < 0.f) val = 0.f;
                    }
                    o[j] = val;
                    gn[j] = (p.gnext && c < p.dout) ? drop_apply(p.next_mask, vo[r], c, val) : 0.f;
                }
                st8_hint(p.out + size_t(v) * p.outstride + 8 * cg, o, pol);
                if (p.gnext) st8_hint(p.gnext + size_t(v) * p.gnstride + 8 * cg, gn, pol);
            }
        }
        __syncthreads();  // this buffer is refilled by the next iteration's prefetch
    }
}

// ---------------------------------------------------------------------------
// Backward transform + epilogue (kernel::backward_out_row nn.hpp:202-218) of
// rows whose dz was written by k_bwd8<PREV, OUT_LAYER, NB, true>:
// dagg = dz.W^T; Gcn2Conv: dagg = (1-beta) dz + beta dagg, dh0 += alpha dagg,
// bg = (1-alpha) dagg; otherwise bg = dagg.
// ---------------------------------------------------------------------------
template <int TR, int WIDTH = 0>
__global__ void __launch_bounds__(kTileThreads, 2) k_bwd_tile(BwdParams p) {
    extern __shared__ float4 smem4[];
    const TileGeom g = tile_geom(p.dout, p.din, TR);
    float* Ws = reinterpret_cast<float*>(smem4);
    float* Ab = Ws + size_t(g.kp) * g.ms + 128;
    const uint32_t ntiles = (p.r1 - p.r0 + g.tm - 1) / g.tm;
    uint32_t t = blockIdx.x;
    stage_w_async(Ws, p.WT, p.dout, p.din, g);  // Ws[j][c] = W[c][j]
    if (t < ntiles) stage_rows_async(Ab, p.dz, p.dzstride, p.r0 + t * g.tm, p.r1, g);
    cp_async_commit();
    const uint64_t pol = evict_first_policy();
    const uint32_t cg = threadIdx.x % g.ncg, rg = threadIdx.x / g.ncg;
    const bool act = rg < g.nrg;
    for (uint32_t it = 0; t < ntiles; t += gridDim.x, ++it) {
        const float* As = Ab + size_t(it & 1) * g.tm * g.ams;
        const uint32_t tn = t + gridDim.x;
        if (tn < ntiles) stage_rows_async(Ab + size_t((it + 1) & 1) * g.tm * g.ams, p.dz, p.dzstride,
                                          p.r0 + tn * g.tm, p.r1, g);
        cp_async_commit();
        cp_async_wait_1();
        __syncthreads();
        if (act) {
            const uint32_t u0 = p.r0 + t * g.tm;
            float acc[TR][8];
#pragma unroll
            for (int r = 0; r < TR; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
            tile_mac_any<TR, WIDTH>(acc, As, Ws, g, rg, cg);
            // dh0 rows of the tile, all in flight before the epilogue consumes them
            float4 d0v[TR][2];
            if (p.gcn2) {
#pragma unroll
                for (int r = 0; r < TR; ++r) {
                    const uint32_t u = u0 + rg + r * g.nrg;
                    const float* d0 = p.dh0 + size_t(u < p.r1 ? u : u0) * p.dh0stride + 8 * cg;
                    d0v[r][0] = ld4_hint(d0, pol);
                    d0v[r][1] = ld4_hint(d0 + 4, pol);
                }
            }
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const uint32_t lr = rg + r * g.nrg, u = u0 + lr;
                if (u >= p.r1) break;
                float o[8];
                if (p.gcn2) {
                    float d[8] = {d0v[r][0].x, d0v[r][0].y, d0v[r][0].z, d0v[r][0].w,
                                  d0v[r][1].x, d0v[r][1].y, d0v[r][1].z, d0v[r][1].w};
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t c = 8 * cg + j;
                        float val = 0.f;
                        if (c < p.din) {
                            val = __fadd_rn(__fmul_rn(p.omb, As[lr * g.ams + c]), __fmul_rn(p.beta, acc[r][j]));
                            d[j] = __fadd_rn(d[j], __fmul_rn(p.alpha, val));
                            val = __fmul_rn(p.oma, val);
                        }
                        o[j] = val;
                    }
                    st8_hint(p.dh0 + size_t(u) * p.dh0stride + 8 * cg, d, pol);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) o[j] = 8 * cg + j < p.din ? acc[r][j] : 0.f;
                }
                st8_hint(p.bg + size_t(u) * p.bgstride + 8 * cg, o, pol);
            }
        }
        __syncthreads();
    }
}

}  // namespace gp

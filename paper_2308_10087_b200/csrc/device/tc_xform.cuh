// Row transforms of the aggregating layers on the 5th-generation tensor cores
// (tcgen05, accumulator in TMEM, weights brought in by the TMA bulk-copy engine).
//
// forward  (kernel::forward_row, nn.hpp:183-196):  out = act(pre . W' + b), then h and
//          the next layer's dropped gather row; Gcn2Conv folds its identity mix into the
//          operand, W' = beta W + (1 - beta) I, so out = (1-beta) pre + beta pre.W in one GEMM
//          (mix = 1: B = W and the epilogue mixes from the unsplit pre row instead)
// backward (kernel::backward_out_row, nn.hpp:202-218): D = dz . W'^T with the same fold
//          (dagg = (1-beta) dz + beta dz.W^T); Gcn2Conv: dh0 += alpha D, bg = (1-alpha) D;
//          otherwise bg = D
//
// GEMM shape per launch: M = the chunk's rows (tiles of 128), N = out width padded to
// 16 (<= 128), K = in width padded to 8 (<= 128). Precision: kind::tf32 with the 3xTF32
// split x = hi + lo on both operands (D += a_hi b_hi + a_hi b_lo + a_lo b_hi): fp32-level
// results, not the reference's bit pattern (its per-term rounding sequence is scalar);
// GP_TC_XFORM=0 selects the bit-exact CUDA-core kernels (dense_tile.cuh).
//
// Data movement per CTA (persistent over 128-row tiles, one CTA per SM):
//   * the prepared operand B = [hi | lo] of W' (k_tc_prep, canonical K-major
//     SWIZZLE_NONE core-matrix layout, <= 128 KB) lands in shared memory once, by two
//     cp.async.bulk copies completing on an mbarrier (TMA engine, no thread involved);
//   * A streams in K-chunks of 32 columns: coalesced 16-byte global loads (8 threads
//     per row), hi/lo split in registers, stored into the core-matrix layout; two
//     stage buffers, the loads of chunk g+1 in flight while chunk g is multiplied;
//   * one elected thread issues the MMAs; two TMEM accumulators (2 x npad columns), so
//     the epilogue of tile j-1 (8 warps: TMEM lane quarter = warp % 4, column half =
//     warp / 4) overlaps the MMAs of tile j.
#pragma once

#include "tc_pgrad.cuh"
#include "kernels.cuh"

namespace gp {

constexpr int kXfThreads = 256;
constexpr int kXfM = 128;   // rows per tile (MMA M)
constexpr int kXfKc = 32;   // K columns per A stage

struct TcXformParams {
    uint32_t r0, r1;
    const float* A;  // pre (forward) / dz (backward), row stride astride
    uint32_t astride;
    uint32_t kdim, kpad;  // contraction width and its padding to 8
    uint32_t ndim, npad;  // output width and its padding to 16
    uint32_t ostride;     // padded row stride of the outputs (pad8(ndim))
    const float* Bop;     // k_tc_prep output: hi block then lo block, kpad * npad floats each
    const float* bias;    // forward bias or null
    uint32_t relu;
    // forward epilogue
    float* out;
    float* out2;  // optional second copy of out (the next epoch's snapshot, lean layout) or null
    float* gnext;
    uint32_t gnstride;
    DropKey next_mask;
    const uint32_t* orig;
    // backward epilogue
    uint32_t gcn2;
    float alpha, oma;
    float* dh0;
    uint32_t dh0stride;
    float* bg;
    // mix = 1 (Gcn2Conv, GP_TC_MIX=1): B holds W itself and the epilogue applies the identity
    // mix in fp32 from the unsplit input row, out = omb * A + beta * (A.W) (the reference's own
    // expression, nn.hpp:188-190 / :207-209), so only the small beta term carries the TF32
    // split error; mix = 0 (default): the mix is folded into B (W' = beta W + (1 - beta) I)
    uint32_t mix;
    float mbeta, momb;
    uint32_t a_lbo;  // A stage k-core stride in bytes: kXfLboDense or kXfLboPad
};

__host__ __device__ constexpr uint32_t xf_pad16(uint32_t x) { return (x + 15u) & ~15u; }
__host__ __device__ constexpr uint32_t xf_pad8k(uint32_t x) { return (x + 7u) & ~7u; }

constexpr uint32_t kXfSmemMax = 200 * 1024;
#ifndef GP_XF_PF
#define GP_XF_PF 3
#endif
// A chunks in flight per thread (K = 32 epoch: 3 -> 0.397-0.400 s, 2 -> 0.400-0.406, 1 -> 0.414-0.420;
// no difference at K = 4; profiles/r2b_xform_prefetch_ab.txt)
constexpr int kXfPf = GP_XF_PF;  // H = 128: 128 + 64 KB

// shared memory: B hi/lo + 2 stages x (A hi, A lo) of 128 x 32 tf32 + bias
// (measured alternatives, Reddit shape, per K = 4 backward launch: this version 59 us;
// two chunks of A in flight in registers, 59 us; a 2-6 deep cp.async raw ring with the
// epilogue's dh0 rows prefetched across the chunk loop, 88 us)
// A stage k-core stride (p.a_lbo): the dense 16 row groups (kXfLboDense), or + 16 bytes
// (kXfLboPad). A 128-bit shared store is served a quarter-warp at a time; the 8 lanes of a
// quarter hold one row's 8 k-cores, which with the dense stride all start in the same 16-byte
// bank group (8-way conflict, 32 wavefronts per warp store). An odd multiple of 16 bytes per
// k-core puts them in 8 different groups (4 wavefronts, the minimum for 512 bytes): forward
// 17.0-18.7 vs 19.2 ms, backward 13.1 vs 15.0 ms per K = 4 epoch, 46.9 / 38.4 vs 51.2 / 42.6 ms at
// K = 32; epoch -1 % at both. GP_XF_PAD=0 restores the dense stride (bitwise equal).
constexpr uint32_t kXfLboDense = (kXfM / 8) * 128;
constexpr uint32_t kXfLboPad = kXfLboDense + 16;
constexpr uint32_t kXfAbytes = kXfLboPad * (kXfKc / 4);  // stage buffer of one of hi / lo (max)
__host__ __device__ inline size_t xf_smem_bytes(uint32_t kpad, uint32_t npad) {
    return size_t(2) * kpad * npad * 4 + size_t(2) * 2 * kXfAbytes + 128 * 4;
}

// Prepared operand of W' (B[n][k], K-major core matrices): element (n, k) of the hi
// (lo) block at float offset (k/4) * npad*4 + (n/8) * 32 + (n%8) * 4 + k%4, i.e.
// [k-core][n-group][8 rows][4], LBO = npad/8 * 128 bytes, SBO = 128 bytes.
//   forward : B[n][k] = W'[k][n], W (kdim x ndim) row-major
//   backward: B[n][k] = W'[n][k], W (ndim x kdim) row-major (dagg = dz . W^T)
// W' = beta W + (1 - beta) I for Gcn2Conv (square), else W; zero padding.
__global__ void k_tc_prep(const float* __restrict__ W, uint32_t kdim, uint32_t ndim, uint32_t kpad, uint32_t npad,
                          uint32_t backward, uint32_t gcn2, float beta, float omb, float* __restrict__ out) {
    const uint32_t total = kpad * npad;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const uint32_t n = idx / kpad, k = idx % kpad;
        float w = 0.f;
        if (n < ndim && k < kdim) {
            w = backward ? W[size_t(n) * kdim + k] : W[size_t(k) * ndim + n];
            if (gcn2) w = __fadd_rn(__fmul_rn(beta, w), n == k ? omb : 0.f);
        }
        const float hi = to_tf32(w), lo = to_tf32(__fsub_rn(w, hi));
        const size_t off = size_t(k >> 2) * npad * 4 + (n >> 3) * 32 + (n & 7) * 4 + (k & 3);
        out[off] = hi;
        out[size_t(total) + off] = lo;
    }
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void st_v4_ef(float* p, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(a), "f"(b),
                 "f"(c), "f"(d), "l"(pol)
                 : "memory");
}

template <bool BWD>
__global__ void __launch_bounds__(kXfThreads, 1) k_tc_xform(TcXformParams p) {
    extern __shared__ __align__(1024) uint8_t xsm[];
    __shared__ __align__(8) uint64_t bars[5];  // 0,1: A stages free; 2,3: accumulators ready; 4: B loaded
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t kpad = p.kpad, npad = p.npad;
    const uint32_t b_bytes = kpad * npad * 4;
    uint8_t* b_hi = xsm;
    uint8_t* b_lo = xsm + b_bytes;
    uint8_t* a_base = xsm + 2 * b_bytes;
    const uint32_t a_lbo = p.a_lbo, a_bytes = a_lbo * (kXfKc / 4);
    float* bias_sh = reinterpret_cast<float*>(a_base + 4 * a_bytes);
    const uint32_t ntiles = (p.r1 - p.r0 + kXfM - 1) / kXfM;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint32_t nchunks = (kpad + kXfKc - 1) / kXfKc;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 5; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (uint32_t c = tid; c < 128; c += kXfThreads) bias_sh[c] = (p.bias && c < p.ndim) ? p.bias[c] : 0.f;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    if (tid == 0 && my_tiles > 0) {  // W' hi / lo through the TMA bulk-copy engine
        mbar_expect_tx(&bars[4], 2 * b_bytes);
        bulk_g2s(b_hi, p.Bop, b_bytes, &bars[4]);
        bulk_g2s(b_lo, reinterpret_cast<const uint8_t*>(p.Bop) + b_bytes, b_bytes, &bars[4]);
    }
    const uint32_t idesc = umma_idesc_tf32(kXfM, npad);
    const uint32_t b_lbo = (npad / 8) * 128;
    const uint64_t pol = evict_first_policy();

    // A staging: thread handles float4 items idx = tid + 256 e (e < 4): row m = idx / 8,
    // k-core kc = idx % 8 of the chunk (8 threads read one row's 128 contiguous bytes)
    // kXfPf A chunks in flight per thread: a register ring over the flattened (tile, chunk)
    // sequence, statically indexed by unrolling the chunk loop kXfPf times
    float4 ring[kXfPf][4];
    auto load_chunk = [&](float4 (&reg)[4], uint32_t tile, uint32_t c) {
        const uint32_t row0 = p.r0 + tile * kXfM, k0 = c * kXfKc;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t idx = tid + kXfThreads * e, m = idx >> 3, kc = idx & 7;
            const uint32_t v = row0 + m, k = k0 + 4 * kc;
            reg[e] = (v < p.r1 && k < p.kdim) ? *reinterpret_cast<const float4*>(p.A + size_t(v) * p.astride + k)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_chunk = [&](const float4 (&reg)[4], uint32_t st) {
        uint8_t* hi = a_base + st * 2 * a_bytes;
        uint8_t* lo = hi + a_bytes;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t idx = tid + kXfThreads * e, m = idx >> 3, kc = idx & 7;
            const float x[4] = {reg[e].x, reg[e].y, reg[e].z, reg[e].w};
            float h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                h[q] = to_tf32(x[q]);
                l[q] = to_tf32(__fsub_rn(x[q], h[q]));
            }
            const uint32_t off = kc * a_lbo + (m >> 3) * 128 + (m & 7) * 16;
            *reinterpret_cast<float4*>(hi + off) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(lo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
    };

    // epilogue of local tile j (accumulator j & 1): TMEM lanes 32 (warp % 4) .. +31 are
    // rows, columns [half * npad / 2, (half + 1) * npad / 2) in groups of 8
    auto epilogue = [&](uint32_t j) {
        const uint32_t acc = j & 1;
        mbar_wait(&bars[2 + acc], (j >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tile = blockIdx.x + j * gridDim.x;
        const uint32_t q = warp & 3, half = warp >> 2;
        const uint32_t row = 32 * q + lane, v = p.r0 + tile * kXfM + row;
        const bool valid = v < p.r1;
        const uint32_t vo = (!BWD && p.gnext && valid) ? p.orig[v] : 0u;
        const uint32_t cw = npad / 2;
        for (uint32_t c0 = half * cw; c0 < (half + 1) * cw; c0 += 8) {
            float a[8];
            tmem_ld8(tmem + ((32u * q) << 16) + acc * npad + c0, a);
            if (!valid || c0 >= p.ostride) continue;
            float o[8];
            float x[8];  // mix: the unsplit input row (pre / dz) at these columns (square layer)
            if (p.mix) {
                const float* xr = p.A + size_t(v) * p.astride + c0;
                const float4 x0 = *reinterpret_cast<const float4*>(xr), x1 = *reinterpret_cast<const float4*>(xr + 4);
                x[0] = x0.x, x[1] = x0.y, x[2] = x0.z, x[3] = x0.w, x[4] = x1.x, x[5] = x1.y, x[6] = x1.z, x[7] = x1.w;
                if (BWD)
#pragma unroll
                    for (int i = 0; i < 8; ++i) a[i] = __fadd_rn(__fmul_rn(p.momb, x[i]), __fmul_rn(p.mbeta, a[i]));
            }
            if (!BWD) {
                float g[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t c = c0 + i;
                    float val = 0.f;
                    if (c < p.ndim) {
                        val = __fadd_rn(a[i], bias_sh[c]);
                        if (p.mix) val = __fadd_rn(__fmul_rn(p.momb, x[i]), __fmul_rn(p.mbeta, val));
                        if (p.relu && val < 0.f) val = 0.f;
                    }
                    o[i] = val;
                    g[i] = (p.gnext && c < p.ndim) ? drop_apply(p.next_mask, vo, c, val) : 0.f;
                }
                float* dst = p.out + size_t(v) * p.ostride + c0;
                st_v4_ef(dst, o[0], o[1], o[2], o[3], pol);
                st_v4_ef(dst + 4, o[4], o[5], o[6], o[7], pol);
                if (p.out2) {
                    float* d2 = p.out2 + size_t(v) * p.ostride + c0;
                    st_v4_ef(d2, o[0], o[1], o[2], o[3], pol);
                    st_v4_ef(d2 + 4, o[4], o[5], o[6], o[7], pol);
                }
                if (p.gnext) {
                    float* gd = p.gnext + size_t(v) * p.gnstride + c0;
                    st_v4_ef(gd, g[0], g[1], g[2], g[3], pol);
                    st_v4_ef(gd + 4, g[4], g[5], g[6], g[7], pol);
                }
            } else {
                if (p.gcn2) {
                    float* d0 = p.dh0 + size_t(v) * p.dh0stride + c0;
                    float4 x0 = *reinterpret_cast<const float4*>(d0), x1 = *reinterpret_cast<const float4*>(d0 + 4);
                    float d[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const bool in = c0 + i < p.ndim;
                        d[i] = in ? __fadd_rn(d[i], __fmul_rn(p.alpha, a[i])) : d[i];
                        o[i] = in ? __fmul_rn(p.oma, a[i]) : 0.f;
                    }
                    st_v4_ef(d0, d[0], d[1], d[2], d[3], pol);
                    st_v4_ef(d0 + 4, d[4], d[5], d[6], d[7], pol);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) o[i] = c0 + i < p.ndim ? a[i] : 0.f;
                }
                float* dst = p.bg + size_t(v) * p.ostride + c0;
                st_v4_ef(dst, o[0], o[1], o[2], o[3], pol);
                st_v4_ef(dst + 4, o[4], o[5], o[6], o[7], pol);
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    const uint32_t total = my_tiles * nchunks;  // A chunks this CTA stages (stage = g & 1)
    auto chunk_at = [&](float4 (&reg)[4], uint32_t g) { load_chunk(reg, blockIdx.x + (g / nchunks) * gridDim.x, g % nchunks); };
#pragma unroll
    for (int u = 0; u < kXfPf; ++u)
        if (uint32_t(u) < total) chunk_at(ring[u], u);
    for (uint32_t g0 = 0; g0 < total; g0 += kXfPf) {
#pragma unroll
        for (int u = 0; u < kXfPf; ++u) {
            const uint32_t g = g0 + u;
            if (g >= total) break;
            const uint32_t j = g / nchunks, c = g % nchunks, acc = j & 1;
            const uint32_t st = g & 1;
            if (g >= 2) mbar_wait(&bars[st], ((g >> 1) - 1) & 1);  // the MMAs that read this stage are done
            store_chunk(ring[u], st);
            if (g + kXfPf < total) chunk_at(ring[u], g + kXfPf);  // refill the slot kXfPf chunks ahead
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                if (g == 0) mbar_wait(&bars[4], 0);  // W' resident
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint8_t* ah = a_base + st * 2 * a_bytes;
                const uint32_t sah = smem_u32(ah), sal = smem_u32(ah + a_bytes);
                const uint32_t sbh = smem_u32(b_hi), sbl = smem_u32(b_lo);
                const uint32_t ksteps = min(uint32_t(kXfKc), kpad - c * kXfKc) / 8;
                const uint32_t d = tmem + acc * npad;
                for (uint32_t s = 0; s < ksteps; ++s) {
                    const uint32_t kcore = c * (kXfKc / 4) + 2 * s;  // B k-core of this k-step
                    const uint64_t dah = umma_desc(sah + 2 * s * a_lbo, a_lbo, 128);
                    const uint64_t dal = umma_desc(sal + 2 * s * a_lbo, a_lbo, 128);
                    const uint64_t dbh = umma_desc(sbh + kcore * b_lbo, b_lbo, 128);
                    const uint64_t dbl = umma_desc(sbl + kcore * b_lbo, b_lbo, 128);
                    const uint32_t accum = (c == 0 && s == 0) ? 0u : 1u;
                    mma_tf32(d, dah, dbh, idesc, accum);
                    mma_tf32(d, dah, dbl, idesc, 1u);
                    mma_tf32(d, dal, dbh, idesc, 1u);
                }
                umma_commit(&bars[st]);
                if (c + 1 == nchunks) umma_commit(&bars[2 + acc]);  // tile j's accumulator is complete
            }
            if (c + 1 == nchunks && j > 0) epilogue(j - 1);  // overlaps tile j's MMAs
        }
    }
    if (my_tiles > 0) epilogue(my_tiles - 1);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// The whole optimizer step of a stage's GCN / GCNII / Dense layers in one launch
// (Optimizer::step nn.hpp:456-467 per parameter, then the derived copies the next epoch
// reads): per weight element the same Adam (or SGD) arithmetic as k_adam, then W^T
// (k_transpose) and, for tcgen05 layers, the element's hi / lo entries of the prepared
// forward and backward operands (k_tc_prep; their zero padding was written by the first
// k_tc_prep and never changes). blockIdx.y = layer; bias elements follow the weights.
struct StepLayer {
    float *W, *gW, *mW, *vW, *WT;
    float *b, *gb, *mb, *vb;
    float *xf_fwd, *xf_bwd;  // null: not a tcgen05 layer
    uint32_t din, dout, g2;
    float beta, omb;
};

__global__ void __launch_bounds__(256) k_param_step(const StepLayer* __restrict__ layers, AdamParams a) {
    const StepLayer L = layers[blockIdx.y];
    const uint32_t nw = L.din * L.dout, nb = L.b ? L.dout : 0u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nw + nb; i += gridDim.x * blockDim.x) {
        const bool isw = i < nw;
        const uint32_t e = isw ? i : i - nw;
        float* P = isw ? L.W : L.b;
        const float g = (isw ? L.gW : L.gb)[e];
        float w;
        if (a.sgd) {
            w = __fsub_rn(P[e], __fmul_rn(a.lr, g));
        } else {
            float* M = isw ? L.mW : L.mb;
            float* V = isw ? L.vW : L.vb;
            const float m = __fadd_rn(__fmul_rn(a.b1, M[e]), __fmul_rn(a.omb1, g));
            const float v = __fadd_rn(__fmul_rn(a.b2, V[e]), __fmul_rn(__fmul_rn(a.omb2, g), g));
            M[e] = m;
            V[e] = v;
            const float mhat = __fdiv_rn(m, a.c1);
            const float vhat = __fdiv_rn(v, a.c2);
            w = __fsub_rn(P[e], __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
        }
        P[e] = w;
        if (!isw) continue;
        const uint32_t r = e / L.dout, c = e % L.dout;  // W[r][c], r < din, c < dout
        L.WT[size_t(c) * L.din + r] = w;
        if (!L.xf_fwd) continue;
        // forward operand: B[n = c][k = r] = W'[r][c] (kpad = pad8(din), npad = pad16(dout));
        // backward: B[n = r][k = c] = W'[r][c] (kpad = pad8(dout), npad = pad16(din))
        const float wp = L.g2 ? __fadd_rn(__fmul_rn(L.beta, w), r == c ? L.omb : 0.f) : w;
        const float hi = to_tf32(wp), lo = to_tf32(__fsub_rn(wp, hi));
        const uint32_t kpf = xf_pad8k(L.din), npf = xf_pad16(L.dout);
        const size_t of = size_t(r >> 2) * npf * 4 + (c >> 3) * 32 + (c & 7) * 4 + (r & 3);
        L.xf_fwd[of] = hi;
        L.xf_fwd[size_t(kpf) * npf + of] = lo;
        const uint32_t kpb = xf_pad8k(L.dout), npb = xf_pad16(L.din);
        const size_t ob = size_t(c >> 2) * npb * 4 + (r >> 3) * 32 + (r & 7) * 4 + (c & 3);
        L.xf_bwd[ob] = hi;
        L.xf_bwd[size_t(kpb) * npb + ob] = lo;
    }
}

}  // namespace gp

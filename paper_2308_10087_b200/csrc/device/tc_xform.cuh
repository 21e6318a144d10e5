// Row transforms of the aggregating layers on the 5th-generation tensor cores
// (tcgen05, accumulator in TMEM, weights brought in by the TMA bulk-copy engine).
//
// forward  (kernel::forward_row, nn.hpp:183-196):  out = act(pre . W' + b), then h and
//          the next layer's dropped gather row; Gcn2Conv folds its identity mix into the
//          operand, W' = beta W + (1 - beta) I, so out = (1-beta) pre + beta pre.W in one GEMM
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
//   * A streams in K-chunks of 32 columns: coalesced 16-byte cp.async copies (8 threads
//     per row) into a raw ring 2-6 chunks deep (16 KB each, as many as shared memory
//     holds next to W'), hi/lo split from the ring into the core-matrix layout of two
//     stage buffers while earlier chunks are multiplied;
//   * one elected thread issues the MMAs; two TMEM accumulators (2 x npad columns), so
//     the epilogue of tile j-1 (8 warps: TMEM lane quarter = warp % 4, column half =
//     warp / 4) overlaps the MMAs of tile j; its dh0 rows (backward) and vertex ids
//     are loaded before tile j's chunk loop, four tcgen05.ld per wait.
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
};

__host__ __device__ constexpr uint32_t xf_pad16(uint32_t x) { return (x + 15u) & ~15u; }
__host__ __device__ constexpr uint32_t xf_pad8k(uint32_t x) { return (x + 7u) & ~7u; }

constexpr uint32_t kXfRawBytes = kXfM * kXfKc * 4;  // one raw fp32 A chunk (16 KB)
constexpr uint32_t kXfSmemMax = 224 * 1024;  // + 2 KB static, under the 227 KB opt-in

// raw A chunks in flight: as many as fit next to W' and the hi/lo stages (2..6)
__host__ __device__ inline uint32_t xf_raw_stages(uint32_t kpad, uint32_t npad) {
    const size_t fixed = size_t(2) * kpad * npad * 4 + size_t(2) * 2 * kXfM * kXfKc * 4;
    const size_t room = fixed < kXfSmemMax ? (kXfSmemMax - fixed) / kXfRawBytes : 0;
    return uint32_t(room < 2 ? 2 : (room > 6 ? 6 : room));
}

// dynamic shared memory: B hi/lo + 2 stages x (A hi, A lo) of 128 x 32 tf32 + the raw ring
// (H = 128: 128 + 64 + 32 KB = the 224 KB cap; the bias lives in static shared memory)
__host__ __device__ inline size_t xf_smem_bytes(uint32_t kpad, uint32_t npad) {
    return size_t(2) * kpad * npad * 4 + size_t(2) * 2 * kXfM * kXfKc * 4 +
           size_t(xf_raw_stages(kpad, npad)) * kXfRawBytes;
}

__device__ __forceinline__ void cp_async16_zfill(void* dst, const float* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16u : 0u)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_xf() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_xf() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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

// 8 columns of this warp's 32 TMEM lanes; completes at tmem_ld_wait()
__device__ __forceinline__ void tmem_ld8_async(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float4 ld4_ef(const float* p, uint64_t pol) {
    float4 a;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                 : "l"(p), "l"(pol));
    return a;
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
    constexpr uint32_t a_bytes = kXfM * kXfKc * 4;  // one of hi / lo of one stage
    const uint32_t raw_stages = xf_raw_stages(kpad, npad);
    uint8_t* raw = a_base + 4 * a_bytes;  // raw_stages x [128 rows][32 fp32]
    __shared__ float bias_sh[128];
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
    const uint32_t a_lbo = (kXfM / 8) * 128, b_lbo = (npad / 8) * 128;
    const uint64_t pol = evict_first_policy();

    // A staging: thread handles float4 items idx = tid + 256 e (e < 4): row m = idx / 8,
    // k-core kc = idx % 8 of the chunk (8 threads read one row's 128 contiguous bytes).
    // Chunks are numbered g = j * nchunks + c over this CTA's tiles. cp.async copies each
    // chunk's raw fp32 into a ring of raw_stages slots, raw_stages - 1 chunks ahead (no
    // registers held); a thread converts exactly the items it copied, so its own
    // wait_group is the only synchronisation the ring needs.
    const uint32_t total_chunks = my_tiles * nchunks;
    auto issue_chunk = [&](uint32_t gg) {
        if (gg < total_chunks) {
            const uint32_t tile = blockIdx.x + (gg / nchunks) * gridDim.x, c = gg % nchunks;
            const uint32_t row0 = p.r0 + tile * kXfM, k0 = c * kXfKc;
            uint8_t* slot = raw + (gg % raw_stages) * kXfRawBytes;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t idx = tid + kXfThreads * e, m = idx >> 3, kc = idx & 7;
                const uint32_t v = row0 + m, k = k0 + 4 * kc;
                const bool ok = v < p.r1 && k < p.kdim;
                cp_async16_zfill(slot + m * 128 + kc * 16, ok ? p.A + size_t(v) * p.astride + k : p.A, ok);
            }
        }
        cp_async_commit_xf();  // one group per chunk index (empty past the end)
    };
    auto store_chunk = [&](uint32_t gg, uint32_t st) {
        const uint8_t* slot = raw + (gg % raw_stages) * kXfRawBytes;
        uint8_t* hi = a_base + st * 2 * a_bytes;
        uint8_t* lo = hi + a_bytes;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t idx = tid + kXfThreads * e, m = idx >> 3, kc = idx & 7;
            const float4 r = *reinterpret_cast<const float4*>(slot + m * 128 + kc * 16);
            const float x[4] = {r.x, r.y, r.z, r.w};
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

    // Epilogue inputs of tile j, loaded while tile j+1's chunks stream in (held across the
    // chunk loop): the thread's row id and, backward Gcn2Conv, its dh0 columns
    constexpr int kMaxGroups = 8;  // npad / 2 <= 64 columns per thread
    float4 dpre[kMaxGroups][2];
    uint32_t vo_pre = 0;
    auto prefetch_epilogue = [&](uint32_t j) {
        const uint32_t tile = blockIdx.x + j * gridDim.x;
        const uint32_t q = warp & 3, half = warp >> 2;
        const uint32_t v = p.r0 + tile * kXfM + 32 * q + lane;
        const bool valid = v < p.r1;
        vo_pre = (!BWD && p.gnext && valid) ? p.orig[v] : 0u;
        if (BWD && p.gcn2) {
            const uint32_t cw = npad / 2, cbeg = half * cw, cend = min(cbeg + cw, p.ostride);
#pragma unroll
            for (int gi = 0; gi < kMaxGroups; ++gi) {
                const uint32_t c0 = cbeg + 8 * gi;
                if (valid && c0 < cend) {
                    const float* src = p.dh0 + size_t(v) * p.dh0stride + c0;
                    dpre[gi][0] = ld4_ef(src, pol);
                    dpre[gi][1] = ld4_ef(src + 4, pol);
                }
            }
        }
    };

    // epilogue of local tile j (accumulator j & 1): TMEM lanes 32 (warp % 4) .. +31 are
    // rows, columns [half * npad / 2, (half + 1) * npad / 2) in passes of up to 4 groups of
    // 8: the pass's global loads (dh0) and TMEM loads are all issued before one wait
    auto epilogue = [&](uint32_t j) {
        const uint32_t acc = j & 1;
        mbar_wait(&bars[2 + acc], (j >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tile = blockIdx.x + j * gridDim.x;
        const uint32_t q = warp & 3, half = warp >> 2;
        const uint32_t row = 32 * q + lane, v = p.r0 + tile * kXfM + row;
        const bool valid = v < p.r1;
        const uint32_t vo = vo_pre;
        const uint32_t cw = npad / 2, cbeg = half * cw, cend = min(cbeg + cw, p.ostride);
        const uint32_t taddr = tmem + ((32u * q) << 16) + acc * npad;
#pragma unroll
        for (int pass = 0; pass < kMaxGroups / 4; ++pass) {
            const uint32_t c1 = cbeg + 32 * pass;
            if (c1 >= cbeg + cw) break;
            uint32_t a[4][8];
#pragma unroll
            for (int gi = 0; gi < 4; ++gi) {
                const uint32_t c0 = c1 + 8 * gi;
                if (c0 < cbeg + cw) tmem_ld8_async(taddr + c0, a[gi]);  // warp-uniform
            }
            tmem_ld_wait();
            if (!valid) continue;
#pragma unroll
            for (int gi = 0; gi < 4; ++gi) {
                const uint32_t c0 = c1 + 8 * gi;
                const float4(&d0g)[2] = dpre[4 * pass + gi];
                if (c0 >= cend) break;
                float o[8];
                if (!BWD) {
                    float gn[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t c = c0 + i;
                        float val = 0.f;
                        if (c < p.ndim) {
                            val = __fadd_rn(__uint_as_float(a[gi][i]), bias_sh[c]);
                            if (p.relu && val < 0.f) val = 0.f;
                        }
                        o[i] = val;
                        gn[i] = (p.gnext && c < p.ndim) ? drop_apply(p.next_mask, vo, c, val) : 0.f;
                    }
                    float* dst = p.out + size_t(v) * p.ostride + c0;
                    st_v4_ef(dst, o[0], o[1], o[2], o[3], pol);
                    st_v4_ef(dst + 4, o[4], o[5], o[6], o[7], pol);
                    if (p.gnext) {
                        float* gd = p.gnext + size_t(v) * p.gnstride + c0;
                        st_v4_ef(gd, gn[0], gn[1], gn[2], gn[3], pol);
                        st_v4_ef(gd + 4, gn[4], gn[5], gn[6], gn[7], pol);
                    }
                } else {
                    if (p.gcn2) {
                        float d[8] = {d0g[0].x, d0g[0].y, d0g[0].z, d0g[0].w,
                                      d0g[1].x, d0g[1].y, d0g[1].z, d0g[1].w};
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const bool in = c0 + i < p.ndim;
                            const float av = __uint_as_float(a[gi][i]);
                            d[i] = in ? __fadd_rn(d[i], __fmul_rn(p.alpha, av)) : d[i];
                            o[i] = in ? __fmul_rn(p.oma, av) : 0.f;
                        }
                        float* dd = p.dh0 + size_t(v) * p.dh0stride + c0;
                        st_v4_ef(dd, d[0], d[1], d[2], d[3], pol);
                        st_v4_ef(dd + 4, d[4], d[5], d[6], d[7], pol);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) o[i] = c0 + i < p.ndim ? __uint_as_float(a[gi][i]) : 0.f;
                    }
                    float* dst = p.bg + size_t(v) * p.ostride + c0;
                    st_v4_ef(dst, o[0], o[1], o[2], o[3], pol);
                    st_v4_ef(dst + 4, o[4], o[5], o[6], o[7], pol);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    uint32_t g = 0;  // A chunks staged so far (stage = g & 1)
    for (uint32_t i = 0; i + 1 < raw_stages; ++i) issue_chunk(i);
    for (uint32_t j = 0; j < my_tiles; ++j) {
        const uint32_t acc = j & 1;
        if (j > 0) prefetch_epilogue(j - 1);
        for (uint32_t c = 0; c < nchunks; ++c, ++g) {
            const uint32_t st = g & 1;
            issue_chunk(g + raw_stages - 1);  // refills the slot chunk g-1 was converted from
            // this thread's copies of chunk g are complete once at most raw_stages - 1
            // younger groups are pending
            switch (raw_stages) {
                case 2: cp_async_wait_xf<1>(); break;
                case 3: cp_async_wait_xf<2>(); break;
                case 4: cp_async_wait_xf<3>(); break;
                case 5: cp_async_wait_xf<4>(); break;
                default: cp_async_wait_xf<5>(); break;
            }
            if (g >= 2) mbar_wait(&bars[st], ((g >> 1) - 1) & 1);  // the MMAs that read this stage are done
            store_chunk(g, st);
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
        }
        if (j > 0) epilogue(j - 1);  // overlaps tile j's MMAs
    }
    if (my_tiles > 0) {
        prefetch_epilogue(my_tiles - 1);
        epilogue(my_tiles - 1);
    }
    cp_async_wait_xf<0>();
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

}  // namespace gp

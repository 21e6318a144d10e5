// Parameter gradients on the 5th-generation tensor cores (tcgen05, TMEM).
//
// dW = pre^T . dz over all N rows (param_grads_for_rows, nn.hpp:269-293) is a GEMM
// with M = k_in (<= 128 per tile), N = out_dim (<= 128), K = rows (10^5..10^6),
// run split-K: each CTA reduces a contiguous row range into a 128 x N fp32
// accumulator that lives in TMEM, then writes it to the split workspace that
// k_pgrad_fold reduces in a fixed order (deterministic).
//
// Precision: kind::tf32 with the 3xTF32 split x = hi + lo (hi = rna_tf32(x),
// lo = rna_tf32(x - hi)); D += hi_a.hi_b + hi_a.lo_b + lo_a.hi_b keeps fp32-level
// accuracy (the dropped lo.lo term is ~2^-22 relative), so the tolerance bar of
// the CUDA-core version (rel 1e-4 vs the reference) is unchanged.
//
// Layout: both operands are staged K-major, SWIZZLE_NONE ("interleaved") in the
// canonical UMMA form ((8,m),(T,2)):((1T,SBO),(1,LBO)) with T = 16 bytes:
// core matrices of 8 rows x 4 tf32 (128 contiguous bytes); LBO = stride between
// the two K-adjacent cores an instruction consumes, SBO = stride between 8-row
// groups. Stage layout: [k-core c][row-group g][row r][4], so LBO = groups*128 B
// and SBO = 128 B; the k-step s of an instruction (K = 8) starts at core 2s.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gp {

constexpr int kTcThreads = 128;  // 4 warps: all load, warp 0 lane 0 issues MMAs
constexpr int kTcKt = 32;        // rows (K) per pipeline stage
constexpr int kTcM = 128;        // M tile (rows of dW)

struct TcPgradParams {
    uint32_t n, rows_per_split;
    const float* pre;
    uint32_t prestride;
    const float* dz;
    uint32_t dzstride;
    uint32_t din, dout;
    uint32_t npad;  // dout rounded up to 16 (MMA N)
    float* ws;      // splits x din x dout
    float* wsb;     // splits x dout (bias partials) or null
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3fff);
    d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
    d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
    d |= uint64_t(1) << 46;  // SM100 descriptor version
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) in bits [61,64)
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major.
__device__ __forceinline__ uint32_t umma_idesc_tf32(uint32_t M, uint32_t N) {
    uint32_t d = 0;
    d |= 1u << 4;         // c_format = F32
    d |= 2u << 7;         // a_format = TF32
    d |= 2u << 10;        // b_format = TF32
    d |= (N >> 3) << 17;  // n_dim
    d |= (M >> 4) << 24;  // m_dim
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

template <int NCOLS>
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Dynamic shared memory: 2 stages x {A_hi, A_lo (128 x 32), B_hi, B_lo (npad x 32)} tf32.
__global__ void __launch_bounds__(kTcThreads, 1) k_pgrad_tc(TcPgradParams p) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ __align__(8) uint64_t bars[3];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t split = blockIdx.x;
    const uint32_t i0 = blockIdx.y * kTcM;
    const uint32_t mvalid = min(uint32_t(kTcM), p.din - i0);
    const uint32_t rbeg = split * p.rows_per_split;
    const uint32_t rend = min(p.n, rbeg + p.rows_per_split);
    const uint32_t npad = p.npad;
    const uint32_t a_bytes = kTcM * kTcKt * 4, b_bytes = npad * kTcKt * 4;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    const uint32_t a_lbo = (kTcM / 8) * 128, b_lbo = (npad / 8) * 128;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    const uint32_t idesc = umma_idesc_tf32(kTcM, npad);

    float bsum = 0.f;
    const uint32_t nst = (rend > rbeg) ? (rend - rbeg + kTcKt - 1) / kTcKt : 0;
    uint32_t uses[2] = {0, 0};
    for (uint32_t it = 0; it < nst; ++it) {
        const uint32_t st = it & 1;
        if (uses[st] > 0) mbar_wait(&bars[st], (uses[st] - 1) & 1);  // MMAs that read this stage are done
        uint8_t* base = tsm + st * stage_bytes;
        float* a_hi = reinterpret_cast<float*>(base);
        float* a_lo = reinterpret_cast<float*>(base + a_bytes);
        float* b_hi = reinterpret_cast<float*>(base + 2 * a_bytes);
        float* b_lo = reinterpret_cast<float*>(base + 2 * a_bytes + b_bytes);
        const uint32_t r0 = rbeg + it * kTcKt;
        // A: thread m owns dW row i0+m; k-core c covers rows r0+4c..r0+4c+3
        {
            const uint32_t m = tid;
            const bool mok = m < mvalid;
#pragma unroll 2
            for (uint32_t c = 0; c < kTcKt / 4; ++c) {
                float hv[4], lv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t row = r0 + 4 * c + e;
                    const float x = (mok && row < rend) ? p.pre[size_t(row) * p.prestride + i0 + m] : 0.f;
                    hv[e] = to_tf32(x);
                    lv[e] = to_tf32(x - hv[e]);
                }
                const uint32_t off = c * a_lbo + (m >> 3) * 128 + (m & 7) * 16;
                *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(a_hi) + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
                *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(a_lo) + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
            }
        }
        // B: thread n owns dW column n
        if (uint32_t(tid) < npad) {
            const uint32_t nn = tid;
            const bool nok = nn < p.dout;
#pragma unroll 2
            for (uint32_t c = 0; c < kTcKt / 4; ++c) {
                float hv[4], lv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t row = r0 + 4 * c + e;
                    const float x = (nok && row < rend) ? p.dz[size_t(row) * p.dzstride + nn] : 0.f;
                    if (blockIdx.y == 0) bsum += x;
                    hv[e] = to_tf32(x);
                    lv[e] = to_tf32(x - hv[e]);
                }
                const uint32_t off = c * b_lbo + (nn >> 3) * 128 + (nn & 7) * 16;
                *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(b_hi) + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
                *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(b_lo) + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
            }
        }
        // generic-proxy smem writes -> visible to the tensor-core (async) proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
            for (uint32_t s = 0; s < kTcKt / 8; ++s) {
                const uint64_t dah = umma_desc(ah + 2 * s * a_lbo, a_lbo, 128);
                const uint64_t dal = umma_desc(al + 2 * s * a_lbo, a_lbo, 128);
                const uint64_t dbh = umma_desc(bh + 2 * s * b_lbo, b_lbo, 128);
                const uint64_t dbl = umma_desc(bl + 2 * s * b_lbo, b_lbo, 128);
                const uint32_t first = (it == 0 && s == 0) ? 0u : 1u;
                mma_tf32(tmem, dah, dbh, idesc, first);
                mma_tf32(tmem, dah, dbl, idesc, 1u);
                mma_tf32(tmem, dal, dbh, idesc, 1u);
            }
            umma_commit(&bars[st]);
        }
        ++uses[st];
    }
    // all MMAs done -> read the accumulator
    if (tid == 0) umma_commit(&bars[2]);
    if (nst > 0) mbar_wait(&bars[2], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    float* w = p.ws + size_t(split) * p.din * p.dout;
    const uint32_t m = 32 * warp + (tid & 31);
    for (uint32_t c0 = 0; c0 < npad; c0 += 16) {
        float v[16];
        tmem_ld16<16>(tmem + ((32u * warp) << 16) + c0, v);
        if (m < mvalid) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t n = c0 + j;
                if (n < p.dout) w[size_t(i0 + m) * p.dout + n] = nst > 0 ? v[j] : 0.f;
            }
        }
    }
    if (p.wsb && blockIdx.y == 0 && uint32_t(tid) < p.dout) p.wsb[size_t(split) * p.dout + tid] = bsum;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace gp

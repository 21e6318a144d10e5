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

constexpr int kTcThreads = 256;  // 8 warps stage operands; warps 0-3 read TMEM; one thread issues MMAs
constexpr int kTcKt = 32;        // rows (K) per pipeline stage
constexpr int kTcM = 128;        // M tile (rows of dW)
// Stage layout strides: 8-row core-matrix groups every kTcSbo = 144 bytes (128 + 16), so the
// 8 lanes of a quarter-warp, which write index quads q = 0..7 (indices 4q + j: group q / 2,
// row 4 (q & 1) + j), start in 8 different 16-byte bank groups: conflict-free 128-bit stores
// (with SBO = 128 they fell into 2 groups, a 4-way conflict on every stage store)
constexpr uint32_t kTcSbo = 144;
#ifndef GP_PGRAD_PF
#define GP_PGRAD_PF 2
#endif
constexpr int kTcPf = GP_PGRAD_PF;  // stages of operand loads in flight per thread
__host__ __device__ constexpr uint32_t tc_lbo(uint32_t rows) { return (rows / 8) * kTcSbo; }
__host__ __device__ constexpr size_t tc_pgrad_smem(uint32_t npad) {
    return size_t(2) * (2 * tc_lbo(kTcM) + 2 * tc_lbo(npad)) * (kTcKt / 4);
}

struct TcPgradParams {
    uint32_t n, rows_per_split;  // n = end row (exclusive); rows start at row0
    uint32_t row0;
    const float* pre;
    uint32_t prestride;
    const float* dz;
    uint32_t dzstride;
    uint32_t din, dout;
    uint32_t npad;  // dout rounded up to 16 (MMA N)
    float* ws;      // splits x din x dout
    float* wsb;     // splits x dout (bias partials) or null
    // row i of the reduction is stash row rows[i] (the own rows in ascending original
    // id, param_grads_for_rows' order, nn.hpp:269-293), so the sum order and the split
    // boundaries do not depend on the chunking; null: row i
    const uint32_t* rows;
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

// Staging work item: (4 consecutive M/N indices q, one k-core c = 4 rows). The
// thread loads 4 x float4 (rows r0+4c..+3, columns 4q..4q+3; coalesced across
// threads), transposes in registers, splits hi/lo and writes 4 x 16 B core-matrix
// rows (K-major). Loads for stage it+1 are issued before stage it's MMAs wait.
struct TcItem {
    float4 v[4];
};

__device__ __forceinline__ void tc_load(TcItem& it, const float* src, uint32_t stride, uint32_t col0,
                                        uint32_t cols_valid, uint32_t row0, uint32_t rend,
                                        const uint32_t* rows = nullptr) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t row = row0 + e;
        if (row < rend && col0 < cols_valid)
            it.v[e] = *reinterpret_cast<const float4*>(src + size_t(rows ? rows[row] : row) * stride + col0);
        else
            it.v[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Write the 4 (index) x 4 (k) block at core (c, q) of a K-major stage buffer.
__device__ __forceinline__ void tc_store(const TcItem& it, uint8_t* hi, uint8_t* lo, uint32_t lbo, uint32_t c,
                                         uint32_t q, uint32_t cols_valid, uint32_t col0, float* colsum) {
    const float t[4][4] = {{it.v[0].x, it.v[0].y, it.v[0].z, it.v[0].w},
                           {it.v[1].x, it.v[1].y, it.v[1].z, it.v[1].w},
                           {it.v[2].x, it.v[2].y, it.v[2].z, it.v[2].w},
                           {it.v[3].x, it.v[3].y, it.v[3].z, it.v[3].w}};
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // index 4q+j; its 4 k values are t[0..3][j]
        const uint32_t m = 4 * q + j;
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float x = (col0 + j < cols_valid) ? t[e][j] : 0.f;
            if (colsum) colsum[j] += x;
            h[e] = to_tf32(x);
            l[e] = to_tf32(x - h[e]);
        }
        const uint32_t off = c * lbo + (m >> 3) * kTcSbo + (m & 7) * 16;
        *reinterpret_cast<float4*>(hi + off) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(lo + off) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

// Dynamic shared memory: 2 stages x {A_hi, A_lo (128 x 32), B_hi, B_lo (npad x 32)} tf32.
__global__ void __launch_bounds__(kTcThreads, 1) k_pgrad_tc(TcPgradParams p) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ __align__(8) uint64_t bars[3];
    __shared__ uint32_t tmem_base_sh;
    __shared__ float bsum_sh[kTcThreads / 32][128];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t split = blockIdx.x;
    const uint32_t i0 = blockIdx.y * kTcM;
    const uint32_t mvalid = min(uint32_t(kTcM), p.din - i0);
    const uint32_t rbeg = p.row0 + split * p.rows_per_split;
    const uint32_t rend = min(p.n, rbeg + p.rows_per_split);
    const uint32_t npad = p.npad;
    const uint32_t a_lbo = tc_lbo(kTcM), b_lbo = tc_lbo(npad);
    const uint32_t a_bytes = a_lbo * (kTcKt / 4), b_bytes = b_lbo * (kTcKt / 4);
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    // work items: A has 32 q x 8 c = 256 (one per thread); B has npad/4 q x 8 c
    const uint32_t a_q = tid & 31, a_c = tid >> 5;
    const uint32_t b_items = (npad / 4) * (kTcKt / 4);
    const bool has_b = uint32_t(tid) < b_items;
    const uint32_t b_q = tid % (npad / 4), b_c = tid / (npad / 4);
    const bool do_bias = p.wsb && blockIdx.y == 0;

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

    float bcol[4] = {0.f, 0.f, 0.f, 0.f};
    const uint32_t nst = (rend > rbeg) ? (rend - rbeg + kTcKt - 1) / kTcKt : 0;
    // kTcPf stages of row loads in flight per thread (a register ring, statically indexed by
    // unrolling the stage loop kTcPf times): the id-ordered rows are random 512-byte reads and
    // the loop is bound by their latency (ncu: long-scoreboard stalls first, DRAM at 1.9 TB/s).
    // Per Reddit epoch: 1 stage 8.14 ms, 2 stages 7.57, 4 stages 8.06 (244 registers)
    TcItem ia[kTcPf], ib[kTcPf];
#pragma unroll
    for (int u = 0; u < kTcPf; ++u)
        if (uint32_t(u) < nst) {
            const uint32_t r1 = rbeg + u * kTcKt;
            tc_load(ia[u], p.pre, p.prestride, i0 + 4 * a_q, p.din, r1 + 4 * a_c, rend, p.rows);
            if (has_b) tc_load(ib[u], p.dz, p.dzstride, 4 * b_q, p.dout, r1 + 4 * b_c, rend, p.rows);
        }
    uint32_t uses[2] = {0, 0};
    for (uint32_t it0 = 0; it0 < nst; it0 += kTcPf) {
#pragma unroll
        for (int u = 0; u < kTcPf; ++u) {
            const uint32_t it = it0 + u;
            if (it >= nst) break;
            const uint32_t st = it & 1;
            if (uses[st] > 0) mbar_wait(&bars[st], (uses[st] - 1) & 1);  // MMAs that read this stage are done
            uint8_t* base = tsm + st * stage_bytes;
            uint8_t* a_hi = base;
            uint8_t* a_lo = base + a_bytes;
            uint8_t* b_hi = base + 2 * a_bytes;
            uint8_t* b_lo = base + 2 * a_bytes + b_bytes;
            tc_store(ia[u], a_hi, a_lo, a_lbo, a_c, a_q, i0 + mvalid, i0 + 4 * a_q, nullptr);
            if (has_b) tc_store(ib[u], b_hi, b_lo, b_lbo, b_c, b_q, p.dout, 4 * b_q, do_bias ? bcol : nullptr);
            if (it + kTcPf < nst) {  // refill the slot kTcPf stages ahead
                const uint32_t r1 = rbeg + (it + kTcPf) * kTcKt;
                tc_load(ia[u], p.pre, p.prestride, i0 + 4 * a_q, p.din, r1 + 4 * a_c, rend, p.rows);
                if (has_b) tc_load(ib[u], p.dz, p.dzstride, 4 * b_q, p.dout, r1 + 4 * b_c, rend, p.rows);
            }
            // generic-proxy smem writes -> visible to the tensor-core (async) proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
                for (uint32_t s = 0; s < kTcKt / 8; ++s) {
                    const uint64_t dah = umma_desc(ah + 2 * s * a_lbo, a_lbo, kTcSbo);
                    const uint64_t dal = umma_desc(al + 2 * s * a_lbo, a_lbo, kTcSbo);
                    const uint64_t dbh = umma_desc(bh + 2 * s * b_lbo, b_lbo, kTcSbo);
                    const uint64_t dbl = umma_desc(bl + 2 * s * b_lbo, b_lbo, kTcSbo);
                    const uint32_t first = (it == 0 && s == 0) ? 0u : 1u;
                    mma_tf32(tmem, dah, dbh, idesc, first);
                    mma_tf32(tmem, dah, dbl, idesc, 1u);
                    mma_tf32(tmem, dal, dbh, idesc, 1u);
                }
                umma_commit(&bars[st]);
            }
            ++uses[st];
        }
    }
    // bias partials: thread (b_q, b_c) summed columns 4b_q..+3 over its rows; fold the 8 k-cores
    if (do_bias) {
        for (int i = tid; i < (kTcThreads / 32) * 128; i += kTcThreads) (&bsum_sh[0][0])[i] = 0.f;
        __syncthreads();
        if (has_b)
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(&bsum_sh[b_c][4 * b_q + j], bcol[j]);
        __syncthreads();
        if (uint32_t(tid) < p.dout) {
            float sacc = 0.f;
            for (int c = 0; c < kTcKt / 4; ++c) sacc += bsum_sh[c][tid];
            p.wsb[size_t(split) * p.dout + tid] = sacc;
        }
    }
    // all MMAs done -> read the accumulator (warps 0-3 own TMEM lanes 0-127)
    if (tid == 0) umma_commit(&bars[2]);
    if (nst > 0) mbar_wait(&bars[2], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        float* w = p.ws + size_t(split) * p.din * p.dout;
        const uint32_t m = 32 * warp + (tid & 31);
        for (uint32_t c0 = 0; c0 < npad; c0 += 16) {
            float v[16];
            tmem_ld16<16>(tmem + ((32u * warp) << 16) + c0, v);
            if (m < mvalid) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t nn = c0 + j;
                    if (nn < p.dout) w[size_t(i0 + m) * p.dout + nn] = nst > 0 ? v[j] : 0.f;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace gp

// Row gather through the copy engine of the SM (TMA, 1-D `cp.async.bulk` of one 416-byte row per
// request into a per-warp shared-memory ring on mbarriers) against the LDG.256 register gather
// (tools/gather_ceiling.cu), and the two mixed in one CTA (odd warps LDG, even warps bulk): does a
// path that does not go through the L1TEX load data pipe lift the random-row gather roof?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bulk_gather_bench.cu -o tools/bulk_gather_bench
//   bulk_gather_bench <rows> <stride> [gathers]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// one warp's span of the index list [p0, p1) in groups of RPS rows, ST groups in flight
template <int ST, int RPS>
__device__ void bulk_span(const float* __restrict__ tab, const unsigned* __restrict__ idx, long p0, long p1, int stride,
                          int lanes, unsigned char* ring, uint64_t* bars, float& acc) {
    const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
    const uint32_t rowb = uint32_t(stride) * 4;
    const long ng = (p1 - p0) / RPS;
    auto issue = [&](long g, int s) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])),
                         "r"(rowb * RPS)
                         : "memory");
        __syncwarp();
        if (lane < RPS) {
            const unsigned r = idx[p0 + g * RPS + lane];
            unsigned char* dst = ring + (size_t(s) * RPS + lane) * rowb;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(dst)),
                "l"(tab + size_t(r) * stride), "r"(rowb), "r"(smem_u32(&bars[s]))
                : "memory");
        }
    };
    for (int s = 0; s < ST && s < ng; ++s) issue(s, s);
    for (long g = 0; g < ng; ++g) {
        const int s = int(g % ST);
        mbar_wait(&bars[s], uint32_t((g / ST) & 1));
        if (hl < lanes) {
#pragma unroll
            for (int r = half; r < RPS; r += 2) {
                const float4* q = reinterpret_cast<const float4*>(ring + (size_t(s) * RPS + r) * rowb) + 2 * hl;
                const float4 a = q[0], b = q[1];
                acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
            }
        }
        __syncwarp();
        if (g + ST < ng) issue(g + ST, s);
    }
}

__device__ void ldg_span(const float* __restrict__ tab, const unsigned* __restrict__ idx, long p0, long p1, int stride,
                         int lanes, float& acc) {
    constexpr int NB = 4;
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const int loff = hl < lanes ? 8 * hl : 0;
    for (long base = p0; base + 32 <= p1; base += 32) {
        const unsigned my = idx[base + lane];
#pragma unroll
        for (int t = 0; t < 16; t += NB) {
            float x[NB][8];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const unsigned r = __shfl_sync(0xffffffff, my, hb + t + i);
                const float* p = tab + (size_t)r * stride + loff;
                asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(x[i][0]), "=f"(x[i][1]), "=f"(x[i][2]), "=f"(x[i][3]), "=f"(x[i][4]),
                               "=f"(x[i][5]), "=f"(x[i][6]), "=f"(x[i][7])
                             : "l"(p));
            }
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc += x[i][c];
        }
    }
}

// mode 0: every warp bulk; mode 1: odd warps LDG, even warps bulk; mode 2: every warp LDG
template <int ST, int RPS>
__global__ void __launch_bounds__(256) gather_bulk(const float* __restrict__ tab, const unsigned* __restrict__ idx,
                                                   long nidx, int stride, int lanes, int mode, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int w = threadIdx.x >> 5, nwb = blockDim.x >> 5, lane = threadIdx.x & 31;
    const size_t ringb = size_t(ST) * RPS * stride * 4;
    unsigned char* ring = sm + w * ringb;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + nwb * ringb) + w * ST;
    if (lane == 0)
        for (int s = 0; s < ST; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long gw = long(blockIdx.x) * nwb + w, nw = long(gridDim.x) * nwb;
    // contiguous spans of 32-index blocks per warp
    const long nblk = nidx / 32, per = (nblk + nw - 1) / nw;
    const long p0 = min(nblk, gw * per) * 32, p1 = min(nblk, (gw + 1) * per) * 32;
    float acc = 0.f;
    const bool use_ldg = mode == 2 || (mode == 1 && (w & 1));
    if (use_ldg)
        ldg_span(tab, idx, p0, p1, stride, lanes, acc);
    else
        bulk_span<ST, RPS>(tab, idx, p0, p1, stride, lanes, ring, bars, acc);
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
    const long rows = argc > 1 ? std::atol(argv[1]) : 232965;
    const int stride = argc > 2 ? std::atoi(argv[2]) : 104;
    const long nidx = argc > 3 ? std::atol(argv[3]) : 64l << 20;
    const int lanes = (stride + 7) / 8;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    unsigned* idx;
    cudaMalloc(&idx, nidx * 4);
    std::vector<unsigned> h(nidx);
    unsigned long long s = 88172645463325252ull;
    for (long i = 0; i < nidx; ++i) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        h[i] = unsigned(s % rows);
    }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    float* tab;
    const size_t tbytes = (size_t)rows * stride * 4;
    cudaMalloc(&tab, tbytes);
    cudaMemset(tab, 0, tbytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = (double)nidx * stride * 4;
    auto run = [&](auto kern, const char* name, int st, int rps) {
        const size_t smem = 8 * (size_t(st) * rps * stride * 4 + st * 8);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
        for (int mode = 0; mode < 3; ++mode) {
            float ms = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                float t = 0;
                cudaEventRecord(a);
                kern<<<nsm * occ, 256, smem>>>(tab, idx, nidx, stride, lanes, mode, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&t, a, b);
                if (rep) ms = t < ms ? t : ms;
            }
            const cudaError_t e = cudaGetLastError();
            std::printf("%s ST=%d RPS=%d smem=%zu occ=%d mode=%s: %.3f ms %.0f GB/s %s\n", name, st, rps, smem, occ,
                        mode == 0 ? "bulk" : mode == 1 ? "mixed" : "ldg", ms, bytes / (ms * 1e-3) / 1e9,
                        e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    };
    run(gather_bulk<4, 8>, "bulk", 4, 8);
    run(gather_bulk<8, 4>, "bulk", 8, 4);
    run(gather_bulk<2, 16>, "bulk", 2, 16);
    run(gather_bulk<3, 8>, "bulk", 3, 8);
    run(gather_bulk<6, 4>, "bulk", 6, 4);
    run(gather_bulk<2, 8>, "bulk", 2, 8);
    return 0;
}

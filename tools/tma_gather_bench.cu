// TMA tile::gather4 ceiling for the row gather (Reddit shape: 232,965 x 104 f32
// table, random rows): each warp keeps STAGES gather4 requests (4 rows = 1664 B
// each) in flight into its shared-memory ring; the two half-warps consume two
// rows each per request (8 floats per lane, weighted accumulate), as the row
// kernels would. Compare with tools/l2_gather_bench_v8 (LDG.256 into registers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_gather_bench.cu -o tools/tma_gather_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e = (x);                                                                        \
        if (e != cudaSuccess) {                                                                     \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));                \
            return 1;                                                                               \
        }                                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity));
}

__device__ __forceinline__ void issue4(const CUtensorMap* tm, uint64_t* bar, void* dst, int r0, int r1, int r2, int r3,
                                       uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

constexpr int kRowB = 416;  // 104 floats

template <int STAGES, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) t1(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx,
                                                 uint64_t nidx, float* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    uint8_t* ring = sm + size_t(warp) * STAGES * 4 * kRowB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + size_t(WARPS) * STAGES * 4 * kRowB) + warp * STAGES;
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // contiguous range of 32-entry blocks per warp
    const uint64_t gw = (blockIdx.x * uint64_t(WARPS)) + warp, nw = uint64_t(gridDim.x) * WARPS;
    const uint64_t nblk = nidx / 32, b0 = nblk * gw / nw, b1 = nblk * (gw + 1) / nw;
    const uint64_t steps = (b1 - b0) * 8;  // gather4 groups
    // idx registers: block of the next issue and the one after it
    uint64_t iblk = 0;  // relative block index held in `cur`
    uint32_t cur = b0 < b1 ? idx[(b0 + 0) * 32 + lane] : 0u;
    uint32_t nxt = b0 + 1 < b1 ? idx[(b0 + 1) * 32 + lane] : 0u;
    auto issue_g = [&](uint64_t g) {  // all lanes call (shuffles)
        const uint64_t blk = g / 8;
        if (blk != iblk) {  // advance one block
            cur = nxt;
            iblk = blk;
            nxt = b0 + blk + 1 < b1 ? idx[(b0 + blk + 1) * 32 + lane] : 0u;
        }
        const int q = int(g % 8) * 4;
        const int r0 = __shfl_sync(0xffffffffu, cur, q), r1 = __shfl_sync(0xffffffffu, cur, q + 1);
        const int r2 = __shfl_sync(0xffffffffu, cur, q + 2), r3 = __shfl_sync(0xffffffffu, cur, q + 3);
        if (lane == 0) {
            const int slot = int(g % STAGES);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue4(&tm, bars + slot, ring + size_t(slot) * 4 * kRowB, r0, r1, r2, r3, 4 * kRowB);
        }
    };
    for (int s = 0; s < STAGES && uint64_t(s) < steps; ++s) issue_g(s);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t s = 0; s < steps; ++s) {
        const int slot = int(s % STAGES);
        mbar_wait(bars + slot, uint32_t((s / STAGES) & 1));
        if (hl < 13) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float4* p = reinterpret_cast<const float4*>(ring + (size_t(slot) * 4 + (hb ? 2 : 0) + r) * kRowB + 32 * hl);
                const float4 a = p[0], b = p[1];
                acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
                acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
            }
        }
        __syncwarp();
        if (s + STAGES < steps) issue_g(s + STAGES);
    }
    float t = 0;
    for (int c = 0; c < 8; ++c) t += acc[c];
    if (t == 1234.5f) out[0] = t;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint32_t N = 232965, W = 104;
    const uint64_t nidx = 114818775 / 4 * 4;
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    float* tab;
    CK(cudaMalloc(&tab, size_t(N) * W * 4));
    CK(cudaMemset(tab, 0, size_t(N) * W * 4));
    uint32_t* idx;
    CK(cudaMalloc(&idx, nidx * 4));
    std::vector<uint32_t> h(nidx);
    uint64_t s = 88172645463325252ull;
    for (uint64_t i = 0; i < nidx; ++i) {
        s ^= s << 13, s ^= s >> 7, s ^= s << 17;
        h[i] = uint32_t(s % N);
    }
    CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    float* out;
    CK(cudaMalloc(&out, 4));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
    CUtensorMap tm;
    const cuuint64_t dims[2] = {W, N}, strides[1] = {W * 4};
    const cuuint32_t box[2] = {W, 1}, es[2] = {1, 1};
    for (auto prom : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
        CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", int(r));
            return 1;
        }
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const double gb = double(nidx) * W * 4 / 1e9;
        auto run = [&](auto kern, int warps, int stages, const char* name) {
            const size_t smem = size_t(warps) * stages * (4 * kRowB + 8);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                kern<<<nsm * occ, warps * 32, smem>>>(tm, idx, nidx, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
            }
            cudaError_t e = cudaGetLastError();
            printf("promo=%d %-16s occ=%d in-flight/SM=%5.0f KB : %.3f ms  %.0f GB/s %s\n", int(prom), name, occ,
                   occ * warps * stages * 4 * kRowB / 1024.0, ms, gb / ms * 1e3, e == cudaSuccess ? "" : cudaGetErrorString(e));
        };
        run(t1<4, 8>, 8, 4, "W8 S4");
        run(t1<8, 8>, 8, 8, "W8 S8");
        run(t1<8, 4>, 4, 8, "W4 S8");
        run(t1<16, 4>, 4, 16, "W4 S16");
        run(t1<4, 16>, 16, 4, "W16 S4");
        run(t1<6, 16>, 16, 6, "W16 S6");
    }
    return 0;
}

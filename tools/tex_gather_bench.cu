// Does the texture path add gather bandwidth on top of LDG? Random 416-byte row
// gathers from a 97 MB table (Reddit shape), half-warp per row as in the row
// kernels: (a) LDG.256 only, (b) TEX (tex1Dfetch<float4>, 2 per lane) only,
// (c) even rows via LDG, odd rows via TEX.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tex_gather_bench.cu -o tools/tex_gather_bench
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ void ld8(const float* p, float (&x)[8]) {
    asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
        : "l"(p));
}

template <int MODE, int NB>
__global__ void __launch_bounds__(256, 4) g(const float* __restrict__ tab, cudaTextureObject_t tex,
                                            const unsigned* __restrict__ idx, long nidx, int stride, float* out) {
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nw = (gridDim.x * (long)blockDim.x) >> 5;
    float acc = 0.f;
    const int loff = hl < 13 ? 8 * hl : 0;
    for (long base = warp * 32; base < nidx; base += nw * 32) {
        const unsigned my = base + lane < nidx ? idx[base + lane] : 0;
#pragma unroll
        for (int t = 0; t < 16; t += NB) {
            float x[NB][8];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const unsigned r = __shfl_sync(0xffffffff, my, hb + t + i);
                const bool use_tex = MODE == 1 || (MODE == 2 && ((t + i) & 1));
                if (use_tex) {
                    const int e = (int)(r * (stride / 4) + loff / 4);
                    const float4 a = tex1Dfetch<float4>(tex, e), b = tex1Dfetch<float4>(tex, e + 1);
                    x[i][0] = a.x, x[i][1] = a.y, x[i][2] = a.z, x[i][3] = a.w;
                    x[i][4] = b.x, x[i][5] = b.y, x[i][6] = b.z, x[i][7] = b.w;
                } else {
                    ld8(tab + (size_t)r * stride + loff, x[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc += x[i][c];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long nidx = 114818775;
    const int N = 232965, stride = 104;
    float* out;
    cudaMalloc(&out, 4);
    unsigned* idx;
    cudaMalloc(&idx, nidx * 4);
    std::vector<unsigned> h(nidx);
    unsigned long long s = 88172645463325252ull;
    for (long i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % N; }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    float* tab;
    const size_t bytes = (size_t)(N + 1) * stride * 4;
    cudaMalloc(&tab, bytes);
    cudaMemset(tab, 0, bytes);
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = tab;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) { printf("tex create failed\n"); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gb = (double)nidx * stride * 4 / 1e9;
    auto run = [&](auto kern, const char* name) {
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            kern<<<nsm * 4, 256>>>(tab, tex, idx, nidx, stride, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("%-24s %.3f ms  %.0f GB/s %s\n", name, ms, gb / ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    run(g<0, 2>, "LDG.256 NB2");
    run(g<0, 4>, "LDG.256 NB4");
    run(g<1, 2>, "TEX x2 NB2");
    run(g<1, 4>, "TEX x2 NB4");
    run(g<2, 2>, "mixed NB2");
    run(g<2, 4>, "mixed NB4");
    return 0;
}

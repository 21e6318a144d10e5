// Gather ceiling with sm_100 256-bit loads: a half-warp (13 active lanes x 32 B)
// fetches one 416-byte row; NB gathers in flight per lane; 2 rows per warp.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int NB>
__global__ void gather8(const float* __restrict__ tab, const unsigned* __restrict__ idx, long nidx, int stride,
                        float* out) {
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nw = (gridDim.x * (long)blockDim.x) >> 5;
    float acc = 0.f;
    const int loff = hl < 13 ? 8 * hl : 0;
    for (long base = warp * 32; base < nidx; base += nw * 32) {
        unsigned my = base + lane < nidx ? idx[base + lane] : 0;
        #pragma unroll
        for (int t = 0; t < 16; t += NB) {
            float x[NB][8];
            #pragma unroll
            for (int i = 0; i < NB; ++i) {
                unsigned r = __shfl_sync(0xffffffff, my, hb + t + i);
                const float* p = tab + (size_t)r * stride + loff;
                asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                    : "=f"(x[i][0]), "=f"(x[i][1]), "=f"(x[i][2]), "=f"(x[i][3]), "=f"(x[i][4]), "=f"(x[i][5]),
                      "=f"(x[i][6]), "=f"(x[i][7]) : "l"(p));
            }
            #pragma unroll
            for (int i = 0; i < NB; ++i)
                #pragma unroll
                for (int c = 0; c < 8; ++c) acc += x[i][c];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void fill_rand(float* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
        p[i] = (float)(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
    }
}

int main(int argc, char** argv) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long nidx = 114818775;
    float* out; cudaMalloc(&out, 4);
    unsigned* idx; cudaMalloc(&idx, nidx * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int N = 232965, stride = 104;
    std::vector<unsigned> h(nidx);
    unsigned long long s = 88172645463325252ull;
    for (long i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % N; }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    float* tab; cudaMalloc(&tab, (size_t)(N + 1) * stride * 4); cudaMemset(tab, 0, (size_t)(N + 1) * stride * 4);
    if (argc > 1) { fill_rand<<<1184, 256>>>(tab, (size_t)(N + 1) * stride); cudaDeviceSynchronize(); printf("random table\n"); }
    const double gb = (double)nidx * stride * 4 / 1e9;
    auto run = [&](auto kern, const char* name, int occ) {
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a); kern<<<nsm * occ, 256>>>(tab, idx, nidx, stride, out); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        }
        printf("v8 %s occ=%d : %.3f ms  %.0f GB/s\n", name, occ, ms, gb / ms * 1e3);
    };
    for (int occ : {4}) {
        run(gather8<2>, "NB2", occ);
        run(gather8<4>, "NB4", occ);
        run(gather8<8>, "NB8", occ);
    }
    return 0;
}

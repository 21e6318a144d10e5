// Microbenchmark: ceiling of random row gathers (the SpMM's access pattern) on B200.
// Rows of `width` floats at stride `stride` from an N-row table; each warp walks a list
// of random row ids, lanes 0..width/4-1 load one float4 per row, U loads in flight.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int U>
__global__ void gather(const float* __restrict__ tab, const unsigned* __restrict__ idx, long nidx,
                       int stride, int w4, float* out) {
    const int lane = threadIdx.x & 31;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nw = (gridDim.x * (long)blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    const bool act = lane < w4;
    for (long base = warp * 32 * U; base < nidx; base += nw * 32 * U) {
        #pragma unroll
        for (int b = 0; b < U; ++b) {
            const long e = base + b * 32 + lane;
            unsigned my = e < nidx ? idx[e] : 0;
            float4 x[8];
            #pragma unroll
            for (int t = 0; t < 32; t += 8) {
                #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    unsigned r = __shfl_sync(0xffffffff, my, t + i);
                    x[i] = act ? __ldg(reinterpret_cast<const float4*>(tab + (size_t)r * stride) + lane) : make_float4(0,0,0,0);
                }
                #pragma unroll
                for (int i = 0; i < 8; ++i) { acc.x += x[i].x; acc.y += x[i].y; acc.z += x[i].z; acc.w += x[i].w; }
            }
        }
    }
    if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void gather_deep(const float* __restrict__ tab, const unsigned* __restrict__ idx, long nidx,
                            int stride, int w4, float* out) {
    // 16 gathers in flight per lane
    const int lane = threadIdx.x & 31;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nw = (gridDim.x * (long)blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    const bool act = lane < w4;
    for (long base = warp * 32; base < nidx; base += nw * 32) {
        unsigned my = base + lane < nidx ? idx[base + lane] : 0;
        #pragma unroll
        for (int t = 0; t < 32; t += 16) {
            float4 x[16];
            #pragma unroll
            for (int i = 0; i < 16; ++i) {
                unsigned r = __shfl_sync(0xffffffff, my, t + i);
                x[i] = act ? __ldg(reinterpret_cast<const float4*>(tab + (size_t)r * stride) + lane) : make_float4(0,0,0,0);
            }
            #pragma unroll
            for (int i = 0; i < 16; ++i) { acc.x += x[i].x; acc.y += x[i].y; acc.z += x[i].z; acc.w += x[i].w; }
        }
    }
    if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void stream_read(const float4* __restrict__ a, long n4, float* out) {
    float4 acc = make_float4(0,0,0,0);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 x = __ldg(a + i); acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    if (acc.x == 1234.5f) out[0] = acc.y;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long nidx = 114818775;
    float* out; cudaMalloc(&out, 4);
    unsigned* idx; cudaMalloc(&idx, nidx * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int N : {232965, 2449029}) {
      for (int stride : {104, 128}) {
        int width = 100;
        std::vector<unsigned> h(nidx);
        unsigned long long s = 88172645463325252ull;
        for (long i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % N; }
        cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
        float* tab; cudaMalloc(&tab, (size_t)N * stride * 4); cudaMemset(tab, 0, (size_t)N * stride * 4);
        int w4 = width / 4;
        for (int occ : {2, 4, 8}) {
            int grid = nsm * occ;
            float ms;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a); gather<1><<<grid, 256>>>(tab, idx, nidx, stride, w4, out); cudaEventRecord(b);
                cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            }
            double gb = (double)nidx * stride * 4 / 1e9;
            printf("N=%d stride=%d occ=%d U8  : %.3f ms  %.0f GB/s (rows*stride)\n", N, stride, occ, ms, gb / ms * 1e3);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a); gather_deep<<<grid, 256>>>(tab, idx, nidx, stride, w4, out); cudaEventRecord(b);
                cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            }
            printf("N=%d stride=%d occ=%d U16 : %.3f ms  %.0f GB/s\n", N, stride, occ, ms, gb / ms * 1e3);
        }
        cudaFree(tab);
      }
    }
    // streaming L2-resident read: 64 MB read 10x
    {
        long n4 = 64l << 20 >> 4; float4* buf; cudaMalloc(&buf, n4 * 16); cudaMemset(buf, 0, n4*16);
        float ms;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a); for (int k = 0; k < 10; ++k) stream_read<<<nsm * 8, 256>>>(buf, n4, out); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        }
        printf("L2-resident stream 64MB x10: %.0f GB/s\n", 10.0 * n4 * 16 / 1e9 / ms * 1e3);
        long m4 = 4l << 30 >> 4; float4* big; cudaMalloc(&big, m4 * 16); cudaMemset(big, 0, m4*16);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a); stream_read<<<nsm * 8, 256>>>(big, m4, out); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        }
        printf("HBM stream 4GB: %.0f GB/s\n", m4 * 16 / 1e9 / ms * 1e3);
    }
    return 0;
}

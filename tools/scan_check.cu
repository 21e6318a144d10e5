// Standalone check of the engine's u64 in-place inclusive scan (kernels.cuh: k_scan_tiles /
// k_scan_totals / k_scan_add) against a host scan, at sizes that need one and several
// k_scan_totals chunks. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. tools/scan_check.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2308_10087_b200/csrc/device/kernels.cuh"
using namespace gp;

int main() {
    const uint32_t sizes[] = {1, 2, 1000, 4096, 4097, 233966, 4194304 + 17, 12000001};
    int bad = 0;
    for (uint32_t n : sizes) {
        std::vector<unsigned long long> h(n), ref(n);
        unsigned long long run = 0;
        for (uint32_t i = 0; i < n; ++i) {
            h[i] = (i * 2654435761u) % 1000u;
            run += h[i];
            ref[i] = run;
        }
        unsigned long long *d, *tot;
        const uint32_t tiles = (n + kScanTile - 1) / kScanTile;
        cudaMalloc(&d, n * 8ull);
        cudaMalloc(&tot, tiles * 8ull);
        cudaMemcpy(d, h.data(), n * 8ull, cudaMemcpyHostToDevice);
        k_scan_tiles<<<tiles, kScanThreads>>>(d, n, tot);
        k_scan_totals<<<1, kScanThreads>>>(tot, tiles);
        k_scan_add<<<tiles, kScanThreads>>>(d, n, tot);
        cudaMemcpy(h.data(), d, n * 8ull, cudaMemcpyDeviceToHost);
        const cudaError_t e = cudaGetLastError();
        uint32_t wrong = 0;
        for (uint32_t i = 0; i < n; ++i) wrong += h[i] != ref[i];
        std::printf("n=%u tiles=%u wrong=%u %s\n", n, tiles, wrong, cudaGetErrorString(e));
        bad |= wrong != 0 || e != cudaSuccess;
        cudaFree(d);
        cudaFree(tot);
    }
    std::printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}

// Allocation cost on the B200: 42 GB as ~500 cudaMalloc'd buffers (zeroed) vs one
// arena, create + free, repeated (engine creation/teardown is part of bench.py's e2e).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    cudaFree(0);
    const size_t total = size_t(42) << 30, nbuf = 500, each = total / nbuf;
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        std::vector<void*> v(nbuf);
        for (auto& p : v) { cudaMalloc(&p, each); cudaMemset(p, 0, each); }
        cudaDeviceSynchronize();
        double t1 = now();
        for (auto p : v) cudaFree(p);
        cudaDeviceSynchronize();
        double t2 = now();
        void* a;
        cudaMalloc(&a, total);
        cudaMemsetAsync(a, 0, total);
        cudaDeviceSynchronize();
        double t3 = now();
        cudaFree(a);
        cudaDeviceSynchronize();
        double t4 = now();
        std::printf("rep %d: %zu buffers create %.3f s free %.3f s | arena create %.3f s free %.3f s\n", rep, nbuf,
                    t1 - t0, t2 - t1, t3 - t2, t4 - t3);
    }
}

// Standalone timing harness for the forward row kernel (Reddit-shaped ER CSR,
// GCNII layer H=100): the engine's k_fwd8 against experimental variants, at the
// launch sizes of K=4 and K=32 chunks. Timing only (results are checked for
// equality between variants that must agree bit-for-bit).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2308_10087_b200/csrc/device \
//        tools/fwd_bench.cu -o tools/fwd_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "dense_tile.cuh"
#include "rows8.cuh"  // -I paper_2308_10087_b200/csrc/device (or an older copy, to compare)

using namespace gp;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

// ---------------------------------------------------------------------------
// Ladder from the pure gather microbenchmark to the row kernel.
// X1: edge-parallel (ignores rows): 32 consecutive CSR entries per warp, 16 per half.
template <int NB>
__global__ void __launch_bounds__(kBlock) x1_edge_par(const uint2* __restrict__ edges, uint64_t nnz,
                                                      const float* __restrict__ tab, uint32_t stride, float* out) {
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * uint64_t(blockDim.x)) >> 5;
    float acc = 0.f;
    const float* ls = tab + (hl < 13 ? 8 * hl : 0);
    for (uint64_t base = warp * 32; base < nnz; base += nw * 32) {
        const uint32_t my = base + lane < nnz ? edges[base + lane].x & kColMask : 0u;
#pragma unroll
        for (int t = 0; t < 16; t += NB) {
            F8 x[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) x[i] = ld8_gather(ls + size_t(__shfl_sync(kFull, my, hb + t + i)) * stride);
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc += x[i].v[c];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// X2/X3: half-warp per row (rows [r0, r1), static pairs), 16-entry batches fully
// unrolled like X1; W=false: acc += x, W=true: weighted per-column mul_add chain.
template <int NB, bool WT>
__global__ void __launch_bounds__(kBlock, 4) x2_row(const uint64_t* __restrict__ rowptr, const uint2* __restrict__ edges,
                                                    uint32_t r0, uint32_t r1, const float* __restrict__ tab,
                                                    uint32_t stride, float* out) {
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const float* ls = tab + (hl < 13 ? 8 * hl : 0);
    for (uint32_t base = r0 + 2 * warp; base < r1; base += 2 * nw) {
        const uint32_t v = base + (hb ? 1 : 0);
        const bool has = v < r1;
        const uint64_t e0 = has ? rowptr[v] : 0, e1 = has ? rowptr[v + 1] : 0;
        const uint32_t n_my = uint32_t(e1 - e0);
        const uint32_t n_max = max(n_my, __shfl_xor_sync(kFull, n_my, 16));
        F8 acc = f8_zero();
        for (uint32_t off = 0; off < n_max; off += 16) {
            const uint2 my = off + hl < n_my ? edges[e0 + off + hl] : make_uint2(has ? v : 0u, 0u);
#pragma unroll
            for (int t = 0; t < 16; t += NB) {
                F8 x[NB];
                float w[NB];
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const uint32_t c = __shfl_sync(kFull, my.x, hb + t + i) & kColMask;
                    w[i] = __uint_as_float(__shfl_sync(kFull, my.y, hb + t + i));
                    x[i] = ld8_gather(ls + size_t(c) * stride);
                }
#pragma unroll
                for (int i = 0; i < NB; ++i)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc.v[c] = WT ? mul_add(acc.v[c], w[i], x[i].v[c]) : acc.v[c] + x[i].v[c];
            }
        }
        if (has && hl < 13) st8_stream(out + size_t(v) * stride + 8 * hl, acc);
    }
}

// ---------------------------------------------------------------------------
__global__ void k_gen_edges(const uint64_t* rowptr, uint2* edges, uint32_t n, uint32_t chunk_rows, int perm) {
    const uint32_t v = blockIdx.x;
    const uint64_t b = rowptr[v], e = rowptr[v + 1];
    const uint32_t d = uint32_t(e - b);
    // sorted random columns: stratified (one per stratum of n/d), plus the row itself somewhere
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
        uint64_t h = mix64(0x1234567ull ^ v, j);
        const uint64_t lo = uint64_t(n) * j / d, hi = uint64_t(n) * (j + 1) / d;
        const uint64_t span = hi > lo ? hi - lo : 1;
        uint32_t c = uint32_t(lo + h % span);
        if (c >= n) c = n - 1;
        if (perm) c = uint32_t((uint64_t(c) * 7919u + 12345u) % n);  // table slot of the column: scattered
        edges[b + j] = make_uint2(c | ((c / chunk_rows) << kColBits), __float_as_uint(1.0f / 492.f));
    }
}

__global__ void k_fill(float* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = float(mix64(seed, i) >> 40) * (1.0f / 16777216.0f) - 0.5f;
}

int main(int argc, char** argv) {
    const uint32_t N = 232965, H = 100, S8 = 104;
    const int reps = 6;
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    // degrees 492 +- 64 (uniformish)
    std::vector<uint64_t> rp(N + 1, 0);
    for (uint32_t v = 0; v < N; ++v) rp[v + 1] = rp[v] + 428 + (mix64(77, v) % 129);
    const uint64_t nnz = rp[N];
    uint64_t* d_rp;
    uint2* d_e;
    CK(cudaMalloc(&d_rp, (N + 1) * 8));
    CK(cudaMalloc(&d_e, nnz * 8));
    CK(cudaMemcpy(d_rp, rp.data(), (N + 1) * 8, cudaMemcpyHostToDevice));
    const bool perm = argc > 1 && std::string(argv[1]) == "perm";
    printf("column slots: %s\n", perm ? "scattered (ascending ids -> random slots)" : "ascending");
    k_gen_edges<<<N, 256>>>(d_rp, d_e, N, (N + 3) / 4, perm ? 1 : 0);
    float *G, *h0, *pre, *out, *gn, *W;
    const size_t tab = size_t(N) * S8;
    CK(cudaMalloc(&G, tab * 4));
    CK(cudaMalloc(&h0, tab * 4));
    CK(cudaMalloc(&pre, tab * 4));
    CK(cudaMalloc(&out, tab * 4));
    CK(cudaMalloc(&gn, tab * 4));
    CK(cudaMalloc(&W, H * H * 4));
    const bool zero_table = argc > 1 && std::string(argv[1]) == "zero";
    if (zero_table) CK(cudaMemset(G, 0, tab * 4));
    else k_fill<<<1184, 256>>>(G, tab, 1);
    printf("gather table: %s\n", zero_table ? "zeros" : "random values");
    k_fill<<<1184, 256>>>(h0, tab, 2);
    k_fill<<<64, 256>>>(W, H * H, 3);
    uint32_t* orig;
    CK(cudaMalloc(&orig, N * 4));
    std::vector<uint32_t> id(N);
    for (uint32_t i = 0; i < N; ++i) id[i] = i;
    CK(cudaMemcpy(orig, id.data(), N * 4, cudaMemcpyHostToDevice));
    uint32_t* tickets;
    CK(cudaMalloc(&tickets, 4096 * 4));
    CK(cudaDeviceSynchronize());
    printf("N=%u nnz=%llu (avg deg %.1f)\n", N, (unsigned long long)nnz, double(nnz) / N);

    FwdParams p{};
    p.rowptr = d_rp;
    p.edges = d_e;
    p.gsrc = G;
    p.gsnap = G;
    p.done = ~0ull;
    p.gstride = S8;
    p.orig = orig;
    p.h0 = h0;
    p.h0stride = S8;
    p.alpha = 0.1f, p.oma = 0.9f, p.beta = 0.05f, p.omb = 0.95f;
    p.W = W;
    p.bias = nullptr;
    p.din = H, p.dout = H;
    p.relu = 1;
    p.pre = pre, p.prestride = S8;
    p.out = out, p.outstride = S8;
    p.gnext = gn, p.gnstride = S8;
    p.next_mask.enabled = 1;
    p.next_mask.k2 = 99;
    p.next_mask.thr = (1ull << 52);
    p.next_mask.scale = 2.f;
    p.next_mask.cols = H;

    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const size_t wsm = row_smem_bytes(H, H, 2);
    auto run = [&](const char* name, const void* fn, size_t smem, int K) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, smem));
        const uint32_t rows = (N + K - 1) / K;
        double tot_ms = 0, edges = 0;
        for (int r = 0; r < reps + 1; ++r) {
            const uint32_t k = uint32_t(r) % uint32_t(K);
            FwdParams q = p;
            q.r0 = k * rows;
            q.r1 = std::min(N, q.r0 + rows);
            q.ticket = tickets + r;
            CK(cudaMemset(q.ticket, 0, 4));
            void* args[] = {&q};
            CK(cudaEventRecord(a));
            CK(cudaLaunchKernel(fn, dim3(nsm * occ), dim3(kBlock), args, smem, 0));
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r > 0) {
                tot_ms += ms;
                edges += double(rp[q.r1] - rp[q.r0]);
            }
        }
        const double ms = tot_ms / reps;
        printf("%-28s K=%-3d occ=%d  %.4f ms/launch  gather %.0f GB/s\n", name, K, occ, ms,
               edges / reps * S8 * 4 / (ms * 1e-3) / 1e9);
    };
    // ladder (K=4 launch sizes: rows of chunk 1)
    {
        const uint32_t rows = (N + 3) / 4, r0 = rows, r1 = 2 * rows;
        const double gb = double(rp[r1] - rp[r0]) * S8 * 4 / 1e9;
        auto tl = [&](const char* name, auto launch) {
            float ms = 0;
            for (int r = 0; r < 4; ++r) {
                CK(cudaEventRecord(a));
                launch();
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                CK(cudaEventElapsedTime(&ms, a, b));
            }
            printf("%-36s %.4f ms  %.0f GB/s\n", name, ms, gb / (ms * 1e-3));
        };
        const uint64_t eb = rp[r0], ne = rp[r1] - rp[r0];
        tl("X1 edge-parallel NB2", [&]() { x1_edge_par<2><<<nsm * 4, kBlock>>>(d_e + eb, ne, G, S8, out); });
        tl("X1 edge-parallel NB4", [&]() { x1_edge_par<4><<<nsm * 4, kBlock>>>(d_e + eb, ne, G, S8, out); });
        tl("X2 row, acc+=x, NB2", [&]() { x2_row<2, false><<<nsm * 4, kBlock>>>(d_rp, d_e, r0, r1, G, S8, out); });
        tl("X2 row, acc+=x, NB4", [&]() { x2_row<4, false><<<nsm * 4, kBlock>>>(d_rp, d_e, r0, r1, G, S8, out); });
        tl("X3 row, weighted, NB2", [&]() { x2_row<2, true><<<nsm * 4, kBlock>>>(d_rp, d_e, r0, r1, G, S8, out); });
        tl("X3 row, weighted, NB4", [&]() { x2_row<4, true><<<nsm * 4, kBlock>>>(d_rp, d_e, r0, r1, G, S8, out); });
        tl("X3 row, weighted, NB8", [&]() { x2_row<8, true><<<nsm * 4, kBlock>>>(d_rp, d_e, r0, r1, G, S8, out); });
    }
    // backward row kernel (PREV_AGG: gather over done chunks; PREV_AGG_HIST) at K=4 sizes
    {
        float *bgn, *bgs, *h, *dz, *dh0, *bg;
        CK(cudaMalloc(&bgn, tab * 4));
        CK(cudaMalloc(&bgs, tab * 4));
        CK(cudaMalloc(&h, tab * 4));
        CK(cudaMalloc(&dz, tab * 4));
        CK(cudaMalloc(&dh0, tab * 4));
        CK(cudaMalloc(&bg, tab * 4));
        k_fill<<<1184, 256>>>(bgn, tab, 5);
        k_fill<<<1184, 256>>>(bgs, tab, 6);
        k_fill<<<1184, 256>>>(h, tab, 7);
        CK(cudaMemset(dh0, 0, tab * 4));
        BwdParams q{};
        q.rowptr = d_rp;
        q.edges = d_e;
        q.bgn = bgn;
        q.bgn_snap = bgs;
        q.bgnstride = S8;
        q.prev_mask = p.next_mask;
        q.orig = orig;
        q.dh_width = H;
        q.dh0stride = S8;
        q.h = h;
        q.hstride = S8;
        q.relu = 1;
        q.dz = dz;
        q.dzstride = S8;
        q.W = W;
        {
            float* WT;
            CK(cudaMalloc(&WT, H * H * 4));
            k_transpose<<<40, 256>>>(W, WT, H, H);
            q.WT = WT;
        }
        q.din = H, q.dout = H;
        q.need_dagg = 1;
        q.gcn2 = 1;
        q.alpha = 0.1f, q.oma = 0.9f, q.beta = 0.05f, q.omb = 0.95f;
        q.dh0 = dh0;
        q.bg = bg;
        q.bgstride = S8;
        const uint32_t rows = (N + 3) / 4;
        auto runb = [&](const char* name, const void* fn, uint64_t done, size_t smem_override = 0) {
            const size_t smem = smem_override ? smem_override : wsm;
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, smem));
            double tot = 0;
            for (int r = 0; r < 4; ++r) {
                BwdParams x = q;
                x.done = done;
                x.r0 = rows;
                x.r1 = 2 * rows;
                x.ticket = tickets + 200 + r;
                CK(cudaMemset(x.ticket, 0, 4));
                void* args[] = {&x};
                CK(cudaEventRecord(a));
                CK(cudaLaunchKernel(fn, dim3(nsm * occ), dim3(kBlock), args, smem, 0));
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                if (r) tot += ms;
            }
            printf("%-34s done=%#llx occ=%d %.4f ms/launch\n", name, (unsigned long long)done, occ, tot / 3);
        };
        for (uint64_t done : {0x2ull, 0x3ull, 0x7ull, 0xfull}) {
            runb("k_bwd8<AGG,LAYER,2>", (const void*)k_bwd8<PREV_AGG, OUT_LAYER, 2>, done);
            runb("k_bwd8<AGG,LAYER,4>", (const void*)k_bwd8<PREV_AGG, OUT_LAYER, 4>, done);
            runb("split k_bwd8<AGG,LAYER,2,1>", (const void*)k_bwd8<PREV_AGG, OUT_LAYER, 2, true>, done);
            runb("split k_bwd8<AGG,LAYER,4,1>", (const void*)k_bwd8<PREV_AGG, OUT_LAYER, 4, true>, done);
            runb("split k_bwd_tile<4>", (const void*)k_bwd_tile<4>, done, tile_smem_bytes(H, H, 4));
            runb("split k_bwd_tile<4,100>", (const void*)k_bwd_tile<4, 100>, done, tile_smem_bytes(H, H, 4));
        }
        runb("k_bwd8<AGG_HIST,LAYER,2>", (const void*)k_bwd8<PREV_AGG_HIST, OUT_LAYER, 2>, 0x3ull);
        std::vector<float> hb(tab);
        // checksum of bg for the 50% done case (compare across builds)
        {
            BwdParams x = q;
            x.done = 0x3ull;
            x.r0 = 0;
            x.r1 = N;
            x.ticket = tickets + 300;
            CK(cudaMemset(x.ticket, 0, 4));
            CK(cudaMemset(dh0, 0, tab * 4));
            void* args[] = {&x};
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k_bwd8<PREV_AGG, OUT_LAYER, 2>, kBlock, wsm));
            CK(cudaLaunchKernel((const void*)k_bwd8<PREV_AGG, OUT_LAYER, 2>, dim3(nsm * occ), dim3(kBlock), args, wsm, 0));
            CK(cudaMemcpy(hb.data(), bg, tab * 4, cudaMemcpyDeviceToHost));
            uint64_t hsh = 1469598103934665603ull;
            for (size_t i = 0; i < tab; ++i) hsh = (hsh ^ reinterpret_cast<uint32_t&>(hb[i])) * 1099511628211ull;
            printf("bwd bg checksum (done=0x3, all rows): %016llx\n", (unsigned long long)hsh);
            // split gather + tiled transform must reproduce bg and dh0 bit for bit
            std::vector<float> hd0(tab), gb(tab), gd0(tab);
            CK(cudaMemcpy(hd0.data(), dh0, tab * 4, cudaMemcpyDeviceToHost));
            const void* fns[2] = {(const void*)k_bwd8<PREV_AGG, OUT_LAYER, 2, true>, (const void*)k_bwd_tile<4>};
            const size_t sms[2] = {kEdgeSlotBytes, tile_smem_bytes(H, H, 4)};
            CK(cudaMemset(dh0, 0, tab * 4));
            CK(cudaMemset(bg, 0, tab * 4));
            for (int f = 0; f < 2; ++f) {
                x.ticket = tickets + 301 + f;
                CK(cudaMemset(x.ticket, 0, 4));
                CK(cudaFuncSetAttribute(fns[f], cudaFuncAttributeMaxDynamicSharedMemorySize, int(sms[f])));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fns[f], kBlock, sms[f]));
                CK(cudaLaunchKernel(fns[f], dim3(nsm * occ), dim3(kBlock), args, sms[f], 0));
            }
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(gb.data(), bg, tab * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(gd0.data(), dh0, tab * 4, cudaMemcpyDeviceToHost));
            size_t bad = 0;
            for (size_t i = 0; i < tab; ++i)
                bad += (reinterpret_cast<uint32_t&>(hb[i]) != reinterpret_cast<uint32_t&>(gb[i])) +
                       (reinterpret_cast<uint32_t&>(hd0[i]) != reinterpret_cast<uint32_t&>(gd0[i]));
            printf("bwd split (gather + tile) vs fused: %zu differing floats\n", bad);
        }
    }
    std::vector<float> ref(tab), got(tab);
    auto snap = [&](std::vector<float>& dst) { CK(cudaMemcpy(dst.data(), out, tab * 4, cudaMemcpyDeviceToHost)); };
    for (int K : {4, 32}) {
        run("k_fwd8<GCN2,2> (engine)", (const void*)k_fwd8<FWD_GCN2, 2>, wsm, K);
        run("k_fwd8<GCN2,4> (engine)", (const void*)k_fwd8<FWD_GCN2, 4>, wsm, K);
        run("split gather k_fwd8<GCN2,2,1>", (const void*)k_fwd8<FWD_GCN2, 2, true>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,4,1>", (const void*)k_fwd8<FWD_GCN2, 4, true>, kEdgeSlotBytes, K);
        // gathers in flight vs resident CTAs (MINB = minimum CTAs per SM for the register cap)
        run("split gather k_fwd8<GCN2,2,1,5> (engine)", (const void*)k_fwd8<FWD_GCN2, 2, true, 5>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,2,1,6>", (const void*)k_fwd8<FWD_GCN2, 2, true, 6>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,4,1,4>", (const void*)k_fwd8<FWD_GCN2, 4, true, 4>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,4,1,3>", (const void*)k_fwd8<FWD_GCN2, 4, true, 3>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,8,1,3>", (const void*)k_fwd8<FWD_GCN2, 8, true, 3>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,8,1,2>", (const void*)k_fwd8<FWD_GCN2, 8, true, 2>, kEdgeSlotBytes, K);
        run("split gather k_fwd8<GCN2,16,1,2>", (const void*)k_fwd8<FWD_GCN2, 16, true, 2>, kEdgeSlotBytes, K);
        {  // one gather table (gsnap = null): no per-entry cur/snapshot choice
            const float* keep = p.gsnap;
            p.gsnap = nullptr;
            run("one-table split gather k_fwd8<GCN2,2,1>", (const void*)k_fwd8<FWD_GCN2, 2, true>, kEdgeSlotBytes, K);
            run("one-table split gather k_fwd8<GCN2,2,1,5>", (const void*)k_fwd8<FWD_GCN2, 2, true, 5>, kEdgeSlotBytes, K);
            run("one-table split gather k_fwd8<GCN2,4,1,4>", (const void*)k_fwd8<FWD_GCN2, 4, true, 4>, kEdgeSlotBytes, K);
            run("one-table split gather k_fwd8<GCN2,4,1,3>", (const void*)k_fwd8<FWD_GCN2, 4, true, 3>, kEdgeSlotBytes, K);
            p.gsnap = keep;
        }
        run("split dense k_fwd_tile<1,4>", (const void*)k_fwd_tile<true, 4>, tile_smem_bytes(H, H, 4), K);
        run("split dense k_fwd_tile<1,4,100>", (const void*)k_fwd_tile<true, 4, 100>, tile_smem_bytes(H, H, 4), K);
        {  // cost of the next-layer dropout epilogue: same transform without gnext
            float* keep = p.gnext;
            p.gnext = nullptr;
            run("  ... without next-layer dropout", (const void*)k_fwd_tile<true, 4, 100>, tile_smem_bytes(H, H, 4), K);
            p.gnext = keep;
        }
        run("split dense k_fwd_tile<1,2>", (const void*)k_fwd_tile<true, 2>, tile_smem_bytes(H, H, 2), K);
        run("split dense k_fwd_tile<1,1>", (const void*)k_fwd_tile<true, 1>, tile_smem_bytes(H, H, 1), K);
        run("k_fwd8 again", (const void*)k_fwd8<FWD_GCN2, 2>, wsm, K);
    }
    // bit-equality of the variants over all rows (K=1 launch)
    auto full = [&](const void* fn, size_t smem) {
        FwdParams q = p;
        q.r0 = 0;
        q.r1 = N;
        q.ticket = tickets + 100;
        CK(cudaMemset(q.ticket, 0, 4));
        CK(cudaMemset(out, 0, tab * 4));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, smem));
        void* args[] = {&q};
        CK(cudaLaunchKernel(fn, dim3(nsm * occ), dim3(kBlock), args, smem, 0));
        CK(cudaDeviceSynchronize());
    };
    full((const void*)k_fwd8<FWD_GCN2, 2>, wsm);
    snap(ref);
    {
        uint64_t hsh = 1469598103934665603ull;
        for (size_t i = 0; i < tab; ++i) hsh = (hsh ^ reinterpret_cast<uint32_t&>(ref[i])) * 1099511628211ull;
        printf("fwd out checksum (all rows): %016llx\n", (unsigned long long)hsh);
    }
    {
        full((const void*)k_fwd8<FWD_GCN2, 2, true>, kEdgeSlotBytes);
        full((const void*)k_fwd_tile<true, 4, 100>, tile_smem_bytes(H, H, 4));
        snap(got);
        size_t bad = 0;
        for (size_t i = 0; i < tab; ++i) bad += (reinterpret_cast<uint32_t&>(ref[i]) != reinterpret_cast<uint32_t&>(got[i]));
        printf("split (gather + tile) vs fused: %zu differing floats\n", bad);
    }
    return 0;
}

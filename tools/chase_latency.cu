// Dependent-load latency on this B200 (one warp, L2-resident / DRAM-resident
// chase), for the walk kernel's per-move latency budget.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chase_latency tools/chase_latency.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_chase(const uint32_t* __restrict__ next, uint64_t hops, uint32_t start, uint32_t* out,
                        unsigned long long* cycles) {
    uint32_t i = start;
    unsigned long long t0 = clock64();
    for (uint64_t h = 0; h < hops; ++h) {
        const uint32_t* p = next + 8ull * i;  // 32 B records
        if (MODE == 0) {  // 32-bit ld.global.cg
            asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(i) : "l"(p));
        } else if (MODE == 1) {  // 256-bit ld.global.cg
            uint32_t a, b, c, d, e, f, g, hh;
            asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(hh) : "l"(p));
            i = a ^ (b & 0);
        } else {  // default caching (L1)
            i = *(volatile const uint32_t*)p;
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) { *out = i; *cycles = t1 - t0; }
}

int main() {
    for (size_t mb : {16ul, 64ul, 4096ul}) {
        const size_t n = mb * (1ul << 20) / 32;
        std::vector<uint32_t> perm(n);
        for (size_t k = 0; k < n; ++k) perm[k] = (uint32_t)k;
        std::mt19937_64 rng(1);
        for (size_t k = n - 1; k > 0; --k) std::swap(perm[k], perm[rng() % (k + 1)]);
        std::vector<uint32_t> h(8 * n, 0);
        for (size_t k = 0; k < n; ++k) h[8ull * perm[k]] = perm[(k + 1) % n];
        uint32_t* d; uint32_t* out; unsigned long long* cyc;
        cudaMalloc(&d, h.size() * 4); cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
        cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        const uint64_t hops = 20000;
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {  // second run: L2 warm for the small sizes
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                if (mode == 0) k_chase<0><<<1, 1>>>(d, hops, perm[0], out, cyc);
                if (mode == 1) k_chase<1><<<1, 1>>>(d, hops, perm[0], out, cyc);
                if (mode == 2) k_chase<2><<<1, 1>>>(d, hops, perm[0], out, cyc);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                if (rep) printf("%5zu MB mode %d (%s): %.0f ns/hop, %.0f cycles/hop\n", mb, mode,
                                mode == 0 ? "cg u32" : mode == 1 ? "cg v8" : "ca u32", ms * 1e6 / hops,
                                (double)c / hops);
            }
        }
        cudaFree(d);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

// Random-access HBM microbenchmark (measurement only): how many random
// aligned G-byte gathers per second B200 sustains, for G = 4..128 B, with the
// L2 fetch-granularity limit at 32 / 64 / 128.  Establishes the random-access
// roofline the walk kernels are judged against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randbw tools/randbw.cu
//   ./randbw [GiB=32]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Each lane performs `iters` dependent-free random gathers of G bytes.
template <int G>
__global__ void gather(const uint4* __restrict__ buf, uint64_t nslots, int iters, uint64_t seed,
                       unsigned long long* sink) {
    uint64_t s = mix(seed ^ (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x));
    uint32_t acc = 0;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t slot = __umul64hi(mix(s), nslots);
        if constexpr (G <= 4) {
            acc += __ldcg(reinterpret_cast<const uint32_t*>(buf) + slot);
        } else if constexpr (G == 8) {
            acc += (uint32_t)__ldcg(reinterpret_cast<const unsigned long long*>(buf) + slot);
        } else if constexpr (G == 33) {  // one 256-bit load of a 32 B sector
            uint32_t a, b, c, d, e, f, g, h;
            asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h)
                         : "l"(buf + slot * 2));
            acc += a ^ h;
        } else {
            const uint4* p = buf + slot * (G / 16);
#pragma unroll
            for (int k = 0; k < G / 16; ++k) {
                uint4 v = __ldcg(p + k);
                acc += v.x ^ v.w;
            }
        }
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// Dependent chain: each lane follows `iters` random pointers (latency-bound
// walk analogue: the next address depends on the loaded value).
__global__ void chase(const uint4* __restrict__ buf, uint64_t nslots, int iters, uint64_t seed,
                      unsigned long long* sink) {
    uint64_t slot = __umul64hi(mix(seed ^ (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x)), nslots);
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint4 v = __ldcg(buf + slot * 2);
        acc += v.x;
        slot = __umul64hi(mix(slot ^ v.y ^ 0x51ED27ULL), nslots);
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int G>
double run(const uint4* buf, uint64_t bytes, int blocks, int iters, unsigned long long* sink) {
    uint64_t nslots = G <= 4 ? bytes / 4 : (G == 8 ? bytes / 8 : (G == 33 ? bytes / 32 : bytes / G));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<G><<<blocks, 256>>>(buf, nslots, iters, 1, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) gather<G><<<blocks, 256>>>(buf, nslots, iters, 2 + r, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double n = 3.0 * blocks * 256.0 * iters;
    return n / (ms * 1e-3);
}

int main(int argc, char** argv) {
    uint64_t gib = argc > 1 ? strtoull(argv[1], nullptr, 10) : 32;
    int only = argc > 2 ? atoi(argv[2]) : 0;  // 1: one pass per variant (for ncu)
    uint64_t bytes = gib << 30;
    uint4* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8;
    const int iters = 256;
    size_t lim = 0;
    for (size_t g : {32, 64, 128}) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
        cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity request %zu -> %s, limit now %zu\n", g, cudaGetErrorString(e), lim);
        double r4 = run<4>(buf, bytes, blocks, iters, sink);
        double r8 = run<8>(buf, bytes, blocks, iters, sink);
        double r16 = run<16>(buf, bytes, blocks, iters, sink);
        double r32 = run<32>(buf, bytes, blocks, iters, sink);
        double r33 = run<33>(buf, bytes, blocks, iters, sink);
        printf("  256-bit sector gathers/s: %.2fG (%.0f GB/s at 32B)\n", r33 / 1e9, r33 * 32 / 1e9);
        double r64 = run<64>(buf, bytes, blocks, iters, sink);
        double r128 = run<128>(buf, bytes, blocks, iters, sink);
        printf("  random gathers/s: 4B %.2fG (%.0f GB/s useful)  8B %.2fG  16B %.2fG  32B %.2fG (%.0f GB/s at 32B)"
               "  64B %.2fG (%.0f GB/s)  128B %.2fG (%.0f GB/s)\n",
               r4 / 1e9, r4 * 4 / 1e9, r8 / 1e9, r16 / 1e9, r32 / 1e9, r32 * 32 / 1e9, r64 / 1e9,
               r64 * 64 / 1e9, r128 / 1e9, r128 * 128 / 1e9);
    }
    // dependent chains at full occupancy
    for (int bpsm : {8, 16}) {
        int bl = sms * bpsm;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        chase<<<bl, 256>>>(buf, bytes / 32, 64, 1, sink);
        cudaEventRecord(a);
        chase<<<bl, 256>>>(buf, bytes / 32, 64, 2, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double n = (double)bl * 256 * 64;
        printf("dependent 16B chase, %d lanes: %.2f G loads/s (%.1f ns per load per lane)\n", bl * 256,
               n / (ms * 1e-3) / 1e9, ms * 1e6 / 64);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}

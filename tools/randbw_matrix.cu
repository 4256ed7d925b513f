// Random-gather counter matrix (measurement only): does any
// load flavour, L2 cache hint, prefetch-size qualifier or fetch-granularity
// limit make a random 4 B / 32 B request that misses L2 cost less than a
// 128 B DRAM line on B200?
//
// Every variant is one launch of the same gather loop (independent random
// requests over a 32 GiB buffer, far beyond L2), differing only in the load
// instruction.  Run once plainly for throughput, then under ncu for the
// per-request counters:
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/randbw_matrix tools/randbw_matrix.cu
//   tools/randbw_matrix 32            # requests/s per variant
//   ncu --clock-control none --metrics <see tools/randbw_matrix.sh> tools/randbw_matrix 32 1
//
// Variants (v = id):
//   0 ld.global.cg.u32            (the walk kernels' flavour, 4 B)
//   1 ld.global.ca.u32            (L1-allocating)
//   2 ld.global.nc.u32            (read-only path, __ldg)
//   3 ld.global.nc.L1::no_allocate.u32
//   4 ld.global.cs.u32            (streaming: evict-first in L1 and L2)
//   5 ld.global.lu.u32            (last use)
//   6 ld.global.L2::cache_hint.u32, createpolicy evict_first
//   7 ld.global.cg.L2::64B.u32    (prefetch-size qualifier)
//   8 ld.global.cg.L2::128B.u32
//   9 ld.global.cg.L2::256B.u32
//  10 ld.global.cg.v4.u32         (16 B)
//  11 ld.global.cg.v8.u32         (32 B, one 256-bit request; the walk kernels' bucket load)
//  12 ld.global.cg.L2::64B.v8.u32
//  13 ld.global.L2::cache_hint.v8.u32, evict_first
//  14 variant 0 with cudaLimitMaxL2FetchGranularity = 32
//  15 variant 11 with cudaLimitMaxL2FetchGranularity = 32
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <int V>
__device__ __forceinline__ uint32_t load(const uint32_t* p, uint64_t pol) {
    uint32_t v = 0;
    if constexpr (V == 0 || V == 14) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 1) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 2) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 3) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 4) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 5) asm volatile("ld.global.lu.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 6) asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    else if constexpr (V == 7) asm volatile("ld.global.cg.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 8) asm volatile("ld.global.cg.L2::128B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 9) asm volatile("ld.global.cg.L2::256B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (V == 10) {
        uint32_t a, b, c, d;
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
        v = a ^ d;
    } else {
        uint32_t a, b, c, d, e, f, g, h;
        if constexpr (V == 11 || V == 15)
            asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
        else if constexpr (V == 12)
            asm volatile("ld.global.cg.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
        else
            asm volatile("ld.global.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h)
                         : "l"(p), "l"(pol));
        v = a ^ h;
    }
    return v;
}

// bytes per request of a variant (the slot size the addresses are aligned to)
__host__ __device__ constexpr int req_bytes(int v) { return v == 10 ? 16 : (v >= 11 && v != 14) ? 32 : 4; }

template <int V>
__global__ void gather(const uint32_t* __restrict__ buf, uint64_t nslots, int iters, uint64_t seed,
                       unsigned long long* sink) {
    uint64_t pol = 0;
    if constexpr (V == 6 || V == 13) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint64_t s = mix(seed ^ (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x));
    uint32_t acc = 0;
    constexpr uint64_t words = req_bytes(V) / 4;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        s += 0x9E3779B97F4A7C15ULL;
        const uint64_t slot = __umul64hi(mix(s), nslots);
        acc += load<V>(buf + slot * words, pol);
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int V>
double run(const uint32_t* buf, uint64_t bytes, int blocks, int iters, int reps, unsigned long long* sink) {
    const uint64_t nslots = bytes / req_bytes(V);
    if (V == 14 || V == 15) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    if (reps > 1) gather<V><<<blocks, 256>>>(buf, nslots, iters, 1, sink);  // warm-up
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) gather<V><<<blocks, 256>>>(buf, nslots, iters, 2 + r, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (V == 14 || V == 15) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 64);
    size_t lim = 0;
    cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
    const double n = double(reps) * blocks * 256.0 * iters;
    const double rate = n / (ms * 1e-3);
    printf("variant %2d  %2d B requests  %.2f G requests/s  (%.0f GB/s of requested bytes)  [limit now %zu]\n", V,
           req_bytes(V), rate / 1e9, rate * req_bytes(V) / 1e9, lim);
    return rate;
}

int main(int argc, char** argv) {
    const uint64_t gib = argc > 1 ? strtoull(argv[1], nullptr, 10) : 32;
    const int once = argc > 2 ? atoi(argv[2]) : 0;  // 1: one launch per variant (ncu)
    const uint64_t bytes = gib << 30;
    uint32_t* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8;
    const int iters = once ? 64 : 256;
    const int reps = once ? 1 : 3;
    size_t lim = 0;
    cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
    printf("buffer %llu GiB, %d blocks x 256 threads x %d requests, default L2 fetch granularity limit %zu\n",
           (unsigned long long)gib, blocks, iters, lim);
    run<0>(buf, bytes, blocks, iters, reps, sink);
    run<1>(buf, bytes, blocks, iters, reps, sink);
    run<2>(buf, bytes, blocks, iters, reps, sink);
    run<3>(buf, bytes, blocks, iters, reps, sink);
    run<4>(buf, bytes, blocks, iters, reps, sink);
    run<5>(buf, bytes, blocks, iters, reps, sink);
    run<6>(buf, bytes, blocks, iters, reps, sink);
    run<7>(buf, bytes, blocks, iters, reps, sink);
    run<8>(buf, bytes, blocks, iters, reps, sink);
    run<9>(buf, bytes, blocks, iters, reps, sink);
    run<10>(buf, bytes, blocks, iters, reps, sink);
    run<11>(buf, bytes, blocks, iters, reps, sink);
    run<12>(buf, bytes, blocks, iters, reps, sink);
    run<13>(buf, bytes, blocks, iters, reps, sink);
    run<14>(buf, bytes, blocks, iters, reps, sink);
    run<15>(buf, bytes, blocks, iters, reps, sink);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}

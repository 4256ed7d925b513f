// Random 32 B requests/s against the footprint they are spread over
// (measurement only): separates the DRAM request-rate
// ceiling from address-translation (TLB) effects of multi-GB random access.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/randbw_sizes tools/randbw_sizes.cu
//   tools/randbw_sizes 96          (largest footprint in GiB)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <bool L64>
__global__ void gather(const uint32_t* __restrict__ buf, uint64_t nslots, int iters, uint64_t seed,
                       unsigned long long* sink) {
    uint64_t s = mix(seed ^ (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x));
    uint32_t acc = 0;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        s += 0x9E3779B97F4A7C15ULL;
        const uint64_t slot = __umul64hi(mix(s), nslots);
        uint32_t a, b, c, d, e, f, g, h;
        if (L64)
            asm volatile("ld.global.cg.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h)
                         : "l"(buf + slot * 8));
        else
            asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h)
                         : "l"(buf + slot * 8));
        acc += a ^ h;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <bool L64>
double rate(const uint32_t* buf, uint64_t bytes, int blocks, unsigned long long* sink) {
    const int iters = 256;
    const uint64_t nslots = bytes / 32;
    gather<L64><<<blocks, 256>>>(buf, nslots, iters, 1, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) gather<L64><<<blocks, 256>>>(buf, nslots, iters, 2 + r, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return 3.0 * blocks * 256.0 * iters / (ms * 1e-3);
}

int main(int argc, char** argv) {
    const double max_gib = argc > 1 ? atof(argv[1]) : 96;
    uint64_t max_bytes = static_cast<uint64_t>(max_gib * (1ull << 30));
    uint32_t* buf = nullptr;
    if (cudaMalloc(&buf, max_bytes) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(buf, 1, max_bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (double gib : {0.25, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0, 96.0}) {
        if (gib > max_gib) break;
        const uint64_t bytes = static_cast<uint64_t>(gib * (1ull << 30));
        for (int bpsm : {4, 8}) {
            const double r = rate<false>(buf, bytes, sms * bpsm, sink);
            const double r64 = rate<true>(buf, bytes, sms * bpsm, sink);
            printf("footprint %6.2f GiB  %d blocks/SM  32 B requests: %.2f G/s   .L2::64B: %.2f G/s\n", gib, bpsm,
                   r / 1e9, r64 / 1e9);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}

// Device->host bandwidth: cudaMemcpyAsync (copy engine) vs a kernel storing
// straight into mapped pinned memory (16 B vector stores), for the end-to-end
// path's design choice.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zerocopy_bw tools/zerocopy_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_store(const uint4* __restrict__ src, uint4* dst, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = 26u << 20;
    void *d, *h;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("memcpy D2H   %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
    }
    for (int blocks : {148, 296, 592, 1184, 2368}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_store<<<blocks, 256>>>((const uint4*)d, (uint4*)h, bytes / 16);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("kernel store %4d blocks %.3f ms  %.1f GB/s\n", blocks, ms, bytes / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

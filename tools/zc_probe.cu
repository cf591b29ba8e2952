// Probe: bandwidth of SM-initiated 16-byte reads of pinned (mapped) host
// memory over PCIe vs cudaMemcpyAsync H2D, 18 MB (the C2 image).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_probe tools/zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void sum_kernel(const uint4* __restrict__ p, size_t n16, unsigned* out)
{
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = p[i];
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u)
        out[0] = acc;
}

int main()
{
    const size_t n = 5184ull * 3456ull;
    unsigned char* h;
    cudaHostAlloc(&h, n, cudaHostAllocMapped);
    for (size_t i = 0; i < n; ++i)
        h[i] = (unsigned char)(i * 131);
    unsigned char* d;
    cudaMalloc(&d, n);
    unsigned* out;
    cudaMalloc(&out, 4);
    unsigned char* hd;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i)
            cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("memcpy H2D: %.1f us  %.1f GB/s\n", ms * 100, n * 10 / ms / 1e6);
        for (int blocks_per_sm : {1, 2, 4, 8}) {
            for (int threads : {256, 512, 1024}) {
                sum_kernel<<<sms * blocks_per_sm, threads>>>((const uint4*)hd, n / 16, out);
                cudaEventRecord(a);
                for (int i = 0; i < 10; ++i)
                    sum_kernel<<<sms * blocks_per_sm, threads>>>((const uint4*)hd, n / 16, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                printf("zero-copy %d x %d: %.1f us  %.1f GB/s\n", blocks_per_sm, threads, ms * 100,
                       n * 10 / ms / 1e6);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

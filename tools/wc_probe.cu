// Pinned H2D rate of a C2-sized copy from default, write-combined and
// portable|mapped pinned host memory (is the e2e path's PCIe floor the same
// for every kind of pinned buffer?).
// Build: nvcc -O3 -o tools/wc_probe tools/wc_probe.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
int main()
{
    const size_t n = 5184ull * 3456ull;
    void* d;
    CK(cudaMalloc(&d, n));
    const unsigned flags[3] = {cudaHostAllocDefault, cudaHostAllocWriteCombined, cudaHostAllocPortable | cudaHostAllocMapped};
    const char* names[3] = {"default", "write_combined", "portable_mapped"};
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int k = 0; k < 3; ++k) {
        void* h;
        CK(cudaHostAlloc(&h, n, flags[k]));
        std::memset(h, 0x5a, n);
        for (int i = 0; i < 20; ++i) CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        float best = 1e30f, tot = 0;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0, s));
            for (int i = 0; i < 20; ++i) CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
            tot += ms;
        }
        std::printf("{\"pinned\":\"%s\",\"best_gbs\":%.2f,\"mean_gbs\":%.2f}\n", names[k], 20.0 * n / (best * 1e6), 100.0 * n / (tot * 1e6));
        CK(cudaFreeHost(h));
    }
    return 0;
}

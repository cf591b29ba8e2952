// Debug harness for the cluster-reduced small-image path (K1 single images):
// runs a few shapes through the C ABI and reports CUDA errors per call.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKOHLER_WALK_THREADS=512 -Iinclude -o X tools/cluster_debug.cu
// (KOHLER_NO_CLUSTER=1 X: the same shapes through the ticket path)
#include "../paper_1707_05062_b200/csrc/kohler_kernels.cu"
#include <vector>
int main()
{
    kohler_cuda_ctx* ctx = nullptr;
    if (kohler_cuda_create(0, &ctx)) { printf("%s\n", kohler_cuda_last_error()); return 1; }
    printf("no_cluster %d\n", (int)ctx->no_cluster);
    const int shapes[][2] = {{16, 1}, {100, 37}, {512, 512}};
    for (auto& s : shapes) {
        const int w = s[0], h = s[1];
        std::vector<uint8_t> img((size_t)w * h);
        uint32_t x = 7;
        for (auto& v : img) { x = x * 1664525u + 1013904223u; v = (uint8_t)(x >> 24); }
        uint8_t* d; cudaMalloc(&d, img.size() + 64); cudaMemcpy(d, img.data(), img.size(), cudaMemcpyHostToDevice);
        uint64_t* sums; cudaMalloc(&sums, 4096);
        int* ints; cudaMalloc(&ints, 256);
        int rc = kohler_cuda_analyze_batch_device(ctx, d, 1, w, h, w, (size_t)w * h, 6, sums, sums + 256, nullptr, nullptr, ints, ints + 8, ints + 16, ints + 24, 0);
        cudaError_t e = cudaDeviceSynchronize();
        uint64_t hs[256]; cudaMemcpy(hs, sums, 2048, cudaMemcpyDeviceToHost);
        unsigned long long tot = 0; for (int i = 0; i < 256; ++i) tot += hs[i];
        printf("%dx%d rc %d (%s) sync %s grid %d sum-of-sums %llu\n", w, h, rc, rc ? kohler_cuda_last_error() : "", cudaGetErrorString(e), ctx->last_grid, tot);
        if (e != cudaSuccess) return 2;
    }
    return 0;
}

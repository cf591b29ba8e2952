// Debug probe of the K5 tile kernel: per-CTA clock64 totals of the
// accumulation phase, the reduce phase, and the rest, for n images of w x h.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKOHLER_PHASES -DKOHLER_WALK_THREADS=512 -Iinclude -o tools/tile_probe tools/tile_probe.cu
#include "../paper_1707_05062_b200/csrc/kohler_kernels.cu"
#include <vector>
int main(int argc, char** argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 65536, w = argc > 2 ? atoi(argv[2]) : 128,
              h = argc > 3 ? atoi(argv[3]) : 128;
    kohler_cuda_ctx* ctx = nullptr;
    if (kohler_cuda_create(0, &ctx)) { printf("%s\n", kohler_cuda_last_error()); return 1; }
    const int fam = argc > 4 ? atoi(argv[4]) : 0;  // 1: the four C5 families by i mod 4
    std::vector<uint8_t> img((size_t)n * w * h);
    uint32_t x = 1;
    auto rnd = [&]() { x = x * 1664525u + 1013904223u; return x >> 8; };
    if (!fam) {
        for (auto& v : img) v = (uint8_t)(rnd() >> 16);
    } else {
        for (int i = 0; i < n; ++i) {
            uint8_t* im = img.data() + (size_t)i * w * h;
            const int f = i & 3, cell = 1 + (int)(rnd() % 8), cval = (int)(rnd() % 256);
            int band = 0, left = 0;
            for (int yy = 0; yy < h; ++yy) {
                if (f == 0 && left-- <= 0) { band = (int)(rnd() % 3); left = 1 + (int)(rnd() % 20); }
                for (int xx = 0; xx < w; ++xx) {
                    int v;
                    if (f == 0) v = band == 0 ? 0 : band == 1 ? 128 : 255;
                    else if (f == 1) v = cval;
                    else if (f == 2) v = ((xx / cell + yy / cell) & 1) ? 255 : 0;
                    else { const int s = (int)(rnd() % 31) - 15 + (int)(rnd() % 31) - 15; v = ((rnd() & 1) ? 60 : 190) + s / 2; }
                    im[(size_t)yy * w + xx] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
                }
            }
        }
    }
    uint8_t* d; cudaMalloc(&d, img.size()); cudaMemcpy(d, img.data(), img.size(), cudaMemcpyHostToDevice);
    uint64_t* sums; cudaMalloc(&sums, (size_t)n * 4096);
    int* ints; cudaMalloc(&ints, (size_t)n * 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        kohler_cuda_analyze_batch_device(ctx, d, n, w, h, w, (size_t)w * h, 6, sums, sums + (size_t)n * 256, nullptr, nullptr, ints, ints + n, ints + 2 * n, ints + 3 * n, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); printf("batch %.3f ms (%.1f Gpx/s)\n", ms, (double)n * w * h / ms / 1e6);
    }
    static unsigned long long ph[2048][12];
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    double t[5] = {0}; int G = 147;
    for (int c = 0; c < G; ++c) for (int i = 0; i < 5; ++i) t[i] += ph[c][i];
    printf("K5 per-CTA cycles: walk %.0f, read+clear %.0f, scratch %.0f, K3 %.0f, clear %.0f\n",
           t[0] / G, t[1] / G, t[2] / G, t[3] / G, t[4] / G);
    return 0;
}

// Phase probe (debug only): builds kohler_kernels.cu with KOHLER_PHASES and
// prints per-CTA globaltimer phase durations of the fused launch on a
// C2-sized image: [0] start -> [1] histogram zeroed (first loads in flight)
// -> [2] main loop done -> [3] CTA exit (flush, and for the last CTA the
// reconstruction + selection).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKOHLER_PHASES \
//        -Iinclude -o tools/phase_probe tools/phase_probe.cu
#include "../paper_1707_05062_b200/csrc/kohler_kernels.cu"

#include <algorithm>
#include <vector>

int main(int argc, char** argv)
{
    const int w = argc > 1 ? atoi(argv[1]) : 5184, h = argc > 2 ? atoi(argv[2]) : 3456;
    const int reps = 20;
    if (argc > 3) { int rot = atoi(argv[3]); cudaMemcpyToSymbol(g_rot, &rot, sizeof(int)); }
    kohler_cuda_ctx* ctx = nullptr;
    if (kohler_cuda_create(0, &ctx)) { printf("create: %s\n", kohler_cuda_last_error()); return 1; }
    size_t pitch = (w + 127) / 128 * 128;
    std::vector<uint8_t> img(pitch * h);
    uint32_t x = 12345;
    for (int y = 0; y < h; ++y)
        for (int i = 0; i < w; ++i) {
            x = x * 1664525u + 1013904223u;
            int v = (i * 200 / w + y * 200 / h) / 2 + (int)((x >> 24) % 11) - 5;
            img[(size_t)y * pitch + i] = (uint8_t)std::min(255, std::max(0, v));
        }
    const int copies = 12;
    uint8_t* d; cudaMalloc(&d, pitch * h * copies);
    for (int c = 0; c < copies; ++c) cudaMemcpy(d + c * pitch * h, img.data(), pitch * h, cudaMemcpyHostToDevice);
    uint64_t* out; cudaMalloc(&out, 8192);
    int* ints; cudaMalloc(&ints, 256);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < 5; ++r)
        kohler_cuda_analyze_batch_device(ctx, d + (r % copies) * pitch * h, 1, w, h, pitch, pitch * h, 6, out, out + 256, nullptr, nullptr, ints, ints + 8, ints + 1, ints + 2, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(a, st);
    for (int r = 0; r < 200; ++r)
        kohler_cuda_analyze_batch_device(ctx, d + (r % copies) * pitch * h, 1, w, h, pitch, pitch * h, 6, out, out + 256, nullptr, nullptr, ints, ints + 8, ints + 1, ints + 2, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("pipelined (PDL) back-to-back: %.2f us/step\n", ms * 1000 / 200);
    {
        // phases of the last pipelined launch (warm instruction / constant caches)
        static unsigned long long pp[2048][12];
        cudaMemcpyFromSymbol(pp, g_phase, sizeof(pp));
        const int G = ctx->last_grid;
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < G; ++c) t0 = std::min(t0, pp[c][0]);
        double pro = 0, zl = 0, sy = 0, mn = 0, fl = 0, mx = 0, pk = 0;
        for (int c = 0; c < G; ++c) {
            pk += (pp[c][6] - pp[c][0]) / 1e3;
            pro += (pp[c][4] - pp[c][0]) / 1e3;
            zl += (pp[c][5] - pp[c][4]) / 1e3;
            sy += (pp[c][1] - pp[c][5]) / 1e3;
            mn += (pp[c][2] - pp[c][1]) / 1e3;
            fl += (pp[c][3] - pp[c][2]) / 1e3;
            mx = std::max(mx, (pp[c][3] - t0) / 1e3);
        }
        printf("raw stamp mod 1000 ns (CTA 0..5, phases 0,4,5,1): ");
        for (int c = 0; c < 6; ++c)
            printf("[%llu %llu %llu %llu] ", pp[c][0] % 1000, pp[c][4] % 1000, pp[c][5] % 1000, pp[c][1] % 1000);
        printf("\n");
        {
            static unsigned long long se[2][256];
            static unsigned smid[2048];
            unsigned nl = 0;
            cudaMemcpyFromSymbol(se, g_sm_end, sizeof(se));
            cudaMemcpyFromSymbol(smid, g_smid, sizeof(smid));
            cudaMemcpyFromSymbol(&nl, g_launch, sizeof(nl));
            double gap = 0, gmax = 0, red = 0, bor = 0, pw = 0, tail = 0, ex = 0;
            for (int c = 0; c < G; ++c) {
                const double g = ((long long)pp[c][0] - (long long)se[nl & 1][smid[c] & 255]) / 1e3;
                gap += g; gmax = std::max(gmax, g);
                red += (pp[c][8] - pp[c][2]) / 1e3;
                bor += (pp[c][9] - pp[c][8]) / 1e3;
                pw += (pp[c][10] - pp[c][9]) / 1e3;
                tail += (pp[c][3] - pp[c][10]) / 1e3;
                ex += (pp[c][7] - pp[c][3]) / 1e3;
            }
            printf("pipelined: previous CTA exit on the SM -> this CTA start: avg %.2f max %.2f us\n", gap / G, gmax);
            {
                static long long cy[2048][8];
                cudaMemcpyFromSymbol(cy, g_cyc, sizeof(cy));
                double d[7] = {0};
                for (int c = 0; c < G; ++c) {
                    d[0] += cy[c][0] - cy[c][4]; d[1] += cy[c][1] - cy[c][0]; d[2] += cy[c][2] - cy[c][1];
                    d[3] += cy[c][3] - cy[c][2]; d[4] += cy[c][5] - cy[c][3]; d[5] += cy[c][6] - cy[c][5];
                }
                printf("border cycles (thread 0): slice %.0f, loads %.0f, atomics %.0f, loop end %.0f, return %.0f, barrier %.0f\n",
                       d[0] / G, d[1] / G, d[2] / G, d[3] / G, d[4] / G, d[5] / G);
            }
            printf("pipelined flush split: reduce %.2f, border %.2f, pdl_wait %.2f, combos+REDG %.2f, to exit %.2f us (avg)\n",
                   red / G, bor / G, pw / G, tail / G, ex / G);
        }
        printf("pipelined: kernel setup %.2f of ", pk / G);
        printf("pipelined last launch: prologue %.2f, zero loop %.2f, barrier %.2f, main %.2f, flush %.2f us (avg); "
               "first start -> last flush end %.2f us\n", pro / G, zl / G, sy / G, mn / G, fl / G, mx);
    }
    std::vector<double> tot;
    for (int r = 0; r < reps; ++r) {
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        kohler_cuda_analyze_batch_device(ctx, d + (r % copies) * pitch * h, 1, w, h, pitch, pitch * h, 6, out, out + 256, nullptr, nullptr, ints, ints + 8, ints + 1, ints + 2, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        tot.push_back(ms * 1000);
    }
    std::sort(tot.begin(), tot.end());
    printf("isolated launch (event): median %.2f us\n", tot[reps / 2]);
    static unsigned long long ph[2048][12];
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    const int G = ctx->last_grid;
    printf("grid %d CTAs\n", G);
    unsigned long long t0 = ~0ull, tend = 0;
    for (int c = 0; c < G; ++c) { t0 = std::min(t0, ph[c][0]); tend = std::max(tend, ph[c][7]); }
    auto us = [&](int c, int i) { return (ph[c][i] - t0) / 1e3; };
    double lastStart = 0, avgZero = 0, avgMain = 0, mainMin = 1e9, mainMax = 0, avgFlush = 0;
    int lastCta = -1;
    for (int c = 0; c < G; ++c) {
        lastStart = std::max(lastStart, us(c, 0));
        avgZero += us(c, 1) - us(c, 0);
        avgMain += us(c, 2) - us(c, 1);
        mainMin = std::min(mainMin, us(c, 2)); mainMax = std::max(mainMax, us(c, 2));
        avgFlush += us(c, 3) - us(c, 2);
    }
    {
        double pro = 0, zl = 0, sy = 0;
        for (int c = 0; c < G; ++c) {
            pro += us(c, 4) - us(c, 0);
            zl += us(c, 5) - us(c, 4);
            sy += us(c, 1) - us(c, 5);
        }
        printf("zero phase split (thread 0): prologue %.2f, zero loop %.2f, barrier wait %.2f us\n",
               pro / G, zl / G, sy / G);
    }
    printf("last CTA start +%.2f us; avg zero %.2f; avg main %.2f; main done min %.2f max %.2f; avg flush %.2f; total %.2f us\n",
           lastStart, avgZero / G, avgMain / G, mainMin, mainMax, avgFlush / G, (tend - t0) / 1e3);
    {
        static unsigned smid[2048];
        cudaMemcpyFromSymbol(smid, g_smid, sizeof(smid));
        std::vector<std::pair<double, int>> v;
        for (int c = 0; c < G; ++c) v.push_back({us(c, 2) - us(c, 1), c});
        std::sort(v.begin(), v.end());
        printf("main-loop us by CTA (sorted): ");
        for (int i = 0; i < (int)v.size(); i += std::max(1, (int)v.size() / 16)) printf("%.1f ", v[i].first);
        printf("| max %.1f\nslowest CTAs (cta/sm): ", v.back().first);
        for (int i = (int)v.size() - 1; i >= std::max(0, (int)v.size() - 8); --i) printf("%d/%u ", v[i].second, smid[v[i].second]);
        printf("\nfastest CTAs (cta/sm): ");
        for (int i = 0; i < std::min(8, (int)v.size()); ++i) printf("%d/%u ", v[i].second, smid[v[i].second]);
        printf("\n");
    }
    {
        static unsigned long long we[2048][32];
        cudaMemcpyFromSymbol(we, g_wend, sizeof(we));
        const int nw = kWalkWarps;
        double spread = 0, avgw = 0;
        for (int c = 0; c < G; ++c) {
            double mn = 1e18, mx = 0;
            for (int w2 = 0; w2 < nw; ++w2) {
                const double t = (we[c][w2] - ph[c][1]) / 1e3;
                mn = std::min(mn, t); mx = std::max(mx, t);
                avgw += t;
            }
            spread += mx - mn;
        }
        printf("warp walk end (us after zeroing): avg %.2f, avg per-CTA spread max-min %.2f\n", avgw / (G * nw), spread / G);
    }
    if (lastCta >= 0)
        printf("tail CTA %d: flush done %.2f, acc read %.2f, scans+mean %.2f, select %.2f, end %.2f us\n", lastCta,
               us(lastCta, 3), us(lastCta, 4), us(lastCta, 5), us(lastCta, 6), us(lastCta, 7));
    return 0;
}

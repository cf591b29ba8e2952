// Debug probe: cycles of the per-image finish (scans + mean + selection) on
// one CTA, single-warp register version vs the block-parallel version.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -o tools/finish_probe tools/finish_probe.cu
#include "../paper_1707_05062_b200/csrc/kohler_kernels.cu"

__global__ void __launch_bounds__(512) probe(const long long* combos, unsigned long long* cyc,
                                             int* outs, double* vals, int mode)
{
    __shared__ long long sval[512];
    __shared__ double mean[256];
    __shared__ uint8_t def[256];
    __shared__ __align__(16) unsigned char scr[256 * 24 + 256];
    __shared__ uint64_t csum[256], ccard[256];
    __shared__ long long tmp[256];
    const int tid = threadIdx.x;
    sval[tid] = combos[tid];
    __syncthreads();
    unsigned long long t0 = clock64(), t1 = 0, t2 = 0;
    if (mode == 0) {
        if (tid < 32) {
            uint64_t card[8], sum[8];
            warp_curve256_regs([&](int t) { return sval[t]; }, [&](int u) { return sval[256 + u]; },
                               card, sum);
            double v[8];
            bool d[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                d[j] = card[j] != 0;
                v[j] = d[j] ? (double)sum[j] / (double)card[j] : 0.0;
                vals[8 * tid + j] = v[j];
            }
            t1 = clock64();
            kohler_walk::warp_select256_regs(v, d, 6, reinterpret_cast<double*>(scr),
                                             reinterpret_cast<int*>(scr + 1024), outs, outs + 1, outs + 7);
            t2 = clock64();
        }
    } else {
        const int warp = tid >> 5;
        if (warp == 0)
            warp_prefix256(sval, reinterpret_cast<long long*>(ccard));
        else if (warp == 1) {
            warp_prefix256(sval + 256, tmp);
            __syncwarp();
            warp_prefix256(tmp, reinterpret_cast<long long*>(csum));
        }
        __syncthreads();
        if (tid < 256) {
            const double v = ccard[tid] ? (double)csum[tid] / (double)ccard[tid] : 0.0;
            mean[tid] = v;
            def[tid] = ccard[tid] ? 1 : 0;
            vals[tid] = v;
        }
        __syncthreads();
        t1 = clock64();
        if (tid < 256)
            block_select256(mean, def, 6, scr, 1, outs, outs + 1, outs + 7);
        __syncthreads();
        t2 = clock64();
    }
    if (tid == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
    }
}

int main()
{
    // combos of a noisy curve: random pixel-pair multiset
    std::vector<long long> c(512, 0);
    uint32_t x = 1;
    auto rnd = [&]() { x = x * 1664525u + 1013904223u; return x >> 8; };
    for (int i = 0; i < 200000; ++i) {
        int a = rnd() % 256, b = (a + (int)(rnd() % 21) - 10 + 256) % 256;
        int lo = a < b ? a : b, hi = a < b ? b : a;
        c[lo] += 1; c[hi] -= 1;  // card first difference
        if (lo < hi) {
            c[256 + lo + 1] += 1; c[256 + hi + 1 < 512 ? 256 + hi + 1 : 511] += 0;
        }
    }
    long long* dc; cudaMalloc(&dc, 4096); cudaMemcpy(dc, c.data(), 4096, cudaMemcpyHostToDevice);
    unsigned long long* cyc; cudaMalloc(&cyc, 16);
    int* outs; cudaMalloc(&outs, 64);
    double* vals; cudaMalloc(&vals, 2048);
    for (int mode = 0; mode < 2; ++mode) {
        for (int r = 0; r < 3; ++r) probe<<<1, 512>>>(dc, cyc, outs, vals, mode);
        cudaDeviceSynchronize();
        unsigned long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
        int o[8]; cudaMemcpy(o, outs, 32, cudaMemcpyDeviceToHost);
        printf("mode %s: scans+mean %llu cyc, select %llu cyc, t0 %d topk %d %d %d .. n %d\n",
               mode == 0 ? "warp" : "block", h[0], h[1], o[0], o[1], o[2], o[3], o[7]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// LSU-side floor of K1's per-step mix: every warp, per
// iteration, does what one K1 ring position does on the shared-memory pipe --
// 48 lane-striped shared atomics on random rows, one 512-byte row arriving in
// its ring, one LDS.128 of an earlier row, optionally two SHFL -- with (almost)
// no ALU work.  The row arrives by
//   mode 0: nothing (atomics only)
//   mode 1: per-lane 16-byte cp.async (LDGSTS.BYPASS), as K1 ships
//   mode 2: one 512-byte cp.async.bulk (TMA) per warp, mbarrier completion
//   mode 3: per-lane LDG.128 straight into registers (no ring)
//   mode 4: K5's pattern with cp.async: 8 lane groups x 64 B from 8 different images
//           (16 KiB apart) + one 16-byte pad copy per group (8 lanes)
//   mode 5: K5's pattern with one 80-byte cp.async.bulk per group (8 per warp row)
// Output: cycles per iteration per SM (16 warps), i.e. the floor of a K1 step
// if nothing but the memory side mattered.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ void red_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }

constexpr int kWarps = 16;
constexpr uint32_t kHist = 128 * 1024;          // counter block
constexpr uint32_t kRing = kWarps * 4 * 640;    // 4 slots x 640 B per warp
constexpr uint32_t kBars = kWarps * 4 * 8;

template <int MODE, bool SHFL>
__global__ void __launch_bounds__(512, 1) probe(uint32_t* out, const uint4* src, size_t rows_per_warp,
                                                int iters, long long* cyc)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < (int)(kHist / 4); i += blockDim.x) hist[i] = 0;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t ring = base + kHist + warp * 2560u;
    const uint32_t bars = base + kHist + kRing + warp * 32u;
    if ((MODE == 2 || MODE == 5) && lane == 0) {
        for (int s = 0; s < 4; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8u * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t seed = mix(blockIdx.x * 4096 + threadIdx.x * 7 + 1);
    // 48 precomputed counter addresses; the per-iteration perturbation x only
    // flips bits 7..9 (base is 1 KiB aligned, so the address stays in its block)
    uint32_t a[16], b[16], c[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        a[j] = base + (mix(seed + j * 0x9e3779b9u) & 1023u) * 128u + lane * 4u;
        b[j] = base + (mix(seed + j * 0x85ebca6bu + 17) & 1023u) * 128u + lane * 4u;
        c[j] = base + (mix(seed + j * 0xc2b2ae35u + 91) & 1023u) * 128u + lane * 4u;
    }
    // this warp's source rows: 512 B each, consecutive
    const uint4* g = src + ((size_t)(blockIdx.x * kWarps + warp) * rows_per_warp) * 32;
    auto fetch = [&](int it) {
        const uint4* row = g + (size_t)(it & 511) * 32;
        const uint32_t slot = ring + (uint32_t)(it & 3) * 640u;
        if (MODE == 1) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot + lane * 16u), "l"(row + lane)
                         : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else if (MODE == 4) {
            // group g = lane / 4 reads image g (16 KiB apart), 64 B per row; pads by lig == 3
            const unsigned char* img = reinterpret_cast<const unsigned char*>(g) + (size_t)(lane >> 2) * 16384 +
                                       (size_t)(it & 127) * 128;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot + lane * 16u),
                         "l"(img + (lane & 3) * 16)
                         : "memory");
            if ((lane & 3) == 3)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot + 512u + (lane >> 2) * 16u),
                             "l"(img + 64)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else if (MODE == 5) {
            const uint32_t bar = bars + 8u * (it & 3);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 640;" ::"r"(bar) : "memory");
            __syncwarp();
            if ((lane & 3) == 0) {
                const unsigned char* img = reinterpret_cast<const unsigned char*>(g) + (size_t)(lane >> 2) * 16384 +
                                           (size_t)(it & 127) * 128;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 80, [%2];" ::"r"(
                        slot + (lane >> 2) * 80u),
                    "l"(img), "r"(bar)
                    : "memory");
            }
        } else if (MODE == 2) {
            if (lane == 0) {
                const uint32_t bar = bars + 8u * (it & 3);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(bar) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(slot),
                    "l"(row), "r"(bar)
                    : "memory");
            }
        }
    };
    uint4 pre[3];
    if (MODE == 3) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
            pre[k] = __ldg(g + (size_t)k * 32 + lane);
    } else if (MODE != 0) {
        fetch(0);
        fetch(1);
        fetch(2);
    }
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint4 r = make_uint4(0, 0, 0, 0);
        const uint32_t slot = ring + (uint32_t)(it & 3) * 640u + (MODE == 5 ? (lane >> 2) * 80u + (lane & 3) * 16u : lane * 16u);
        if (MODE == 1 || MODE == 4) {
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncwarp();
        } else if (MODE == 2 || MODE == 5) {
            const uint32_t bar = bars + 8u * (it & 3);
            const uint32_t parity = (uint32_t)(it >> 2) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra W;\n\t}" ::"r"(bar),
                "r"(parity)
                : "memory");
            __syncwarp();
        }
        if (MODE == 1 || MODE == 2 || MODE == 4 || MODE == 5) {
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                         : "r"(slot)
                         : "memory");
            fetch(it + 3);
        } else if (MODE == 3) {
            r = pre[0];
            pre[0] = pre[1];
            pre[1] = pre[2];
            pre[2] = __ldg(g + (size_t)((it + 3) & 511) * 32 + lane);
        }
        if (SHFL) {
            r.y ^= __shfl_up_sync(0xFFFFFFFFu, r.w, 1);
            r.z ^= __shfl_down_sync(0xFFFFFFFFu, r.x, 1);
        }
        // the loaded data perturbs the rows a little (keeps the loads live, the lane stripe intact)
        const uint32_t x = ((r.x ^ r.y ^ r.z ^ r.w) & 7u) << 7;
        acc += x;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            red_inc(a[j] ^ x);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            red_inc(b[j] ^ x);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            red_inc(c[j] ^ x);
    }
    const long long t1 = clock64();
    if (MODE == 1 || MODE == 4)
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (MODE == 2 || MODE == 5) {
        // drain the three copies still in flight
        for (int it = iters; it < iters + 3; ++it) {
            const uint32_t bar = bars + 8u * (it & 3);
            const uint32_t parity = (uint32_t)(it >> 2) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra W2;\n\t}" ::"r"(bar),
                "r"(parity)
                : "memory");
        }
    }
    __syncthreads();
    uint32_t s = acc + pre[0].x * (MODE == 3);
    for (int i = threadIdx.x; i < (int)(kHist / 4); i += blockDim.x) s += hist[i];
    atomicAdd(out, s);
    if (threadIdx.x == 0)
        cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, bool SHFL>
void run(const char* name, uint32_t* d, const uint4* src, size_t rows_per_warp, int sms, long long* dcyc)
{
    const int iters = 4096;
    const size_t smem = kHist + kRing + kBars;
    CK(cudaFuncSetAttribute(probe<MODE, SHFL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe<MODE, SHFL><<<sms, 512, smem>>>(d, src, rows_per_warp, 64, dcyc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        probe<MODE, SHFL><<<sms, 512, smem>>>(d, src, rows_per_warp, iters, dcyc);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    long long* h = (long long*)std::malloc(sizeof(long long) * sms);
    CK(cudaMemcpy(h, dcyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double cs = 0;
    for (int i = 0; i < sms; ++i) cs += (double)h[i];
    std::free(h);
    // a K1 "step" is one warp iteration (512 px); per SM, 16 warps run concurrently
    const double cyc_per_step = cs / sms / iters / kWarps;
    std::printf("{\"mode\":\"%s\",\"shfl\":%d,\"ms\":%.4f,\"cycles_per_warp_step_per_sm\":%.2f,\"px_per_clk_per_sm\":%.2f}\n",
                name, (int)SHFL, best, cyc_per_step, 512.0 / cyc_per_step);
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* d;
    CK(cudaMalloc(&d, 4));
    long long* dcyc;
    CK(cudaMalloc(&dcyc, sizeof(long long) * sms));
    const size_t rows_per_warp = 512;  // 256 KiB per warp, 600 MB in all: streams from HBM / L2
    uint4* src;
    const size_t bytes = (size_t)sms * kWarps * (rows_per_warp + 4) * 512;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMemset(src, 0x5a, bytes));
    run<0, false>("atomics_only", d, src, rows_per_warp, sms, dcyc);
    run<1, false>("cp_async_16B", d, src, rows_per_warp, sms, dcyc);
    run<2, false>("bulk_512B", d, src, rows_per_warp, sms, dcyc);
    run<3, false>("ldg_128", d, src, rows_per_warp, sms, dcyc);
    run<1, true>("cp_async_16B", d, src, rows_per_warp, sms, dcyc);
    run<2, true>("bulk_512B", d, src, rows_per_warp, sms, dcyc);
    run<3, true>("ldg_128", d, src, rows_per_warp, sms, dcyc);
    run<4, true>("k5_cp_async_8x64B_plus_pads", d, src, rows_per_warp, sms, dcyc);
    run<5, true>("k5_bulk_8x80B", d, src, rows_per_warp, sms, dcyc);
    return 0;
}

// Shared-atomic probe for the K1 counter layout: is a
// lane-striped update (lane L only touches bank L) really one wavefront per
// warp instruction when the 32 lanes hit 32 DIFFERENT 128-byte rows, and what
// do back-to-back updates of the same word by the same lane cost?
// ncu reports ~14-16 % "bank conflicts" on K1's atomics although every lane
// owns its bank; this isolates the address patterns K1 produces.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atom_probe tools/atom_probe.cu
// Run:   tools/atom_probe            (one JSON line per pattern)
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
__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) { asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v)); }

// Rows of 128 B (32 lane words); 1024 rows = 128 KiB, like K1's counter block.
// PATTERN
//  0 same row for all lanes, row changes per instruction      (microbench "conflict free")
//  1 lane-striped, every lane its own random row               (K1 on i.i.d. data)
//  2 as 1, but each instruction repeats the previous address   (same word back to back)
//  3 as 1, every 2nd instruction repeats the previous address
//  4 lane-striped, rows = base + small per-lane offset (0..15) (K1 on smooth data)
//  5 as 1, ADD of a register value instead of +1
//  6 as 1, rows drawn from 256 (one table half), +1
//  7 as 1, 16 instructions alternate between two tables 64 KiB apart
// Pattern 8: warps 0-7 run the random-row lane-striped atomics of pattern 1
// while warps 8-15 stream 16-byte cp.async copies from global memory into a
// separate shared buffer (like K1/K5's row ring): does ncu's
// l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom count the
// arriving copy data as atomic "conflicts"?
__global__ void __launch_bounds__(512, 1) probe_mixed(uint32_t* out, const uint4* src, int iters)
{
    extern __shared__ __align__(16) uint32_t hist[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(hist);
    if (warp < 8) {
        uint32_t seed = mix(blockIdx.x * 4096 + threadIdx.x * 7 + 1);
        uint32_t a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            a[j] = base + (mix(seed + j * 0x9e3779b9u) & 511u) * 128u + lane * 4u;  // rows 0..511
        for (int it = 0; it < iters; ++it) {
            const uint32_t x = (uint32_t)(it & 7) << 7;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                red_inc(a[j] ^ x);
        }
    } else {
        // copy ring: 4 slots x 512 B per warp above row 512 (bytes 64 KiB+)
        const uint32_t ring = base + 65536u + (warp - 8) * 2048u + lane * 16u;
        const uint4* g = src + (size_t)blockIdx.x * 65536 + (warp - 8) * 32 + lane;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring + j * 512u),
                             "l"(g + ((it * 4 + j) & 255) * 256)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 2;" ::: "memory");
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) s += hist[i];
    atomicAdd(out, s);
}

template <int PATTERN>
__global__ void __launch_bounds__(512, 1) probe(uint32_t* out, int iters)
{
    extern __shared__ __align__(16) uint32_t hist[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(hist);
    uint32_t seed = mix(blockIdx.x * 4096 + threadIdx.x * 7 + 1);
    uint32_t a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t r = mix(seed + j * 0x9e3779b9u);
        uint32_t row;
        if (PATTERN == 0) row = (uint32_t)j * 37u & 1023u;
        else if (PATTERN == 4) row = (mix(threadIdx.x >> 5) & 1007u) + (r & 15u);
        else if (PATTERN == 6) row = r & 255u;
        else if (PATTERN == 7) row = (r & 511u) + ((j & 1) ? 512u : 0u);
        else row = r & 1023u;
        if (PATTERN == 2 && j > 0) row = (a[j - 1] - base) >> 7;
        if (PATTERN == 3 && (j & 1)) row = (a[j - 1] - base) >> 7;
        a[j] = base + row * 128u + lane * 4u;
    }
    uint32_t v = lane | 1u;
    for (int it = 0; it < iters; ++it) {
        // rotate the rows a little per iteration (keeps the lane stripe)
        const uint32_t x = (uint32_t)(it & 7) << 7;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (PATTERN == 5)
                red_add(a[j] ^ x, v);
            else
                red_inc(a[j] ^ x);
        }
        v += 2;
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) s += hist[i];
    atomicAdd(out, s);
}

template <int P>
void run(const char* name, uint32_t* d, int sms)
{
    const int iters = 4096;
    const size_t smem = 128 * 1024;
    CK(cudaFuncSetAttribute(probe<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe<P><<<sms, 512, smem>>>(d, 16);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        probe<P><<<sms, 512, smem>>>(d, iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const double instr = (double)sms * 16 * iters * 16;  // warp instructions
    const double per_sm_clk = instr / sms / (best * 1e-3 * clk_khz * 1e3);
    std::printf("{\"pattern\":\"%s\",\"ms\":%.4f,\"warp_atoms_per_sm_clk_at_max\":%.3f}\n", name, best, per_sm_clk);
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* d;
    CK(cudaMalloc(&d, 4));
    run<0>("same_row_lane_stripe", d, sms);
    run<1>("random_rows_lane_stripe", d, sms);
    run<2>("random_rows_repeat_every", d, sms);
    run<3>("random_rows_repeat_every_2nd", d, sms);
    run<4>("clustered_rows_lane_stripe", d, sms);
    run<5>("random_rows_add_reg", d, sms);
    run<6>("random_rows_256", d, sms);
    run<7>("random_rows_two_tables", d, sms);
    {
        uint4* src;
        CK(cudaMalloc(&src, (size_t)sms * 65536 * 16));
        CK(cudaMemset(src, 1, (size_t)sms * 65536 * 16));
        CK(cudaFuncSetAttribute(probe_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
        probe_mixed<<<sms, 512, 128 * 1024>>>(d, src, 4096);
        CK(cudaDeviceSynchronize());
        std::printf("{\"pattern\":\"mixed_atomics_and_cp_async\",\"ran\":1}\n");
    }
    return 0;
}

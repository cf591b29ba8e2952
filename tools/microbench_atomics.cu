// Shared-memory atomic and streaming-read microbenchmarks for B200 (sm_100a).
// Decides the histogram layout of the accumulation kernel:
// how many ATOMS.POPC.INC per cycle an SM retires for the key patterns the
// configs produce (spread, clustered, single hot key, wide joint keys).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_atomics tools/microbench_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// pattern: 0 = lane (conflict-free), 1 = warp-uniform, 2 = random in [0,mask],
// 3 = lane*32 (32-way bank conflict), 4 = random clustered: base(warp,iter) + (r & 63)
template <int PATTERN>
__global__ void __launch_bounds__(1024) atoms_kernel(uint32_t* out, int iters, uint32_t mask, int bins)
{
    extern __shared__ uint32_t hist[];
    for (int i = threadIdx.x; i < bins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t seed = mix(blockIdx.x * 1024 + threadIdx.x);
    uint32_t k[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        uint32_t r = mix(seed + j * 0x9e3779b9U);
        if (PATTERN == 0) k[j] = (lane + 32 * j) & mask;
        else if (PATTERN == 1) k[j] = (j * 97) & mask;
        else if (PATTERN == 2) k[j] = r & mask;
        else if (PATTERN == 3) k[j] = (lane * 32 + j) & mask;
        else k[j] = ((j * 611) + (r & 63)) & mask;
    }
    for (int it = 0; it < iters; ++it) {
        const uint32_t x = (PATTERN == 2) ? (mix(it) & mask) : ((it * 64) & mask & ~63u);
#pragma unroll
        for (int j = 0; j < 16; ++j) atomicAdd(&hist[k[j] ^ x], 1u);
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < bins; i += blockDim.x) s += hist[i];
    atomicAdd(out, s);
}

// 1 byte/px streaming read: 16 B vector loads, XOR-reduce so nothing is dead.
__global__ void __launch_bounds__(512) stream_read(const uint4* __restrict__ p, size_t n16, uint32_t* out)
{
    uint32_t acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < n16; i += stride) { uint4 a = __ldg(p + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
    if (acc == 0x12345678u) atomicAdd(out, 1u);
}

template <int P>
void run_atoms(const char* name, uint32_t mask, int bins, int threads, int ctas_per_sm, int sms, uint32_t* dout)
{
    const int iters = 2000;
    size_t smem = (size_t)bins * 4;
    CK(cudaFuncSetAttribute(atoms_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    atoms_kernel<P><<<grid, threads, smem>>>(dout, 10, mask, bins);
    CK(cudaEventRecord(a));
    atoms_kernel<P><<<grid, threads, smem>>>(dout, iters, mask, bins);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    double ops = (double)grid * threads * iters * 16;
    int clk_khz; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    double sm_cycles = ms * 1e-3 * clk_khz * 1e3;  // at the nominal max clock
    std::printf("{\"bench\":\"atoms\",\"pattern\":\"%s\",\"bins\":%d,\"threads\":%d,\"ctas_per_sm\":%d,"
                "\"ms\":%.3f,\"gatoms_per_s\":%.1f,\"atoms_per_sm_cycle_at_max_clk\":%.2f}\n",
                name, bins, threads, ctas_per_sm, ms, ops / ms * 1e-6, ops / sms / sm_cycles);
}

int main()
{
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* dout; CK(cudaMalloc(&dout, 4));
    std::printf("{\"sms\":%d}\n", sms);
    for (int occ : {1, 2}) {
        run_atoms<0>("lane_conflict_free", 1023, 1024, 1024, occ, sms, dout);
        run_atoms<1>("warp_uniform_same_addr", 1023, 1024, 1024, occ, sms, dout);
        run_atoms<2>("random_1024", 1023, 1024, 1024, occ, sms, dout);
        run_atoms<4>("clustered_64", 1023, 1024, 1024, occ, sms, dout);
        run_atoms<3>("bank_conflict_32way", 1023, 1024, 1024, occ, sms, dout);
    }
    run_atoms<2>("random_32768", 32767, 32896, 1024, 1, sms, dout);
    run_atoms<4>("clustered_64_of_32768", 32767, 32896, 1024, 1, sms, dout);
    run_atoms<0>("lane_conflict_free_512t", 1023, 1024, 512, 4, sms, dout);
    run_atoms<2>("random_1024_512t", 1023, 1024, 512, 4, sms, dout);

    // streaming read bandwidth over 1 GiB (>> L2)
    size_t bytes = (size_t)1 << 30;
    uint8_t* buf; CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    for (int g : {sms * 2, sms * 4, sms * 8}) {
        stream_read<<<g, 512>>>((const uint4*)buf, bytes / 16, dout);
        CK(cudaEventRecord(a));
        for (int r = 0; r < 5; ++r) stream_read<<<g, 512>>>((const uint4*)buf, bytes / 16, dout);
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("{\"bench\":\"stream_read\",\"grid\":%d,\"GBps\":%.1f}\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
    }
    CK(cudaGetLastError());
    return 0;
}

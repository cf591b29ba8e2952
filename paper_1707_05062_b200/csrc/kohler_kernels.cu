// kohler_kernels.cu — sm_100a kernels of the Köhler contrast-curve path and
// the C ABI (include/kohler_cuda.h) that launches them.  DESIGN.md §3 has
// the full description; in short:
//
//   K1  walk_kernel    : persistent, one 512-thread CTA per SM (or 1/d of the
//                        SMs in pipelined mode); every lane walks down a
//                        16-pixel column segment, rows streamed through a
//                        cp.async ring, three shared atomics per pixel into a
//                        lane-striped 128 KiB counter block (kohler_walk.cuh);
//                        the CTA flush turns the counters into 512 exact
//                        integer combinations, REDG.ADD.64 into the image's
//                        accumulators.
//   K3/K4 finish      : PDL-chained finish_kernel after K1, one CTA per image:
//                        sums and resets the accumulators, int64 prefix scans
//                        (count, sum), IEEE f64 mean curve, optimal threshold,
//                        top-k.  Single images with small grids finish inside
//                        K1 instead: one thread-block cluster reduced over DSMEM
//                        (<= 8 CTAs) or the last-flushing CTA (ticket, <= 24).
//   K5  twalk_kernel   : batches of small images (lane groups own images;
//                        curves rebuilt in the CTA), + select256_kernel (K4).
//   select_kernel / select256_kernel : selection on given curves.
//   direct_kernel      : definition-level curve (direct.cpp restated).
//   hist_kernel / map_kernel : segmentation (classify / quantize).
//   luma_kernel        : Rec. 601 colour ingest.
// kohler_multi.cuh (included at the end) holds the multi-GPU device groups:
// row bands of one image over several GPUs whose K1 flushes add into ONE
// accumulator on the first GPU over peer memory (no collective), or partial
// curves merged by one NCCL all-reduce; batches sharded by image.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kohler_cuda.h"
#include "kohler_device.cuh"
#include "kohler_walk.cuh"

using namespace kohler_dev;

namespace {

#ifndef KOHLER_MAX_WALK_ROWS
#define KOHLER_MAX_WALK_ROWS 144
#endif
constexpr int kMaxWalkRows = KOHLER_MAX_WALK_ROWS;  // longest K1 column walk (rows)
constexpr int kAccCopiesSingle = 8;  // spread the per-image REDG contention
constexpr int kMaxDepth = 4;         // K1 launches in flight (pipelined mode)
constexpr int kMaxSelectLevels = 4096;

struct WideParams {
    const uint8_t* px;
    size_t pitch;
    size_t image_stride;
    int n;          // images
    int w;          // width
    int band_rows;  // own rows per image (band)
    int buf_rows;   // rows present in the buffer (own rows + halo row if any)
    int h_total;    // global height
    int r0;         // global row of buffer row 0
    int nseg;       // S: 16-pixel segments per row
    int R;          // rows per column walk (16 .. kMaxWalkRows)
    long long T;    // walk tasks per image (S * ceil(band_rows / R))
    long long gpi;  // 32-lane groups per image
    long long upi;  // units per image: gpi * R (unit = one row of a group's 32 walks)
    long long total_units;
    int epoch;      // max units between W spills (kohler_walk::kMaxEventsPerWord)
    unsigned long long seg_magic;  // floor(2^64 / nseg) + 1 (nseg > 1)
    long long cta_q, cta_r;        // total_units = cta_q * G + cta_r
    unsigned long long* acc;  // [n][copies][512]
    int copies;
    unsigned* tickets;  // [n]
    int k;
    int select;
    int no_finish;  // accumulate only (a band of a chunked image; a later launch finishes)
    int early_trigger;  // pipelined launches: let the next launch start at once (disjoint SMs)
    int self_finish;    // single-image launch: the CTA that flushes last runs K3 + K4 (no finish_kernel)
    int cluster;        // single small image: the grid is one cluster, reduced over DSMEM (no accumulator)
    int acc_sys;        // acc is another GPU's memory (device groups, peer mode): system-scope REDs
#ifdef KOHLER_CHECKED
    int inject;  // negative control of the checked build: read one row past the buffer end
#endif
    uint32_t* hist_out;  // [n][256] pixel histogram (atomically accumulated), or null
    uint64_t* sums;
    uint64_t* cards;
    double* values;
    uint8_t* defined;
    int* t0s;
    int* topks;
    int* topk_counts;
    int* status;
};

#ifndef KOHLER_WALK_THREADS
#define KOHLER_WALK_THREADS 384
#endif
constexpr int kWalkThreads = KOHLER_WALK_THREADS;  // K1
constexpr int kWalkWarps = kWalkThreads / 32;
constexpr int kTwThreads = 512;                     // K5 (its round layout assumes 16 warps)
constexpr int kTwWarps = kTwThreads / 32;

// Shared-memory map of K1 (dynamic), after the striped counters and corr
// (kohler_walk.cuh).
// Shared-memory map of K1 (dynamic).  The striped counter block (128 KiB,
// kohler_walk.cuh) sits at the fixed shared-window address kHistAbs, so every
// counter address is "register + compile-time immediate" (no base register
// in the hot loop); everything else lives in the gap below it, at offsets
// from the dynamic base.
constexpr uint32_t kHistAbs = kWalkWarps > 16 ? 0x12000 : 0x10000;  // above the ring + scratch
// Row ring of the column walks (cp.async destination): per warp kRingSlots
// slots of 32 lane segments + a 16-byte pad on each side.  Idle during the
// flush, so the reconstruction / selection scratch aliases it.
constexpr int kRingSlots = 4;
// slot: 32 lane segments (512 B, 128-byte aligned: cp.async writes whole
// lines), then the left pad (lane 0) and the right pad (lane 31)
constexpr uint32_t kSlotBytes = 640;
constexpr uint32_t kSmRing = 0;  // + up to 127 B to align the ring to 128 B
constexpr uint32_t kRingBytes = kWalkWarps * kRingSlots * kSlotBytes + 128;
constexpr uint32_t kSmWacc = kSmRing + kRingBytes;   // u64 [2 copies][2 fields][256]
constexpr uint32_t kSmHsTot = kSmWacc + 8192;        // u64[512]
constexpr uint32_t kSmCorrTot = kSmHsTot + 4096;     // int[256]
constexpr uint32_t kSmCorr = kSmCorrTot + 1024;      // int[256] border terms (corr)
// border rows of the CTA's first image (first own row, last own row, halo):
// the CTA's column slice, prefetched as 4-byte words at kernel start
constexpr int kBorderPx = 1024;                        // widest prefetched slice
constexpr uint32_t kBorderRow = kBorderPx + 32;        // 16-byte chunks of a slice + slack
constexpr uint32_t kSmBorder = kSmCorr + 1024;         // u8 [3][kBorderRow]
constexpr uint32_t kSmHb = (kSmBorder + 3 * kBorderRow + 15) & ~15u;  // u32 [2][256] halo W events
// a copy of the launch parameters for the flush: by then the constant cache
// has lost them to the walk's instruction stream (each cold LDC cost ~0.25 us)
constexpr uint32_t kSmParams = kSmHb + 2048;
constexpr uint32_t kSmBslice = kSmParams + 256;  // BorderSlice of the CTA's first image
constexpr uint32_t kSmFlag = kSmBslice + 12;     // int: this CTA finishes the image (self_finish)
constexpr uint32_t kSmMiscEnd = kSmBslice + 16;
constexpr uint32_t kSmVal = kSmRing;                 // i64[512]
constexpr uint32_t kSmCurve = kSmVal + 4096;         // u64 sum[256], card[256]
constexpr uint32_t kSmMean = kSmCurve + 4096;        // f64[256]
constexpr uint32_t kSmDef = kSmMean + 2048;          // u8[256]
constexpr uint32_t kSmScratch = kSmDef + 256;        // block_select256 scratch
constexpr uint32_t kSmFinishEnd = kSmScratch + 256 * (8 + 4 + 8 + 4);
static_assert(kSmFinishEnd <= kRingBytes, "finish scratch aliases the ring");
// the dynamic base is below 16 KiB in practice (1 KiB driver reserve + static);
// the kernel checks kSmMiscEnd fits under kHistAbs
constexpr uint32_t kSmWideBytes = kHistAbs + kohler_walk::kHistBytes;
static_assert(kSmWideBytes <= 227 * 1024, "K1 shared memory");
// K1 over interleaved RGB (colour ingest fused into the walk, SURVEY.md §8f
// rank 3): a lane segment is 48 bytes (16 pixels), so the ring slots triple;
// the scratch block moves up by the ring's growth (kRgbShift) and the
// counter block sits at kHistAbsRgb, whose end is the 227 KiB opt-in limit
// for any dynamic base <= 1 KiB (the kernel checks both ends).
constexpr uint32_t kSlotBytesRgb = 1664;  // 32 x 48 B, left pad, right pad, 128-byte multiple
constexpr int kRingSlotsRgb = 3;          // 2 positions in flight (3 x 1.5 KiB per warp)
constexpr uint32_t kRingBytesRgb = kWalkWarps * kRingSlotsRgb * kSlotBytesRgb + 128;
constexpr uint32_t kRgbShift = kRingBytesRgb - kRingBytes;
constexpr uint32_t kHistAbsRgb = 0x18C00;
constexpr uint32_t kSmWideBytesRgb = 227 * 1024;
static_assert(kRgbShift + kSmMiscEnd + 1024 <= kHistAbsRgb, "K1 RGB scratch under the counters");
static_assert(kHistAbsRgb + kohler_walk::kHistBytes <= kSmWideBytesRgb + 1024, "K1 RGB shared memory");

// Per-input-format constants of K1 (gray: 1 byte per pixel; RGB: 3).
template <bool RGB>
struct K1Fmt {
    static constexpr uint32_t bpp = RGB ? 3 : 1;
    static constexpr uint32_t seg = 16 * bpp;              // bytes of a lane segment
    static constexpr uint32_t slot = RGB ? kSlotBytesRgb : kSlotBytes;
    static constexpr int slots = RGB ? kRingSlotsRgb : kRingSlots;
    static constexpr int ahead = slots - 1;
    static constexpr uint32_t lpad = 32 * seg;             // left pad (lane 0) in a slot
    static constexpr uint32_t rpad = 32 * seg + 16;        // right pad (lane 31)
    static constexpr uint32_t shift = RGB ? kRgbShift : 0; // scratch offset from the gray map
    static constexpr uint32_t hist_abs = RGB ? kHistAbsRgb : kHistAbs;
    static constexpr uint32_t smem = RGB ? kSmWideBytesRgb : kSmWideBytes;
};

// CTA owning unit u under the balanced partition (first cta_r CTAs hold
// cta_q + 1 units, the rest cta_q).
__device__ __forceinline__ long long cta_of_unit(long long u, long long q, long long r)
{
    const long long big = r * (q + 1);
    return u < big ? u / (q + 1) : r + (u - big) / q;
}

// Programmatic dependent launch (sm_90+): a step's prologue and main loop may
// run while the previous step's tail finishes; everything that touches the
// shared workspace or the outputs waits for the previous grid first.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

#ifdef KOHLER_PHASES
// Debug builds only (tools/phase_probe.cu): per-CTA globaltimer stamps.
__device__ unsigned long long g_phase[2048][12];
__device__ unsigned g_smid[2048];
__device__ int g_rot;
__device__ unsigned long long g_sm_end[2][256];  // per SM: exit stamp of the last two launches
__device__ unsigned g_launch;
__device__ long long g_cyc[2048][8];
#define KCYC(i) do { if (threadIdx.x == 0 && blockIdx.x < 2048) g_cyc[blockIdx.x][i] = clock64(); } while (0)
__device__ unsigned long long g_wend[2048][32];  // per-warp end of its last walk
__device__ __forceinline__ void phase(int i)
{
    if (threadIdx.x == 0 && blockIdx.x < 2048) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_phase[blockIdx.x][i] = t;
        if (i == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_smid[blockIdx.x] = sm;
        }
        if (i == 7) {  // exit stamp per SM, alternating by launch parity
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_sm_end[g_launch & 1][sm & 255] = t;
        }
    }
}
__device__ __forceinline__ void warp_end()
{
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 2048) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_wend[blockIdx.x][threadIdx.x >> 5] = t;
    }
}
#else
#define KCYC(i) do { } while (0)
__device__ __forceinline__ void phase(int) {}
__device__ __forceinline__ void warp_end() {}
#endif

} // namespace

#include "kohler_luma.cuh"  // luma4 / luma_div, also used by K1 over RGB
#include "kohler_k1.cuh"
#include "kohler_k5.cuh"
#include "kohler_select.cuh"
#include "kohler_segment.cuh"

namespace {

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------

thread_local std::string g_last_error;

int fail(int code, const std::string& msg)
{
    g_last_error = msg;
    return code;
}

#define KC_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(e_ == cudaErrorMemoryAllocation ? KOHLER_OUT_OF_MEMORY           \
                                                        : KOHLER_CUDA_ERROR,             \
                        std::string(#call) + ": " + cudaGetErrorString(e_));             \
    } while (0)

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes)
    {
        if (bytes <= cap)
            return KOHLER_OK;
        if (p)
            cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        KC_CUDA(cudaMallocHost(&p, bytes));
        cap = bytes;
        return KOHLER_OK;
    }
    void release()
    {
        if (p)
            cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

} // namespace

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes, bool zero = false)
    {
        if (bytes <= cap)
            return KOHLER_OK;
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
        KC_CUDA(cudaMalloc(&p, bytes));
        if (zero)
            KC_CUDA(cudaMemset(p, 0, bytes));
        cap = bytes;
        return KOHLER_OK;
    }
    void release()
    {
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

} // namespace

constexpr int kMaxChunks = 8;

struct kohler_cuda_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;   // host-API uploads, overlapped with compute
    cudaEvent_t chunk_ev[kMaxChunks] = {};
    cudaEvent_t done_ev = nullptr;        // compute of the previous call finished
    std::mutex mu;
    DevBuf acc;      // zero-initialised, self-cleaning
    DevBuf tickets;  // zero-initialised, self-cleaning
    DevBuf img;      // staging for host images
    DevBuf out;      // staging for host outputs
    DevBuf curves;   // K5 curve scratch when the caller wants no curves
    DevBuf stage;    // 16-byte aligned copy of unaligned device inputs for K1
    HostBuf hout;    // pinned staging for small results (one D2H per call)
    DevBuf rgb;      // staging for host RGB images (colour ingest)
    // streaming host API (kohler_cuda_submit / kohler_cuda_collect): two
    // slots of device image + packed results + pinned host results
    DevBuf simg[2];
    DevBuf sout[2];
    HostBuf shout[2];
    cudaEvent_t sup[2] = {};    // slot's upload finished (copy stream)
    cudaEvent_t sdone[2] = {};  // slot's results are in shout (compute stream)
    long long sticket = 0;      // next ticket
    long long spend[2] = {-1, -1};  // ticket in flight per slot
    int sn[2] = {}, sk[2] = {};     // its image count and k
    DevBuf gray;     // luma of device RGB inputs (16-byte pitched)
    DevBuf seg;      // segmentation scratch (histograms, thresholds)
    int last_launches = 0;
    int last_grid = 0;  // grid of the last K1 launch (debug tools)
    int depth = 1;      // K1 launches in flight (kohler_cuda_set_pipeline_depth)
    bool rgb_fused = true;  // K1 reads RGB itself where the layout allows (env KOHLER_RGB_UNFUSED=1: off)
    bool no_cluster = false;  // env KOHLER_NO_CLUSTER=1: small single images take the ticket path (A/B, tests)
    int cluster_ok = -1;      // -1 unknown; 1 if an 8-CTA cluster of K1 fits this device (checked once)
    bool inject = false;      // checked builds, env KOHLER_CHECKED_INJECT=1: deliberate off-by-one (tests)
    bool wide_attr_set = false;
    bool select_attr_set = false;
    bool select256_attr_set = false;
};

#include "kohler_launch.cuh"


extern "C" {

int kohler_cuda_abi_version(void) { return 104; }

const char* kohler_cuda_last_error(void) { return g_last_error.c_str(); }

int kohler_cuda_create(int device, kohler_cuda_ctx** out)
{
    if (!out)
        return fail(KOHLER_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    KC_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0)
        KC_CUDA(cudaGetDevice(&device));
    if (device >= ndev)
        return fail(KOHLER_INVALID_ARGUMENT, "no such CUDA device");
    DeviceGuard g(device);
    int major = 0, minor = 0;
    KC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    KC_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
        return fail(KOHLER_CUDA_ERROR, "this build targets sm_100a (B200) only; device is sm_" +
                                           std::to_string(major) + std::to_string(minor));
    auto* ctx = new kohler_cuda_ctx();
    ctx->device = device;
    {
        const char* e = std::getenv("KOHLER_RGB_UNFUSED");
        ctx->rgb_fused = !(e && e[0] && e[0] != '0');
        const char* c = std::getenv("KOHLER_NO_CLUSTER");
        ctx->no_cluster = c && c[0] && c[0] != '0';
        const char* inj = std::getenv("KOHLER_CHECKED_INJECT");
        ctx->inject = inj && inj[0] && inj[0] != '0';
    }
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < kMaxChunks && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&ctx->chunk_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&ctx->done_ev, cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ctx->sup[i], cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&ctx->sdone[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        delete ctx;
        return fail(KOHLER_CUDA_ERROR, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    *out = ctx;
    return KOHLER_OK;
}

void kohler_cuda_destroy(kohler_cuda_ctx* ctx)
{
    if (!ctx)
        return;
    {
        DeviceGuard g(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->acc.release();
        ctx->tickets.release();
        ctx->img.release();
        ctx->out.release();
        ctx->curves.release();
        ctx->stage.release();
        ctx->hout.release();
        ctx->seg.release();
        ctx->rgb.release();
        ctx->gray.release();
        cudaStreamDestroy(ctx->stream);
        if (ctx->copy_stream)
            cudaStreamDestroy(ctx->copy_stream);
        for (int i = 0; i < kMaxChunks; ++i)
            if (ctx->chunk_ev[i])
                cudaEventDestroy(ctx->chunk_ev[i]);
        for (int i = 0; i < 2; ++i) {
            if (ctx->sup[i])
                cudaEventDestroy(ctx->sup[i]);
            if (ctx->sdone[i])
                cudaEventDestroy(ctx->sdone[i]);
            ctx->simg[i].release();
            ctx->sout[i].release();
            ctx->shout[i].release();
        }
        if (ctx->done_ev)
            cudaEventDestroy(ctx->done_ev);
    }
    delete ctx;
}

int kohler_cuda_device(const kohler_cuda_ctx* ctx) { return ctx ? ctx->device : -1; }

int kohler_cuda_last_launch_count(const kohler_cuda_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

int kohler_cuda_set_pipeline_depth(kohler_cuda_ctx* ctx, int depth)
{
    if (!ctx)
        return fail(KOHLER_INVALID_ARGUMENT, "null context");
    if (depth < 1 || depth > kMaxDepth)
        return fail(KOHLER_INVALID_ARGUMENT, "pipeline depth must be in [1, 4]");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->depth = depth;
    return KOHLER_OK;
}

int kohler_cuda_curve(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                      uint64_t* sum, uint64_t* card)
{
    if (!ctx || !px || !sum || !card)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(1, w, h, pitch);
    if (rc)
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    BatchOut o{sum, card, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    return host_batch(ctx, px, 1, w, h, pitch, pitch * (size_t)h, 1, 0, o);
}

int kohler_cuda_direct_curve(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                             uint64_t* sum, uint64_t* card)
{
    if (!ctx || !px || !sum || !card)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(1, w, h, pitch);
    if (rc)
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t bytes = (size_t)w * h;
    rc = ctx->img.ensure(std::max<size_t>(bytes, 16));
    if (rc)
        return rc;
    rc = ctx->out.ensure(512 * sizeof(unsigned long long));
    if (rc)
        return rc;
    uint8_t* dimg = static_cast<uint8_t*>(ctx->img.p);
    auto* dout = static_cast<unsigned long long*>(ctx->out.p);
    KC_CUDA(cudaMemcpy2DAsync(dimg, (size_t)w, px, pitch, (size_t)w, (size_t)h,
                              cudaMemcpyHostToDevice, st));
    ctx->last_launches = 1;
    direct_kernel<<<256, 256, 0, st>>>(dimg, w, h, (size_t)w, dout);
    KC_CUDA(cudaGetLastError());
    KC_CUDA(cudaMemcpyAsync(sum, dout, 256 * 8, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaMemcpyAsync(card, dout + 256, 256 * 8, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    return KOHLER_OK;
}

int kohler_cuda_analyze(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                        int k, uint64_t* sum, uint64_t* card, double* values, uint8_t* defined,
                        int* t0, int* topk, int* topk_count)
{
    int status = 0;
    const int rc = kohler_cuda_analyze_batch(ctx, px, 1, w, h, pitch, pitch * (size_t)h, k, sum,
                                             card, values, defined, t0, topk, topk_count, &status);
    if (rc)
        return rc;
    return status;
}

int kohler_cuda_analyze_batch(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h,
                              size_t pitch, size_t image_stride, int k, uint64_t* sums,
                              uint64_t* cards, double* values, uint8_t* defined, int* t0s,
                              int* topks, int* topk_counts, int* status)
{
    if (!ctx || (!px && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(n, w, h, pitch);
    if (rc)
        return rc;
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    if (n > 1 && image_stride < pitch * (size_t)h)
        return fail(KOHLER_INVALID_ARGUMENT, "image stride smaller than one image");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    BatchOut o{sums, cards, values, defined, t0s, topks, topk_counts, status};
    return host_batch(ctx, px, n, w, h, pitch, image_stride, k, 1, o);
}

int kohler_cuda_analyze_batch_device(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w,
                                     int h, size_t pitch, size_t image_stride, int k,
                                     uint64_t* sums, uint64_t* cards, double* values,
                                     uint8_t* defined, int* t0s, int* topks, int* topk_counts,
                                     int* status, void* stream)
{
    if (!ctx || (!px && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(n, w, h, pitch);
    if (rc)
        return rc;
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    if (n > 1 && image_stride < pitch * (size_t)h)
        return fail(KOHLER_INVALID_ARGUMENT, "image stride smaller than one image");
    rc = check_out_align(sums, cards, values, defined, t0s, topks, topk_counts, status);
    if (rc)
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    BatchOut o{sums, cards, values, defined, t0s, topks, topk_counts, status};
    const bool select = t0s || topks || topk_counts || status;
    if (use_tile(n, w, h))
        return launch_tile(ctx, px, n, w, h, pitch, image_stride, k, select ? 1 : 0, o,
                           static_cast<cudaStream_t>(stream));
    return launch_wide(ctx, px, n, w, h, h, 0, pitch, image_stride, k, select ? 1 : 0, o,
                       static_cast<cudaStream_t>(stream));
}

int kohler_cuda_submit(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h, size_t pitch,
                       size_t image_stride, int k, long long* ticket)
{
    if (!ctx || !ticket || (!px && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(n, w, h, pitch);
    if (rc)
        return rc;
    if (n < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "submit: at least one image");
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    if (n > 1 && image_stride < pitch * (size_t)h)
        return fail(KOHLER_INVALID_ARGUMENT, "image stride smaller than one image");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const int slot = (int)(ctx->sticket & 1);
    if (ctx->spend[slot] >= 0)
        return fail(KOHLER_INVALID_ARGUMENT, "submit: collect the ticket submitted two calls ago first");
    const size_t dpitch = round_up((size_t)w, 16), dstride = dpitch * (size_t)h;
    const size_t n256 = (size_t)n * 256;
    const size_t tail_off = round_up(n256 * 25, 16);
    const size_t bytes = tail_off + (size_t)n * 4 * 3 + (size_t)n * k * 4;
    if ((rc = ctx->simg[slot].ensure(dstride * (size_t)n)) || (rc = ctx->sout[slot].ensure(bytes + 64)) ||
        (rc = ctx->shout[slot].ensure(bytes)))
        return rc;
    uint8_t* dimg = static_cast<uint8_t*>(ctx->simg[slot].p);
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    ctx->last_launches = 0;
    // the upload overlaps the previous submission's kernels (other slot)
    if (pitch == dpitch && (n == 1 || image_stride == dstride))
        KC_CUDA(cudaMemcpyAsync(dimg, px, dstride * (size_t)n, cudaMemcpyHostToDevice, cs));
    else if (n == 1 || image_stride == pitch * (size_t)h)
        KC_CUDA(cudaMemcpy2DAsync(dimg, dpitch, px, pitch, (size_t)w, (size_t)h * n,
                                  cudaMemcpyHostToDevice, cs));
    else
        for (int i = 0; i < n; ++i)
            KC_CUDA(cudaMemcpy2DAsync(dimg + dstride * i, dpitch, px + image_stride * i, pitch,
                                      (size_t)w, (size_t)h, cudaMemcpyHostToDevice, cs));
    KC_CUDA(cudaEventRecord(ctx->sup[slot], cs));
    KC_CUDA(cudaStreamWaitEvent(st, ctx->sup[slot], 0));
    char* b = static_cast<char*>(ctx->sout[slot].p);
    BatchOut d{};
    d.sums = reinterpret_cast<uint64_t*>(b);
    d.cards = reinterpret_cast<uint64_t*>(b + n256 * 8);
    d.values = reinterpret_cast<double*>(b + n256 * 16);
    d.defined = reinterpret_cast<uint8_t*>(b + n256 * 24);
    d.t0s = reinterpret_cast<int*>(b + tail_off);
    d.topk_counts = d.t0s + n;
    d.status = d.topk_counts + n;
    d.topks = d.status + n;
    rc = use_tile(n, w, h) ? launch_tile(ctx, dimg, n, w, h, dpitch, dstride, k, 1, d, st)
                           : launch_wide(ctx, dimg, n, w, h, h, 0, dpitch, dstride, k, 1, d, st);
    if (rc)
        return rc;
    KC_CUDA(cudaMemcpyAsync(ctx->shout[slot].p, b, bytes, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaEventRecord(ctx->sdone[slot], st));
    ctx->spend[slot] = ctx->sticket;
    ctx->sn[slot] = n;
    ctx->sk[slot] = k;
    *ticket = ctx->sticket++;
    return KOHLER_OK;
}

int kohler_cuda_collect(kohler_cuda_ctx* ctx, long long ticket, uint64_t* sums, uint64_t* cards,
                        double* values, uint8_t* defined, int* t0s, int* topks, int* topk_counts,
                        int* status)
{
    if (!ctx || ticket < 0)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument / bad ticket");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const int slot = (int)(ticket & 1);
    if (ctx->spend[slot] != ticket)
        return fail(KOHLER_INVALID_ARGUMENT, "collect: no such ticket in flight");
    KC_CUDA(cudaEventSynchronize(ctx->sdone[slot]));
    const int n = ctx->sn[slot], k = ctx->sk[slot];
    const size_t n256 = (size_t)n * 256;
    const size_t tail_off = round_up(n256 * 25, 16);
    const char* hb = static_cast<const char*>(ctx->shout[slot].p);
    if (sums)
        std::memcpy(sums, hb, n256 * 8);
    if (cards)
        std::memcpy(cards, hb + n256 * 8, n256 * 8);
    if (values)
        std::memcpy(values, hb + n256 * 16, n256 * 8);
    if (defined)
        std::memcpy(defined, hb + n256 * 24, n256);
    const int* ht = reinterpret_cast<const int*>(hb + tail_off);
    if (t0s)
        std::memcpy(t0s, ht, (size_t)n * 4);
    if (topk_counts)
        std::memcpy(topk_counts, ht + n, (size_t)n * 4);
    if (status)
        std::memcpy(status, ht + 2 * n, (size_t)n * 4);
    if (topks)
        std::memcpy(topks, ht + 3 * n, (size_t)n * k * 4);
    ctx->spend[slot] = -1;
    return KOHLER_OK;
}

int kohler_cuda_rgb_to_gray_device(kohler_cuda_ctx* ctx, const uint8_t* rgb, int n, int w, int h,
                                   size_t rgb_pitch, size_t rgb_stride, uint8_t* gray,
                                   size_t gray_pitch, size_t gray_stride, void* stream)
{
    if (!ctx || ((!rgb || !gray) && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_rgb(n, w, h, rgb_pitch, rgb_stride);
    if (rc)
        return rc;
    if (gray_pitch < (size_t)w || (n > 1 && gray_stride < gray_pitch * (size_t)h))
        return fail(KOHLER_INVALID_ARGUMENT, "grey pitch / stride too small");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    return launch_luma(ctx, rgb, n, w, h, rgb_pitch, rgb_stride, gray, gray_pitch, gray_stride,
                       static_cast<cudaStream_t>(stream));
}

int kohler_cuda_rgb_to_gray(kohler_cuda_ctx* ctx, const uint8_t* rgb, int w, int h,
                            size_t rgb_pitch, uint8_t* gray, size_t gray_pitch)
{
    if (!ctx || !rgb || !gray)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_rgb(1, w, h, rgb_pitch, 0);
    if (rc)
        return rc;
    if (gray_pitch < (size_t)w)
        return fail(KOHLER_INVALID_ARGUMENT, "grey pitch must be >= width");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    const size_t up = round_up(3 * (size_t)w, 16), dp = round_up((size_t)w, 16);
    rc = ctx->rgb.ensure(up * (size_t)h);
    if (rc)
        return rc;
    rc = ctx->gray.ensure(dp * (size_t)h);
    if (rc)
        return rc;
    uint8_t* drgb = static_cast<uint8_t*>(ctx->rgb.p);
    uint8_t* dg = static_cast<uint8_t*>(ctx->gray.p);
    cudaStream_t st = ctx->stream;
    KC_CUDA(cudaMemcpy2DAsync(drgb, up, rgb, rgb_pitch, 3 * (size_t)w, (size_t)h,
                              cudaMemcpyHostToDevice, st));
    rc = launch_luma(ctx, drgb, 1, w, h, up, up * (size_t)h, dg, dp, dp * (size_t)h, st);
    if (rc)
        return rc;
    KC_CUDA(cudaMemcpy2DAsync(gray, gray_pitch, dg, dp, (size_t)w, (size_t)h, cudaMemcpyDeviceToHost,
                              st));
    KC_CUDA(cudaStreamSynchronize(st));
    return KOHLER_OK;
}

int kohler_cuda_analyze_rgb_batch(kohler_cuda_ctx* ctx, const uint8_t* rgb, int n, int w, int h,
                                  size_t rgb_pitch, size_t rgb_stride, int k, uint64_t* sums,
                                  uint64_t* cards, double* values, uint8_t* defined, int* t0s,
                                  int* topks, int* topk_counts, int* status)
{
    if (!ctx || (!rgb && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_rgb(n, w, h, rgb_pitch, rgb_stride);
    if (rc)
        return rc;
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    BatchOut o{sums, cards, values, defined, t0s, topks, topk_counts, status};
    return host_batch(ctx, rgb, n, w, h, rgb_pitch, n > 1 ? rgb_stride : rgb_pitch * (size_t)h, k, 1,
                      o, 3);
}

int kohler_cuda_analyze_rgb_batch_device(kohler_cuda_ctx* ctx, const uint8_t* rgb, int n, int w,
                                         int h, size_t rgb_pitch, size_t rgb_stride, int k,
                                         uint64_t* sums, uint64_t* cards, double* values,
                                         uint8_t* defined, int* t0s, int* topks, int* topk_counts,
                                         int* status, void* stream)
{
    if (!ctx || (!rgb && n > 0))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_rgb(n, w, h, rgb_pitch, rgb_stride);
    if (rc)
        return rc;
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    rc = check_out_align(sums, cards, values, defined, t0s, topks, topk_counts, status);
    if (rc)
        return rc;
    if (n == 0)
        return KOHLER_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    BatchOut o{sums, cards, values, defined, t0s, topks, topk_counts, status};
    const bool select = t0s || topks || topk_counts || status;
    if (rgb_fused_ok(ctx, rgb, n, w, h, rgb_pitch, rgb_stride))  // one pass: K1 computes the luma
        return launch_wide(ctx, rgb, n, w, h, h, 0, rgb_pitch, rgb_stride, k, select ? 1 : 0, o, st,
                           0, nullptr, true);
    const size_t dp = round_up((size_t)w, 16), ds = dp * (size_t)h;
    rc = ctx->gray.ensure(ds * (size_t)n);
    if (rc)
        return rc;
    uint8_t* dg = static_cast<uint8_t*>(ctx->gray.p);
    rc = launch_luma(ctx, rgb, n, w, h, rgb_pitch, rgb_stride, dg, dp, ds, st);
    if (rc)
        return rc;
    if (use_tile(n, w, h))
        return launch_tile(ctx, dg, n, w, h, dp, ds, k, select ? 1 : 0, o, st);
    return launch_wide(ctx, dg, n, w, h, h, 0, dp, ds, k, select ? 1 : 0, o, st);
}

int kohler_cuda_classify(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                         const int* thresholds, int nts, uint8_t* labels)
{
    if (!ctx || !px || !labels || (nts > 0 && !thresholds))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(1, w, h, pitch);
    if (rc)
        return rc;
    if (nts < 0 || nts > 255)
        return fail(KOHLER_INVALID_ARGUMENT, "classify: 0..255 thresholds");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return host_classify_quantize(ctx, px, w, h, pitch, thresholds, nts, labels, 0);
}

int kohler_cuda_quantize(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                         const int* thresholds, int nts, uint8_t* out)
{
    if (!ctx || !px || !out || (nts > 0 && !thresholds))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(1, w, h, pitch);
    if (rc)
        return rc;
    if (nts < 0 || nts > 255)
        return fail(KOHLER_INVALID_ARGUMENT, "quantize: 0..255 thresholds");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return host_classify_quantize(ctx, px, w, h, pitch, thresholds, nts, out, 1);
}

int kohler_cuda_segment_batch_device(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w,
                                     int h, size_t pitch, size_t image_stride, int k,
                                     uint8_t* out, size_t out_pitch, size_t out_stride,
                                     int* thresholds, int* ts_counts, int* status, void* stream)
{
    if (!ctx || (n > 0 && (!px || !out || !thresholds || !status)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(n, w, h, pitch);
    if (rc)
        return rc;
    if (k < 0)
        return fail(KOHLER_INVALID_ARGUMENT, "segment: k must be >= 0");
    if (out_pitch < (size_t)w || (n > 1 && (image_stride < pitch * (size_t)h ||
                                            out_stride < out_pitch * (size_t)h)))
        return fail(KOHLER_INVALID_ARGUMENT, "segment: bad pitch or stride");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    return segment_device(ctx, px, n, w, h, pitch, image_stride, k, out, out_pitch, out_stride,
                          thresholds, ts_counts, status, static_cast<cudaStream_t>(stream));
}

int kohler_cuda_segment_batch(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h,
                              int k, uint8_t* out, int* thresholds, int* ts_counts, int* status)
{
    if (!ctx || (n > 0 && (!px || !out || !thresholds || !status)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(n, w, h, (size_t)w);
    if (rc)
        return rc;
    if (k < 0)
        return fail(KOHLER_INVALID_ARGUMENT, "segment: k must be >= 0");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    if (n == 0)
        return KOHLER_OK;
    const size_t dpitch = round_up((size_t)w, 16);
    const size_t dstride = dpitch * (size_t)h;
    const int kk = std::max(k, 1);
    const size_t small = (size_t)n * (kk + 2) * 4;
    rc = ctx->img.ensure(2 * dstride * (size_t)n + small + 64);
    if (rc)
        return rc;
    uint8_t* din = static_cast<uint8_t*>(ctx->img.p);
    uint8_t* dout = din + dstride * (size_t)n;
    int* dts = reinterpret_cast<int*>(round_up(reinterpret_cast<uintptr_t>(dout + dstride * (size_t)n), 16));
    int* dcnt = dts + (size_t)n * kk;
    int* dst = dcnt + n;
    cudaStream_t st = ctx->stream;
    KC_CUDA(cudaMemcpy2DAsync(din, dpitch, px, (size_t)w, (size_t)w, (size_t)h * n,
                              cudaMemcpyHostToDevice, st));
    rc = segment_device(ctx, din, n, w, h, dpitch, dstride, k, dout, dpitch, dstride, dts, dcnt,
                        dst, st);
    if (rc)
        return rc;
    KC_CUDA(cudaMemcpy2DAsync(out, (size_t)w, dout, dpitch, (size_t)w, (size_t)h * n,
                              cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaMemcpyAsync(thresholds, dts, (size_t)n * kk * 4, cudaMemcpyDeviceToHost, st));
    if (ts_counts)
        KC_CUDA(cudaMemcpyAsync(ts_counts, dcnt, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaMemcpyAsync(status, dst, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    return KOHLER_OK;
}

int kohler_cuda_band_curve_device(kohler_cuda_ctx* ctx, const uint8_t* band, int w, size_t pitch,
                                  int h_total, int r0, int r1, uint64_t* sum, uint64_t* card,
                                  void* stream)
{
    if (!ctx || !band || !sum || !card)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int rc = check_image(1, w, h_total, pitch);
    if (rc)
        return rc;
    if (r0 < 0 || r1 <= r0 || r1 > h_total)
        return fail(KOHLER_INVALID_ARGUMENT, "band rows must satisfy 0 <= r0 < r1 <= h");
    if (reinterpret_cast<uintptr_t>(sum) % 8 || reinterpret_cast<uintptr_t>(card) % 8)
        return fail(KOHLER_INVALID_ARGUMENT, "device sum / card must be 8-byte aligned");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    BatchOut o{sum, card, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    return launch_wide(ctx, band, 1, w, r1 - r0, h_total, r0, pitch, 0, 1, 0, o,
                       static_cast<cudaStream_t>(stream));
}

int kohler_cuda_select_device(kohler_cuda_ctx* ctx, const uint64_t* sums, const uint64_t* cards,
                              int n_curves, int levels, int k, double* values, uint8_t* defined,
                              int* t0s, int* topks, int* topk_counts, int* status, void* stream)
{
    if (!ctx || (n_curves > 0 && (!sums || !cards)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    if (levels < 1 || levels > kMaxSelectLevels)
        return fail(KOHLER_INVALID_ARGUMENT, "levels must be in [1, 4096]");
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    if (int rc = check_out_align(sums, cards, values, defined, t0s, topks, topk_counts, status))
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    SelectParams sp{sums,  cards,   nullptr, nullptr, n_curves,    levels, k,
                    1,     values,  defined, t0s,     topks,       topk_counts, status};
    return launch_select(ctx, sp, static_cast<cudaStream_t>(stream));
}

// Host-curve selection helpers (drop-in mean_contrast / optimal_threshold /
// top_k_local_maxima): stage, run select_kernel, copy back.
static int host_select(kohler_cuda_ctx* ctx, const uint64_t* sum, const uint64_t* card,
                       const double* values_in, const uint8_t* defined_in, int n, int k,
                       double* values, uint8_t* defined, int* t0, int* topk, int* count,
                       int* status_out)
{
    if (n < 0 || n > kMaxSelectLevels)
        return fail(KOHLER_INVALID_ARGUMENT, "levels must be in [0, 4096]");
    if (n == 0) {
        if (t0)
            *t0 = -1;
        if (count)
            *count = 0;
        if (status_out)
            *status_out = KOHLER_NO_BOUNDARY;
        return KOHLER_OK;
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t need = (size_t)n * (8 + 8 + 1 + 1 + 8) + (size_t)k * 4 + 64;
    int rc = ctx->out.ensure(need);
    if (rc)
        return rc;
    char* b = static_cast<char*>(ctx->out.p);
    uint64_t* dsum = reinterpret_cast<uint64_t*>(b);
    uint64_t* dcard = dsum + n;
    double* dval = reinterpret_cast<double*>(dcard + n);
    uint8_t* ddef = reinterpret_cast<uint8_t*>(dval + n);
    int* dint = reinterpret_cast<int*>(round_up(reinterpret_cast<uintptr_t>(ddef + n), 16));
    SelectParams sp{};
    sp.n_curves = 1;
    sp.levels = n;
    sp.k = k;
    if (sum) {
        KC_CUDA(cudaMemcpyAsync(dsum, sum, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        KC_CUDA(cudaMemcpyAsync(dcard, card, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        sp.sums = dsum;
        sp.cards = dcard;
        sp.values = dval;
        sp.defined = ddef;
        sp.want_select = 0;
    } else {
        // values/defined in: reuse dsum/dcard space
        double* vin = reinterpret_cast<double*>(dsum);
        uint8_t* din = reinterpret_cast<uint8_t*>(dcard);
        KC_CUDA(cudaMemcpyAsync(vin, values_in, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        KC_CUDA(cudaMemcpyAsync(din, defined_in, (size_t)n, cudaMemcpyHostToDevice, st));
        sp.in_values = vin;
        sp.in_defined = din;
        sp.want_select = 1;
        sp.t0s = dint;
        sp.topk_counts = dint + 1;
        sp.status = dint + 2;
        sp.topks = dint + 4;
    }
    ctx->last_launches = 0;
    rc = launch_select(ctx, sp, st);
    if (rc)
        return rc;
    int hint[4] = {0, 0, 0, 0};
    if (sum) {
        KC_CUDA(cudaMemcpyAsync(values, dval, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
        KC_CUDA(cudaMemcpyAsync(defined, ddef, (size_t)n, cudaMemcpyDeviceToHost, st));
    } else {
        KC_CUDA(cudaMemcpyAsync(hint, dint, 16, cudaMemcpyDeviceToHost, st));
        if (topk)
            KC_CUDA(cudaMemcpyAsync(topk, dint + 4, (size_t)k * 4, cudaMemcpyDeviceToHost, st));
    }
    KC_CUDA(cudaStreamSynchronize(st));
    if (!sum) {
        if (t0)
            *t0 = hint[0];
        if (count)
            *count = hint[1];
        if (status_out)
            *status_out = hint[2];
    }
    return KOHLER_OK;
}

int kohler_cuda_mean_contrast(kohler_cuda_ctx* ctx, const uint64_t* sum, const uint64_t* card,
                              int n, double* values, uint8_t* defined)
{
    if (!ctx || (n > 0 && (!sum || !card || !values || !defined)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    return host_select(ctx, sum, card, nullptr, nullptr, n, 1, values, defined, nullptr, nullptr,
                       nullptr, nullptr);
}

int kohler_cuda_optimal_threshold(kohler_cuda_ctx* ctx, const double* values,
                                  const uint8_t* defined, int n, int* t0)
{
    if (!ctx || !t0 || (n > 0 && (!values || !defined)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    int st = 0, count = 0;
    const int rc = host_select(ctx, nullptr, nullptr, values, defined, n, 1, nullptr, nullptr, t0,
                               nullptr, &count, &st);
    if (rc)
        return rc;
    return st ? KOHLER_NO_BOUNDARY : KOHLER_OK;
}

int kohler_cuda_top_k_local_maxima(kohler_cuda_ctx* ctx, const double* values,
                                   const uint8_t* defined, int n, int k, int* out, int* count)
{
    if (!ctx || !count || (n > 0 && (!values || !defined)))
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    *count = 0;
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "top_k_local_maxima: k must be at least 1");
    if (!out)
        return fail(KOHLER_INVALID_ARGUMENT, "NULL argument");
    // at most n maxima exist: a larger k means "all of them" (the reference
    // truncates a shorter list); clamping keeps the staging O(n)
    k = std::min(k, std::max(n, 1));
    int st = 0, t0 = -1;
    const int rc =
        host_select(ctx, nullptr, nullptr, values, defined, n, k, nullptr, nullptr, &t0, out, count, &st);
    if (rc)
        return rc;
    return st ? KOHLER_NO_BOUNDARY : KOHLER_OK;
}

} // extern "C"

#include "kohler_multi.cuh"  // multi-GPU C ABI (device groups, NCCL)

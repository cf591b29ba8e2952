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
//   K3/K4 finish_kernel: PDL-chained after K1, one CTA per image: sums and
//                        resets the accumulators, int64 prefix scans (count,
//                        sum), IEEE f64 mean curve, optimal threshold, top-k.
//   K5  twalk_kernel   : batches of small images (lane groups own images;
//                        curves rebuilt in the CTA), + select256_kernel (K4).
//   select_kernel / select256_kernel : selection on given curves.
//   direct_kernel      : definition-level curve (direct.cpp restated).
//   hist_kernel / map_kernel : segmentation (classify / quantize).
//   luma_kernel        : Rec. 601 colour ingest.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
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
    int R;          // rows per column walk (even)
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

// K3 + K4, one CTA (256 threads) per image, launched right after K1 with
// programmatic dependent launch: waits for K1, sums the accumulator copies
// (resetting them: the workspace is self-cleaning), rebuilds count/sum with
// int64 prefix scans, writes the curve and the IEEE f64 mean curve, selects.
struct FinishParams {
    unsigned long long* acc;  // [n][copies][512]
    int copies;
    int k;
    int select;
    uint64_t* sums;
    uint64_t* cards;
    double* values;
    uint8_t* defined;
    int* t0s;
    int* topks;
    int* topk_counts;
    int* status;
};

__global__ void __launch_bounds__(256) finish_kernel(const FinishParams p)
{
    __shared__ long long sval[512];
    __shared__ long long tmp[256];
    __shared__ uint64_t csum[256], ccard[256];
    __shared__ double mean[256];
    __shared__ uint8_t def[256];
    __shared__ __align__(16) unsigned char scr[256 * (8 + 4 + 8 + 4) + 64];
    const int tid = threadIdx.x;
    const int img = blockIdx.x;
    pdl_trigger();  // the next K1 may start its walk; its flush waits for us
    pdl_wait();     // K1's accumulation of this image is complete and visible
    for (int r = tid; r < 512; r += 256) {
        unsigned long long* a = p.acc + (size_t)img * p.copies * 512 + r;
        unsigned long long v[kAccCopiesSingle];
#pragma unroll
        for (int c = 0; c < kAccCopiesSingle; ++c)
            v[c] = c < p.copies ? __ldcg(a + c * 512) : 0ull;
        unsigned long long s = 0;
#pragma unroll
        for (int c = 0; c < kAccCopiesSingle; ++c) {
            s += v[c];
            if (c < p.copies)
                __stcg(a + c * 512, 0ull);
        }
        sval[r] = (long long)s;
    }
#ifdef KOHLER_PHASES
    if (tid == 0 && img == 0)
        ++g_launch;
#endif
    __syncthreads();
    const int warp = tid >> 5;
    if (warp == 0)
        warp_prefix256(sval, reinterpret_cast<long long*>(ccard));
    else if (warp == 1) {
        warp_prefix256(sval + 256, tmp);
        __syncwarp();
        warp_prefix256(tmp, reinterpret_cast<long long*>(csum));
    }
    __syncthreads();
    {
        const uint64_t cs = csum[tid], cc = ccard[tid];
        const double v = cc ? (double)cs / (double)cc : 0.0;
        mean[tid] = v;
        def[tid] = cc ? 1 : 0;
        if (p.sums) {
            p.sums[(size_t)img * 256 + tid] = cs;
            p.cards[(size_t)img * 256 + tid] = cc;
        }
        if (p.values)
            p.values[(size_t)img * 256 + tid] = v;
        if (p.defined)
            p.defined[(size_t)img * 256 + tid] = cc ? 1 : 0;
    }
    __syncthreads();
    if (p.select) {
        const int st = block_select256(mean, def, p.k, scr, 1, p.t0s ? p.t0s + img : nullptr,
                                       p.topks ? p.topks + (size_t)img * p.k : nullptr,
                                       p.topk_counts ? p.topk_counts + img : nullptr);
        if (tid == 0 && p.status)
            p.status[img] = st;
    }
}

// Fold the packed W words (both copies) into the u64 per-CTA accumulators
// and clear them.  Thread t owns (copy t >> 8, key t & 255): 32 lane words
// read rotated by t & 7 so a warp's LDS.128 hit distinct bank quads.
__device__ __forceinline__ void spill_w(unsigned char* sm, unsigned char* hist, int tid,
                                        bool clear = true)
{
    using namespace kohler_walk;
    const int copy = tid >> 8, key = tid & 255;
    uint4* row = reinterpret_cast<uint4*>(hist + (key + 256 * copy) * 256 + 128);
    uint32_t h = 0, b = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint4 v = row[(j + tid) & 7];
        h += (v.x & 0xFFFFu) + (v.y & 0xFFFFu) + (v.z & 0xFFFFu) + (v.w & 0xFFFFu);
        b += (v.x >> 16) + (v.y >> 16) + (v.z >> 16) + (v.w >> 16);
        if (clear)
            row[(j + tid) & 7] = make_uint4(0, 0, 0, 0);
    }
    unsigned long long* wacc = reinterpret_cast<unsigned long long*>(sm + kSmWacc);
    wacc[copy * 512 + key] += h;        // hist field
    wacc[copy * 512 + 256 + key] += b;  // B field
}

// Border terms of an image band, split by columns over the CTAs that cover
// the image (balanced: no CTA re-reads whole border rows), added straight
// into the CTA's u64 totals after the striped counters are reduced:
//   band first row      : corr +1 per pixel (up pair missing or not owned)
//   last image row      : corr -1 per pixel (its down pairs were emitted as
//                         equal fakes: the down row was the row itself)
//   halo row (band end) : per halo pixel d under c, its owned up pair as a W
//                         event B = 4 + sign(c - d), corr +3
// (The halo pixels' W counts thus enter hist(); hist_out is only requested
// for whole images, which have no halo.)
struct BorderSlice {
    int xa, xb;  // columns of this CTA's share
    int ca;      // first 16-byte chunk of the prefetched slice (pre != null)
};

__device__ __forceinline__ BorderSlice border_slice(const WideParams& p, int img)
{
    // the CTAs covering the image: the whole grid for one image (no divisions)
    uint32_t cnt = gridDim.x, idx = blockIdx.x;
    if (p.n > 1) {
        const long long c0 = cta_of_unit((long long)img * p.upi, p.cta_q, p.cta_r);
        const long long c1 = cta_of_unit((long long)(img + 1) * p.upi - 1, p.cta_q, p.cta_r);
        cnt = (uint32_t)(c1 - c0 + 1);
        idx = (uint32_t)((long long)blockIdx.x - c0);
    }
    BorderSlice s;
    if (p.w < (1 << 22)) {  // 32-bit products (cnt <= 1024)
        s.xa = (int)((uint32_t)p.w * idx / cnt);
        s.xb = (int)((uint32_t)p.w * (idx + 1) / cnt);
    } else {
        s.xa = (int)((long long)p.w * idx / cnt);
        s.xb = (int)((long long)p.w * (idx + 1) / cnt);
    }
    s.ca = s.xa >> 4;
    return s;
}

// Issue the cp.async copies of the slice's border rows in 16-byte chunks
// (rows are 16-byte aligned: K1 inputs are staged otherwise; a chunk stays
// inside the pitch).  One commit group.
__device__ __forceinline__ void border_prefetch(const WideParams& p, int img, const BorderSlice& s,
                                                uint32_t dst)
{
    const uint8_t* base = p.px + (size_t)img * p.image_stride;
    const int ylast = p.band_rows - 1;
    const int rows = p.r0 + ylast != p.h_total - 1 ? 3 : 2;  // + the halo row
    const int nc = ((s.xb + 15) >> 4) - s.ca;
    for (int i = threadIdx.x; i < rows * nc; i += kWalkThreads) {
        const int r = i >= nc ? (i >= 2 * nc ? 2 : 1) : 0, ci = i - r * nc;
        const int y = r == 0 ? 0 : ylast + (r - 1);
        const uint8_t* src = base + (size_t)y * p.pitch + 16 * (s.ca + ci);
#ifndef KOHLER_PROBE_NO_BORDER_COPY
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + r * kBorderRow + 16 * ci),
                     "l"(src)
                     : "memory");
#else
        asm volatile("" ::"r"(dst + r * kBorderRow + 16 * ci), "l"(src));
#endif
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void border_pass(const WideParams& p, int img, const BorderSlice& s,
                                            const uint8_t* pre, uint32_t* hb, int* corr_tot)
{
    // 32-bit shared atomics only (a u64 shared atomicAdd is a CAS loop, and
    // border values repeat: it serialised the whole pass)
    const uint8_t* base = p.px + (size_t)img * p.image_stride;
    const int ylast = p.band_rows - 1;
    const bool img_last = p.r0 + ylast == p.h_total - 1;
    const uint8_t* rl = base + (size_t)ylast * p.pitch;
    KCYC(0);
    for (int x = s.xa + (int)threadIdx.x; x < s.xb; x += kWalkThreads) {
        const int o = x - 16 * s.ca;
        const int v0 = pre ? pre[o] : base[x];
        const int c = pre ? pre[kBorderRow + o] : rl[x];
        KCYC(1);
        atomicAdd(&corr_tot[v0], 1);
        if (img_last) {
            atomicAdd(&corr_tot[c], -1);
        } else {
            const int d = pre ? pre[2 * kBorderRow + o] : rl[p.pitch + x];
            atomicAdd(&hb[d], 1u);
            atomicAdd(&hb[256 + d], (uint32_t)(4 + (c > d) - (c < d)));
            atomicAdd(&corr_tot[d], 3);
        }
        KCYC(2);
    }
    KCYC(3);
}

// CTA flush of one image's partial: reduce the striped counters (clearing
// them for the next image), form the 512 combinations, REDG them into the
// image's accumulator (finish_kernel takes it from there).
__device__ void flush_image(const WideParams& p, int img, unsigned char* sm, unsigned char* hist,
                            bool clear, bool two_w, bool prefetched, bool first)
{
    using namespace kohler_walk;
    const int tid = threadIdx.x;
    unsigned long long* hs_tot = reinterpret_cast<unsigned long long*>(sm + kSmHsTot);
    int* corr_tot = reinterpret_cast<int*>(sm + kSmCorrTot);
    unsigned long long* wacc = reinterpret_cast<unsigned long long*>(sm + kSmWacc);
    for (int t = tid; t < 512; t += kWalkThreads) {
        uint4* row = reinterpret_cast<uint4*>(hist + t * 256);  // half 0: Hs[t] / dummy
        unsigned long long s = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 v = row[(j + t) & 7];
            s += (unsigned long long)v.x + v.y + v.z + v.w;
            if (clear)  // the CTA's last image: nothing reads the counters again
                row[(j + t) & 7] = make_uint4(0, 0, 0, 0);
        }
        hs_tot[t] = s;
        if (two_w || t < 256)
            spill_w(sm, hist, t, clear);
        if (t < 256) {
            int* cr = reinterpret_cast<int*>(sm + kSmCorr);
            corr_tot[t] = cr[t];
            cr[t] = 0;
        }
    }
    __syncthreads();
    phase(8);
    uint32_t* hb = reinterpret_cast<uint32_t*>(sm + kSmHb);
    KCYC(4);
    // the first image's slice was computed at kernel start (gridDim / params
    // are cold in the constant cache by now)
    border_pass(p, img, first ? *reinterpret_cast<const BorderSlice*>(sm + kSmBslice) : border_slice(p, img),
                prefetched ? sm + kSmBorder : nullptr, hb, corr_tot);
    KCYC(5);
    __syncthreads();
    KCYC(6);
    phase(9);
    // the accumulators may still be read / reset by the previous finish_kernel
    pdl_wait();
    phase(10);
    for (int t = tid; t < 512; t += kWalkThreads) {
        auto hist = [&](int v) { return (long long)(wacc[v] + wacc[512 + v] + hb[v]); };
        long long val;
        if (t < 256) {
            const long long bs = (long long)(wacc[256 + t] + wacc[512 + 256 + t] + hb[256 + t]);
            val = bs - 4ll * hist(t);  // card first difference
        } else {
            const int u = t - 256;  // sum second difference
            if (u == 0) {
                val = 0;
            } else {
                val = 4ll * hist(u - 1) - (long long)corr_tot[u - 1] -
                      2ll * (long long)hs_tot[2 * u - 2] - (long long)hs_tot[2 * u - 1];
                if (u >= 2)
                    val -= (long long)hs_tot[2 * u - 3];
            }
        }
        if (val != 0) {
            const int copy = blockIdx.x % p.copies;
            atomicAdd(p.acc + ((size_t)img * p.copies + copy) * 512 + t, (unsigned long long)val);
        }
        if (p.hist_out && t < 256) {
            const uint32_t hv = (uint32_t)hist(t);  // the W words' pixel counts
            if (hv)
                atomicAdd(p.hist_out + (size_t)img * 256 + t, hv);
        }
    }
    if (clear) {
        __syncthreads();
        for (int t = tid; t < 1024; t += kWalkThreads) {
            wacc[t] = 0;
            if (t < 512)
                hb[t] = 0;
        }
    }
    phase(3);
}

// ---------------------------------------------------------------------------
// K1 walk_kernel: persistent, one 512-thread CTA per SM.  Work unit: a
// "group" of 32 column walks (lane L: task 32g + L of its image, task
// tau -> segment column tau % S, row chunk tau / S, rows [cR, cR + R)).
// CTAs own balanced contiguous group ranges; within an image range, epochs of
// at most p.epoch groups bound the packed W words (kohler_walk.cuh), and each
// warp walks a balanced contiguous sub-range of the epoch, streaming rows
// through a 4-slot register ring (3 rows in flight) across group boundaries.
// ---------------------------------------------------------------------------
struct LaneGeo {
    const uint8_t* p;  // row y0 - 1, column x0 (dereferenced only for valid rows)
    uint32_t pad;      // lane 0 / 31: also copy the 16 bytes left / right (neighbour exists)
    int pd;            // -16 (lane 0) or +16: global offset of the pad copy
    int pds;           // shared offset of the pad copy from the lane's segment
    int x0;
    int y0;            // first own row (band-relative)
    int nrows;         // own rows of the walk (0: no task)
    int e;             // index of the last real pixel of the segment if < 16
    int jlo, jcl;      // ring position j loads row y0 - 1 + clamp(j, jlo, jcl)
};

__device__ __forceinline__ LaneGeo lane_geo(const WideParams& p, const uint8_t* base, long long g,
                                            int lane)
{
    LaneGeo L;
    const unsigned long long tau = (unsigned long long)g * 32ull + (unsigned)lane;
    const bool act = tau < (unsigned long long)p.T;
    const unsigned long long c = p.nseg == 1 ? tau : __umul64hi(tau, p.seg_magic);
    const int s = (int)(tau - c * (unsigned long long)p.nseg);
    L.x0 = s << 4;
    L.e = p.w - 1 - L.x0;
    if (act) {
        L.y0 = (int)c * p.R;
        L.nrows = min(L.y0 + p.R, p.band_rows) - L.y0;
        L.jlo = L.y0 == 0 ? 1 : 0;
        // loads past the buffer's last row re-read it: the down row of the
        // image's last row is the row itself (equal "fake" down pairs)
        L.jcl = p.buf_rows - L.y0;
    } else {
        L.y0 = 1;  // a valid address (row 0), never used
        L.nrows = 0;
        L.jlo = 0;
        L.jcl = 0;
    }
    L.p = base + ((long long)L.y0 - 1) * (long long)p.pitch + L.x0;
    L.pd = lane == 0 ? -16 : 16;
    L.pds = lane == 0 ? 512 : 528 - 16 * 31;
    L.pad = ((lane == 0) & (L.x0 > 0)) | ((lane == 31) & (L.e > 15)) ? 1u : 0u;
    return L;
}

// Issue the copies of ring position j of a lane's walk into ring slot `dst`
// (shared address of this lane's 16-byte segment in the slot): the segment,
// from a clamped valid row, and for lane 0 / lane 31 the 16 bytes left /
// right of it where that neighbour exists.  One cp.async group per position.
__device__ __forceinline__ void fetch_row(const LaneGeo& L, int j, uint32_t pitch, uint32_t dst)
{
    const uint32_t off = (uint32_t)min(max(j, L.jlo), L.jcl) * pitch;
    const uint8_t* src = L.p + off;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
        "cp.async.cg.shared.global [%0], [%1], 16;\n\t"
        "@p cp.async.cg.shared.global [%3], [%4], 16;\n\t"
        "cp.async.commit_group;\n\t}" ::"r"(dst),
        "l"(src), "r"(L.pad), "r"(dst + L.pds), "l"(src + L.pd)
        : "memory");
}

// Steady-state prefetch of a segment (positions >= 3: no top clamp): the
// lane's source row pointer advances by one pitch per position until the
// walk reaches the buffer's last row (then it re-reads it).  The pad copies
// of lanes 0 / 31 use immediate offsets (left pad: slot + 512 <- src - 16,
// right pad: slot + 528 = lane 31's segment + 32 <- src + 16).
struct FetchStream {
    const uint8_t* src;
    int left;     // positions the pointer may still advance
    uint32_t pl;  // lane 0 with a left neighbour
    uint32_t pr;  // lane 31 with a right neighbour
};

__device__ __forceinline__ FetchStream fetch_stream(const LaneGeo& L, int j, uint32_t pitch,
                                                    int lane)
{
    FetchStream f;
    const int jj = min(j, L.jcl);  // j >= 3 > jlo
    f.src = L.p + (size_t)((uint32_t)jj * pitch);
    f.left = L.jcl - j;
    f.pl = L.pad && lane == 0;
    f.pr = L.pad && lane == 31;
    return f;
}

__device__ __forceinline__ void fetch_next(FetchStream& f, uint32_t pitch, uint32_t dst)
{
    asm volatile(
        "{\n\t.reg .pred pl, pr;\n\tsetp.ne.u32 pl, %2, 0;\n\tsetp.ne.u32 pr, %3, 0;\n\t"
        "cp.async.cg.shared.global [%0], [%1], 16;\n\t"
#ifndef KOHLER_PROBE_NO_PADS
        "@pl cp.async.cg.shared.global [%0+512], [%1+-16], 16;\n\t"
        "@pr cp.async.cg.shared.global [%0+32], [%1+16], 16;\n\t"
#endif
        "cp.async.commit_group;\n\t}" ::"r"(dst),
        "l"(f.src), "r"(f.pl), "r"(f.pr)
        : "memory");
    f.src += f.left > 0 ? pitch : 0u;
    --f.left;
}

// Neighbour bytes by warp shuffles instead of byte loads: 16-byte-strided
// LDS.U8 from 32 lanes is a 4-way bank conflict (5 wavefronts each, ~10 of a
// step's ~65 MIO wavefronts); two SHFL + one single-lane pad load cost 3.
// Per lane and segment: the left neighbour is the pixel itself (row start),
// the pad byte (first lane of a run, not at a row start) or the previous
// lane's last byte; the right one likewise (row end / last lane / next lane).
struct NbrSel {
    uint32_t pad_off;  // shared offset of this lane's pad byte from its segment (if any)
    bool pad;          // lane reads a pad byte
    bool l_own, l_pad;
    bool r_own, r_pad;
};

__device__ __forceinline__ void read_row_shfl(kohler_walk::Row& r, uint32_t seg, const NbrSel& n)
{
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                 : "r"(seg)
                 : "memory");
    uint32_t pb = 0;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
                 "@p ld.shared.u8 %0, [%2];\n\t}"
                 : "+r"(pb)
                 : "r"((uint32_t)n.pad), "r"(seg + n.pad_off)
                 : "memory");
    const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, r.w[3], 1);
    const uint32_t dn = __shfl_down_sync(0xFFFFFFFFu, r.w[0], 1);
    r.ln = n.l_own ? (r.w[0] & 0xFFu) : n.l_pad ? pb : (up >> 24);
    r.rn = n.r_own ? (r.w[3] >> 24) : n.r_pad ? pb : (dn & 0xFFu);
}

// Per-group, warp-uniform flags.
struct GroupFlags {
    bool edge;    // some lane is at a row start or row end (corr terms)
    bool ragged;  // some lane's segment runs past the row end (garbage bytes)
};

__device__ __forceinline__ GroupFlags group_flags(const LaneGeo& L, bool aligned)
{
    GroupFlags f;
    const bool act = L.nrows > 0;
    f.edge = __any_sync(0xFFFFFFFFu, act && (L.x0 == 0 || L.e <= 15));
    f.ragged = !aligned && __any_sync(0xFFFFFFFFu, act && L.e < 15);
    return f;
}

// A warp walks the contiguous run [ua, ub) of "units" of one image: unit u =
// row u % R of the 32 column walks of group u / R.  The run is a sequence of
// segments (one per group touched); a segment of L rows is L + 2 ring
// positions: row r0 - 1 (absorbed), row r0 (prime: q of the up pairs), then
// one position per row.  Rows stream through the warp's 4-slot shared ring,
// prefetched 3 positions ahead across segment boundaries.  The W copy
// alternates with the position parity (bounds each copy's events).
// Clear the counter block (one W copy: rows 256..511 only have their Hs half
// in use) and the per-CTA scratch.
template <bool TWO_W>
__device__ __forceinline__ void zero_counters(unsigned char* sm, unsigned char* hist)
{
    using namespace kohler_walk;
    uint4* z = reinterpret_cast<uint4*>(hist);
    constexpr int kFull = TWO_W ? (int)(kHistBytes / 16) : (int)(kHistBytes / 32);
    for (int i = threadIdx.x; i < kFull; i += kWalkThreads)
        z[i] = make_uint4(0, 0, 0, 0);
    if (!TWO_W) {
        // rows 256..511, bytes [0, 128) of each: 8 uint4 per row
        for (int i = threadIdx.x; i < 256 * 8; i += kWalkThreads)
            z[kFull + (i >> 3) * 16 + (i & 7)] = make_uint4(0, 0, 0, 0);
    }
    uint4* zw = reinterpret_cast<uint4*>(sm + kSmWacc);
    for (int i = threadIdx.x; i < 8192 / 16; i += kWalkThreads)
        zw[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 256)
        reinterpret_cast<int*>(sm + kSmCorr)[threadIdx.x] = 0;
    for (int i = threadIdx.x; i < 512; i += kWalkThreads)
        reinterpret_cast<uint32_t*>(sm + kSmHb)[i] = 0;
}

template <bool ALIGNED, bool TWO_W>
__device__ __forceinline__ void walk_range(const WideParams& p, unsigned char* sm,
                                           unsigned char* hist, uint32_t smbase,
                                           const uint8_t* base, long long ua, long long ub,
                                           bool zero_first)
{
    using namespace kohler_walk;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane4 = (uint32_t)lane * 4u;
    const uint32_t kneg = kHistAbs - lane4;  // pair event at A_a + A_b + kneg
    const uint32_t dummy = kHistAbs + kDummy + lane4;
    // corr[v] of a pixel with W address A: corr_base + (A >> 6) (A >> 6 = 4v + (lane4 >> 6))
    const uint32_t corr_base = smbase + kSmCorr - (lane4 >> 6);
    const int R = p.R;
    const uint32_t pitch = (uint32_t)p.pitch;  // < 2^31 / 64 (checked by the host)
    const bool any = ua < ub;
    // this lane's segment in slot 0 of the warp's ring; slot s is + s * kSlotBytes
    const uint32_t ring = (smbase + kSmRing + 127u) & ~127u;
    const uint32_t seg0 = ring + (uint32_t)warp * (kRingSlots * kSlotBytes) + (uint32_t)lane * 16u;

    // current segment: group g, rows [r0, r1) of its walks; next segment
    long long g = 0;
    int r0 = 0, r1 = 0;
    LaneGeo G{};
    if (any) {
        g = ua / R;
        r0 = (int)(ua - g * R);
        r1 = (int)(ub - g * R < (long long)R ? (int)(ub - g * R) : R);
        G = lane_geo(p, base, g, lane);
        // positions 0, 1, 2 of the first segment (rows r0 - 1, r0, r0 + 1 of the walk)
        fetch_row(G, r0, pitch, seg0);
        fetch_row(G, r0 + 1, pitch, seg0 + kSlotBytes);
        fetch_row(G, r0 + 2, pitch, seg0 + 2 * kSlotBytes);
    }
    if (zero_first) {
        // clear the counters while the first rows are in flight
        phase(4);
        zero_counters<TWO_W>(sm, hist);
        phase(5);
        __syncthreads();
        phase(1);
    }
    if (!any)
        return;

    Car X, Y;
    // ring slots of the current position and of the previous one (which the
    // current step refills: (q + 3) & 3 == (q - 1) & 3)
    const uint32_t slot_end = seg0 + kRingSlots * kSlotBytes;
    uint32_t sl_cur = seg0, sl_prev = seg0 + (kRingSlots - 1) * kSlotBytes;
    for (;;) {
        const int L = r1 - r0;
        const int P = L + 2;
        FetchStream fs = fetch_stream(G, r0 + 3, pitch, lane);
        const long long gn = g + 1;
        const bool has_next = gn * R < ub;
        const int nr1 = has_next ? (int)(ub - gn * R < (long long)R ? (int)(ub - gn * R) : R) : 0;
        const LaneGeo N = has_next ? lane_geo(p, base, gn, lane) : G;
        const GroupFlags F = group_flags(G, ALIGNED);
        const bool row_start = G.x0 == 0, row_end = G.e <= 15;
        // neighbour bytes: the adjacent lane's segment, lanes 0 / 31 their pad,
        // a row start / end the pixel itself
        NbrSel nb;
        nb.l_own = G.x0 == 0;
        nb.l_pad = !nb.l_own && lane == 0;
        nb.r_own = G.e <= 15;
        nb.r_pad = !nb.r_own && lane == 31;
        nb.pad = nb.l_pad || nb.r_pad;
        nb.pad_off = lane == 0 ? 512u + 15u : 528u - 16u * 31u;

        // One ring position j: prefetch position j + 3 (of this segment or,
        // past its end, of the next), absorb row r0 - 1 + j into D and
        // process row r0 - 2 + j (C) against it.
        auto step = [&](Car& D, Car& C, int j, auto kind, auto wc, auto cross) {
            constexpr int KIND = decltype(kind)::value;  // 0 absorb, 1 prime, 2 process
            constexpr bool CROSS = decltype(cross)::value;  // prefetch may cross into the next segment
            constexpr int WC = decltype(wc)::value;
            constexpr uint32_t kOffW = (WC && TWO_W) ? kOffW1 : kOffW0;
            // slot q & 3 was committed 3 groups ago; <= 2 younger groups may pend
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            // all lanes' copies into slot q & 3 are visible, and all lanes have
            // read slot (q - 1) & 3 (the previous position), which is refilled now
            __syncwarp();
            // read this position's row first: the prefetch issue below
            // covers the LDS latency before the unpack needs the data
            Row r;
            read_row_shfl(r, sl_cur, nb);
            const uint32_t pref = sl_prev;
            sl_prev = sl_cur;
            sl_cur = sl_cur + kSlotBytes == slot_end ? seg0 : sl_cur + kSlotBytes;
            if (!CROSS || j + 3 < P)
                fetch_next(fs, pitch, pref);
            else if (has_next)
                fetch_row(N, j + 3 - P, pitch, pref);
            else
                asm volatile("cp.async.commit_group;" ::: "memory");
            absorb<ALIGNED>(D, r, lane4, G.e);
            if (KIND == 1) {
                // prime: q(up -> row r0) from row r0 - 1 (neutral at the band's first row)
                const bool has_up = G.y0 + r0 > 0;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    D.ue[jj] = has_up ? qstep(qfrom(C.e[jj]), D.e[jj]) : kNeutral;
                    D.uo[jj] = has_up ? qstep(qfrom(C.o[jj]), D.o[jj]) : kNeutral;
                }
            }
            if (KIND < 2)
                return;
            const bool live = r0 + j - 2 < G.nrows;
            uint32_t qre[4], qro[4], qde[4], qdo[4], Be[4], Bo[4];
            pair_q(C, D.e, D.o, qre, qro, qde, qdo);
            b_terms(C, qre, qro, qde, qdo, Be, Bo);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                D.ue[jj] = qde[jj];
                D.uo[jj] = qdo[jj];
            }
            const uint32_t Arn = __byte_perm(C.rn, lane4, 0x5504);
            if (ALIGNED || !F.ragged) {
                if (live) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_add_imm<kHistAbs + kOffW>(C.A[i], b_of(Be, Bo, i));
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_inc(C.A[i] + (i < 15 ? C.A[i + 1] : Arn) + kneg);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_inc(C.A[i] + D.A[i] + kneg);
                }
            } else if (live) {
                // ragged row ends: bytes past the row end neutralised
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const bool real = i <= G.e;
                    red_add_imm<kHistAbs + kOffW>(C.A[i], real ? b_of(Be, Bo, i) : 0u);
                    red_inc(real ? C.A[i] + (i < 15 ? C.A[i + 1] : Arn) + kneg : dummy);
                    red_inc(real ? C.A[i] + D.A[i] + kneg : dummy);
                }
            }
            if (F.edge && live) {
                if (row_start)
                    red_add(corr_base + (C.A[0] >> 6), 1u);
                if (row_end)
                    red_add(corr_base + (Arn >> 6), 0xFFFFFFFFu);
            }
        };
        using K0 = std::integral_constant<int, 0>;
        using K1 = std::integral_constant<int, 1>;
        using K2 = std::integral_constant<int, 2>;
        using W0 = std::integral_constant<int, 0>;
        using W1 = std::integral_constant<int, 1>;
        using NC = std::false_type;
        using CR = std::true_type;
        // positions whose prefetch stays in this segment: j + 3 < P
        if (P > 4) {
            step(X, Y, 0, K0{}, W0{}, NC{});
            step(Y, X, 1, K1{}, W1{}, NC{});
        } else {
            step(X, Y, 0, K0{}, W0{}, CR{});
            step(Y, X, 1, K1{}, W1{}, CR{});
        }
        int j = 2;
        for (; j + 4 < P; j += 2) {
            step(X, Y, j, K2{}, W0{}, NC{});
            step(Y, X, j + 1, K2{}, W1{}, NC{});
        }
        for (; j + 1 < P; j += 2) {
            step(X, Y, j, K2{}, W0{}, CR{});
            step(Y, X, j + 1, K2{}, W1{}, CR{});
        }
        if (j < P)
            step(X, Y, j, K2{}, W0{}, CR{});
        if (!has_next)
            break;
        g = gn;
        r0 = 0;
        r1 = nr1;
        G = N;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <bool ALIGNED, bool TWO_W>
__global__ void __launch_bounds__(kWalkThreads, 1) walk_kernel(const __grid_constant__ WideParams p)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t smbase = (uint32_t)__cvta_generic_to_shared(sm);
    if (smbase + kSmMiscEnd > kHistAbs)
        __trap();  // the fixed counter address would overlap the scratch (never seen)
    unsigned char* hist = sm + (kHistAbs - smbase);
    const int tid = threadIdx.x;
    static_assert(sizeof(WideParams) <= 256 && sizeof(WideParams) % 4 == 0, "params copy");
    if (tid < (int)(sizeof(WideParams) / 4))  // read back after the zeroing barrier
        reinterpret_cast<uint32_t*>(sm + kSmParams)[tid] = reinterpret_cast<const uint32_t*>(&p)[tid];
    const WideParams& ps = *reinterpret_cast<const WideParams*>(sm + kSmParams);
    const int warp = tid >> 5;
    phase(0);
    // Touch every 64-byte line of the parameter block at once: a launch's
    // parameters are cold in the constant cache, and the prologue's branches
    // on them would otherwise serialise one miss per line.
    asm volatile("" ::"l"(p.px), "r"(p.band_rows), "l"(p.T), "r"(p.epoch), "l"(p.cta_q),
                 "l"(p.acc), "l"(p.hist_out), "l"(p.t0s), "l"(p.status));
    if (p.early_trigger)
        pdl_trigger();  // pipeline depth > 1: the next launch takes the SMs this grid leaves free
    const long long rb = blockIdx.x;
    const long long cs = rb * p.cta_q + (rb < p.cta_r ? rb : p.cta_r);
    const long long ce = cs + p.cta_q + (rb < p.cta_r ? 1 : 0);

    bool zeroed = false;
    bool flushed = false;
    if (cs < ce) {
        int i_first = 0, i_last = 0;
        if (p.n > 1) {
            i_first = (int)(cs / p.upi);
            i_last = (int)((ce - 1) / p.upi);
        }
        // the first image's border slice arrives with the first ring rows
        const BorderSlice bs = border_slice(p, i_first);
        if (tid == 0)
            *reinterpret_cast<BorderSlice*>(sm + kSmBslice) = bs;
        const bool prefetched = bs.xb - bs.xa <= kBorderPx;
        if (prefetched)
            border_prefetch(p, i_first, bs, smbase + kSmBorder);
        for (int img = i_first; img <= i_last; ++img) {
            const long long ibase = (long long)img * p.upi;
            const long long a = (cs > ibase ? cs : ibase) - ibase;
            const long long b = (ce < ibase + p.upi ? ce : ibase + p.upi) - ibase;
            const uint8_t* base = p.px + (size_t)img * p.image_stride;
            for (long long ea = a; ea < b; ea += p.epoch) {
                const long long eb = ea + p.epoch < b ? ea + p.epoch : b;
                const long long n = eb - ea;
                const long long wa = ea + n * warp / kWalkWarps;
                const long long wb = ea + n * (warp + 1) / kWalkWarps;
                walk_range<ALIGNED, TWO_W>(p, sm, hist, smbase, base, wa, wb, !zeroed);
                warp_end();
                zeroed = true;
                __syncthreads();
                if (eb < b) {
                    for (int t = tid; t < (TWO_W ? 512 : 256); t += kWalkThreads)
                        spill_w(sm, hist, t);
                    __syncthreads();
                }
            }
            if (img == i_last) {
                phase(2);
                pdl_trigger();  // the next launch may start as SMs free up
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");  // border words (walk-less threads)
            flush_image(ps, img, sm, hist, img < i_last, TWO_W, prefetched && img == i_first, img == i_first);
            // (the last image: no re-zeroing)
            flushed = true;
        }
    }
    if (!flushed)
        pdl_trigger();
    phase(7);
}

// ---------------------------------------------------------------------------
// K5 twalk_kernel: batches of small images with the three-event column walk.
// The 32 lanes of every warp are split into NG = 32/LG lane groups; group g
// of all 16 warps walks image i0 + g of the round, so the image's counters
// are exactly its LG lane stripes of the shared block (conflict free across
// images) and one round accumulates NG whole images.  Walker (warp w, lane
// l in group g) takes task w*LG + l of its image: segment column task % S,
// rows [R*(task/S), +R).  Each group's first / last lane also copies the 16
// bytes left / right of the group's run into the group's pads.  After the
// walk, warp g rebuilds image i0+g's curve straight from its stripes (K3) and
// zeroes them; the per-image selection runs in select_kernel (K4).
// ---------------------------------------------------------------------------
struct TwParams {
    const uint8_t* px;
    size_t pitch;
    size_t image_stride;
    int n, w, h;
    int S;  // segments per row
    int R;  // rows per walk
    int C;  // walk chunks per image (S * C <= 16 * LG)
    uint64_t* sums;
    uint64_t* cards;
    uint32_t* hist_out;  // [n][256] pixel histogram, or null
};

// K5 per-image totals scratch (u32, padded): hs[512] at pad16, then
// h0, b0, h1, b1 [256] at pad8 (kTwArr words each)
constexpr int kTwArr = 288;                               // pad8(255) = 286
constexpr int kTwH = 560;                                 // pad16(511) = 542
__device__ __forceinline__ int pad8(int x) { return x + (x >> 3); }    // 9*lane + j: conflict free
__device__ __forceinline__ int pad16(int x) { return x + (x >> 4); }   // 17*lane + c
constexpr int kTwImgWords = (kTwH + 4 * kTwArr + 3) / 4 * 4;

template <int LG>
struct TwLayout {
    static constexpr int NG = 32 / LG;
    // 32 lane segments (512 B, 128-byte aligned), then 2 pads per group
    static constexpr uint32_t kSlot = (512 + 32 * NG + 127) / 128 * 128;
    static constexpr uint32_t kRing = 0;  // + up to 127 B of alignment
    static constexpr uint32_t kRingBytes = kTwWarps * kRingSlots * kSlot + 128;
    static constexpr uint32_t kCorr = kRingBytes;  // int[NG][256]
    static constexpr uint32_t kTot = kCorr + NG * 1024;  // i64 [3][16 warps][NG] scan carries
    static constexpr uint32_t kEnd = kTot + 3 * 16 * NG * 8;
    static_assert(kEnd + 1024 <= kHistAbs, "K5 scratch under the counter block");
};

__device__ __forceinline__ LaneGeo tw_geo(const TwParams& p, long long img, int task)
{
    LaneGeo L;
    const bool act = img < p.n && task < p.S * p.C;
    const int s = act ? task % p.S : 0;
    const int c = act ? task / p.S : 0;
    L.x0 = s << 4;
    L.e = p.w - 1 - L.x0;
    if (act) {
        L.y0 = c * p.R;
        L.nrows = min(p.R, p.h - L.y0);
        L.jlo = L.y0 == 0 ? 1 : 0;
        L.jcl = p.h - L.y0;
    } else {
        L.y0 = 1;
        L.nrows = 0;
        L.jlo = 0;
        L.jcl = 0;
    }
    L.p = p.px + (size_t)(act ? img : 0) * p.image_stride + (long long)(L.y0 - 1) * (long long)p.pitch +
          L.x0;
    return L;
}

template <bool ALIGNED, int LG>
__global__ void __launch_bounds__(kTwThreads, 1) twalk_kernel(const TwParams p)
{
    using namespace kohler_walk;
    using Lay = TwLayout<LG>;
    constexpr int NG = Lay::NG;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t smbase = (uint32_t)__cvta_generic_to_shared(sm);
    if (smbase + Lay::kEnd > kHistAbs)
        __trap();
    unsigned char* hist = sm + (kHistAbs - smbase);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane / LG, lig = lane % LG;
    const uint32_t lane4 = (uint32_t)lane * 4u;
    const uint32_t kneg = kHistAbs - lane4;
    const uint32_t dummy = kHistAbs + kDummy + lane4;
    const uint32_t corr_g = smbase + Lay::kCorr + (uint32_t)g * 1024u;
    const uint32_t corr_base = corr_g - (lane4 >> 6);
    const uint32_t pitch = (uint32_t)p.pitch;
    const int task = warp * LG + lig;
    const int P = p.R + 2;
    const uint32_t ring = (smbase + Lay::kRing + 127u) & ~127u;
    const uint32_t seg0 = ring + (uint32_t)warp * (kRingSlots * Lay::kSlot) + (uint32_t)lane * 16u;
    const uint32_t padl = 512u + 32u * g - 16u * lane;  // group pads, relative to the segment
    const uint32_t padr = padl + 16u;
    auto geo = [&](long long i0) {
        LaneGeo L = tw_geo(p, i0 + g, task);
        L.pd = lig == 0 ? -16 : 16;
        L.pds = (int)(lig == 0 ? padl : padr);
        L.pad = ((lig == 0) & (L.x0 > 0)) | ((lig == LG - 1) & (L.e > 15)) ? 1u : 0u;
        return L;
    };
    const long long stride = (long long)gridDim.x * NG;
    long long i0 = (long long)blockIdx.x * NG;
    LaneGeo G = geo(i0);
    fetch_row(G, 0, pitch, seg0);
    fetch_row(G, 1, pitch, seg0 + Lay::kSlot);
    fetch_row(G, 2, pitch, seg0 + 2 * Lay::kSlot);
    {
        uint4* z = reinterpret_cast<uint4*>(hist);
        for (int i = tid; i < (int)(kHistBytes / 16); i += kTwThreads)
            z[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < NG * 256; i += kTwThreads)
            reinterpret_cast<int*>(sm + Lay::kCorr)[i] = 0;
    }
    __syncthreads();
    bool waited = false;
    Car X, Y;
    uint32_t pos = 0;
#ifdef KOHLER_PHASES  // tools/tile_probe.cu: per-CTA cycles of the round phases
    long long tw_t = clock64(), tw_acc[5] = {0, 0, 0, 0, 0};
#define TWCYC(i) do { const long long t_ = clock64(); tw_acc[i] += t_ - tw_t; tw_t = t_; } while (0)
#else
#define TWCYC(i) do { } while (0)
#endif
    for (; i0 < p.n; i0 += stride) {
        const bool has_next = i0 + stride < p.n;
        LaneGeo N = G;
        const GroupFlags F = group_flags(G, ALIGNED);
        const bool row_start = G.x0 == 0, row_end = G.e <= 15;
        NbrSel nb;  // neighbour bytes: shuffles inside the group, pads at its ends
        nb.l_own = G.x0 == 0;
        nb.l_pad = !nb.l_own && lig == 0;
        nb.r_own = G.e <= 15;
        nb.r_pad = !nb.r_own && lig == LG - 1;
        nb.pad = nb.l_pad || nb.r_pad;
        nb.pad_off = lig == 0 ? padl + 15u : padr;
        auto step = [&](Car& D, Car& C, int j, auto kind, auto wc, auto cross) {
            constexpr int KIND = decltype(kind)::value;
            constexpr int WC = decltype(wc)::value;
            constexpr bool CROSS = decltype(cross)::value;
            constexpr uint32_t kOffW = WC ? kOffW1 : kOffW0;
            const uint32_t q = pos + (uint32_t)j;
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncwarp();
            Row r;  // read first: the prefetch issue covers the LDS latency
            read_row_shfl(r, seg0 + (q & 3u) * Lay::kSlot, nb);
            const uint32_t pref = seg0 + ((q + 3u) & 3u) * Lay::kSlot;
            if (!CROSS || j + 3 < P)
                fetch_row(G, j + 3, pitch, pref);
            else if (has_next)
                fetch_row(N, j + 3 - P, pitch, pref);
            else
                asm volatile("cp.async.commit_group;" ::: "memory");
            absorb<ALIGNED>(D, r, lane4, G.e);
            if (KIND == 1) {
                const bool has_up = G.y0 > 0;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    D.ue[jj] = has_up ? qstep(qfrom(C.e[jj]), D.e[jj]) : kNeutral;
                    D.uo[jj] = has_up ? qstep(qfrom(C.o[jj]), D.o[jj]) : kNeutral;
                }
            }
            if (KIND < 2)
                return;
            const bool live = j - 2 < G.nrows;
            uint32_t qre[4], qro[4], qde[4], qdo[4], Be[4], Bo[4];
            pair_q(C, D.e, D.o, qre, qro, qde, qdo);
            b_terms(C, qre, qro, qde, qdo, Be, Bo);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                D.ue[jj] = qde[jj];
                D.uo[jj] = qdo[jj];
            }
            const uint32_t Arn = __byte_perm(C.rn, lane4, 0x5504);
            if (ALIGNED || !F.ragged) {
                if (live) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_add_imm<kHistAbs + kOffW>(C.A[i], b_of(Be, Bo, i));
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_inc(C.A[i] + (i < 15 ? C.A[i + 1] : Arn) + kneg);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_inc(C.A[i] + D.A[i] + kneg);
                }
            } else if (live) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const bool real = i <= G.e;
                    red_add_imm<kHistAbs + kOffW>(C.A[i], real ? b_of(Be, Bo, i) : 0u);
                    red_inc(real ? C.A[i] + (i < 15 ? C.A[i + 1] : Arn) + kneg : dummy);
                    red_inc(real ? C.A[i] + D.A[i] + kneg : dummy);
                }
            }
            if (F.edge && live) {
                if (row_start)
                    red_add(corr_base + (C.A[0] >> 6), 1u);
                if (row_end)
                    red_add(corr_base + (Arn >> 6), 0xFFFFFFFFu);
            }
        };
        using K0 = std::integral_constant<int, 0>;
        using K1 = std::integral_constant<int, 1>;
        using K2 = std::integral_constant<int, 2>;
        using W0 = std::integral_constant<int, 0>;
        using W1 = std::integral_constant<int, 1>;
        using NC = std::false_type;
        using CR = std::true_type;
        if (P > 4) {
            step(X, Y, 0, K0{}, W0{}, NC{});
            step(Y, X, 1, K1{}, W1{}, NC{});
        } else {
            if (has_next)
                N = geo(i0 + stride);
            step(X, Y, 0, K0{}, W0{}, CR{});
            step(Y, X, 1, K1{}, W1{}, CR{});
        }
        int j = 2;
        for (; j + 4 < P; j += 2) {
            step(X, Y, j, K2{}, W0{}, NC{});
            step(Y, X, j + 1, K2{}, W1{}, NC{});
        }
        if (has_next)
            N = geo(i0 + stride);
        for (; j + 1 < P; j += 2) {
            step(X, Y, j, K2{}, W0{}, CR{});
            step(Y, X, j + 1, K2{}, W1{}, CR{});
        }
        if (j < P)
            step(X, Y, j, K2{}, W0{}, CR{});
        // border rows of the image: first row +1, last row -1 (its down pairs
        // were emitted as equal fakes: the down row was the row itself)
        if (__any_sync(0xFFFFFFFFu, G.nrows > 0 && (G.y0 == 0 || G.y0 + G.nrows == p.h))) {
            const int nreal = ALIGNED ? 16 : min(16, G.e + 1);
            if (G.nrows > 0 && G.y0 == 0) {
                const uint8_t* rp = G.p + p.pitch;
                for (int i = 0; i < nreal; ++i)
                    red_add(corr_g + ((uint32_t)rp[i] << 2), 1u);
            }
            if (G.nrows > 0 && G.y0 + G.nrows == p.h) {
                const uint8_t* rp = G.p + (size_t)G.nrows * p.pitch;
                for (int i = 0; i < nreal; ++i)
                    red_add(corr_g + ((uint32_t)rp[i] << 2), 0xFFFFFFFFu);
            }
        }
        __syncthreads();
        TWCYC(0);  // walk (incl. the wait for the slowest warp)
        if (!waited) {
            pdl_wait();  // the previous launch may still read our outputs
            waited = true;
        }
        if constexpr (LG == 4) {
            // Cooperative flush for 8 images per round (C5): warp w owns the
            // keys [16 w, 16 w + 16) of all 8 images; lane L takes image
            // L & 7, keys t0 .. t0 + 3 (t0 = 16 w + 4 (L >> 3)).  A group's 4
            // lane words of a counter row are one 16-byte piece, and the 8
            // lanes of a quarter warp (one LDS.128 wavefront) hit 8 bank quads, so
            // the counters are read once, conflict free, straight into the
            // per-image combinations; the scans run across the 4 lanes of an
            // image and then across warps (two small carry exchanges).  No
            // transposed scratch copy, no second clearing pass.
            // (the 8 lanes of each quarter warp -- one LDS.128 wavefront --
            // take 8 different images, i.e. 8 different bank quads)
            const int gi = lane & 7, q4 = lane >> 3;
            const int t0 = 16 * warp + 4 * q4;
            auto grp = [&](int row, int half) -> uint4 {
                return *reinterpret_cast<const uint4*>(hist + row * 256 + half * 128 + gi * 16);
            };
            auto wsum = [](const uint4& v, long long& h, long long& b) {
                h += (long long)((v.x & 0xFFFFu) + (v.y & 0xFFFFu) + (v.z & 0xFFFFu) + (v.w & 0xFFFFu));
                b += (long long)((v.x >> 16) + (v.y >> 16) + (v.z >> 16) + (v.w >> 16));
            };
            long long hv[5] = {0, 0, 0, 0, 0};  // hist(t0 - 1 + i)
            long long cd[4], h2[4];
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const int t = t0 - 1 + i;
                long long hh = 0, bb = 0;
                if (t >= 0) {
                    wsum(grp(t, 1), hh, bb);        // W copy 0
                    wsum(grp(256 + t, 1), hh, bb);  // W copy 1
                }
                hv[i] = hh;
                if (i > 0)
                    cd[i - 1] = bb - 4ll * hh;
            }
            long long hs[9];  // Hs rows 2 t0 - 3 .. 2 t0 + 5
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const int r = 2 * t0 - 3 + i;
                long long v = 0;
                if (r >= 0) {
                    const uint4 c = grp(r, 0);
                    v = (long long)c.x + c.y + c.z + c.w;
                }
                hs[i] = v;
            }
            const int* cr = reinterpret_cast<const int*>(sm + Lay::kCorr + gi * 1024);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int u = t0 + i;  // h2(u) = 4 hist(u-1) - corr(u-1) - hs(2u-3) - 2 hs(2u-2) - hs(2u-1)
                h2[i] = u == 0 ? 0
                               : 4ll * hv[i] - (long long)cr[u - 1] - hs[2 * i] - 2ll * hs[2 * i + 1] -
                                     hs[2 * i + 2];
            }
            // hs[0] (row 2 t0 - 3) is counted for u = t0 only when u >= 2: a
            // negative row is 0 already, so the formula matches warp_curve256's
            uint32_t hist_keep[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                hist_keep[i] = (uint32_t)hv[i + 1];
            __syncthreads();  // every counter read: clear the block for the next round
            {
                uint4* z = reinterpret_cast<uint4*>(hist);
                for (int i = tid; i < (int)(kHistBytes / 16); i += kTwThreads)
                    z[i] = make_uint4(0, 0, 0, 0);
            }
            // scans: lane-local, then across the image's 4 lanes (a quad)
            long long* tot = reinterpret_cast<long long*>(sm + Lay::kTot);  // [3][16][NG]
            auto quad_scan = [&](long long (&v)[4]) -> long long {
#pragma unroll
                for (int i = 1; i < 4; ++i)
                    v[i] += v[i - 1];
                long long x = v[3];  // the image's 4 lanes are gi, gi + 8, gi + 16, gi + 24
#pragma unroll
                for (int off = 1; off < 4; off <<= 1) {
                    const long long y = __shfl_up_sync(0xFFFFFFFFu, x, 8 * off);
                    if (q4 >= off)
                        x += y;
                }
                const long long ex = x - v[3];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    v[i] += ex;
                return __shfl_sync(0xFFFFFFFFu, x, 24 + gi);  // the image's (= warp's) total
            };
            const long long tc = quad_scan(cd);
            const long long tg = quad_scan(h2);  // h2 -> g (sum first difference)
            if (q4 == 0) {
                tot[(0 * 16 + warp) * NG + gi] = tc;
                tot[(1 * 16 + warp) * NG + gi] = tg;
            }
            __syncthreads();
            long long cc = 0, cg = 0;
            for (int w2 = 0; w2 < warp; ++w2) {
                cc += tot[(0 * 16 + w2) * NG + gi];
                cg += tot[(1 * 16 + w2) * NG + gi];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                cd[i] += cc;  // card
                h2[i] += cg;  // g
            }
            const long long ts = quad_scan(h2);  // g -> sum, without the carry of earlier warps' g
            if (q4 == 0)
                tot[(2 * 16 + warp) * NG + gi] = ts;
            __syncthreads();
            long long cs = 0;
            for (int w2 = 0; w2 < warp; ++w2)
                cs += tot[(2 * 16 + w2) * NG + gi];
            const long long im = i0 + gi;
            if (im < p.n) {
                uint64_t* os = p.sums + (size_t)im * 256 + t0;
                uint64_t* oc = p.cards + (size_t)im * 256 + t0;
                *reinterpret_cast<ulonglong2*>(oc) = make_ulonglong2((uint64_t)cd[0], (uint64_t)cd[1]);
                *reinterpret_cast<ulonglong2*>(oc + 2) = make_ulonglong2((uint64_t)cd[2], (uint64_t)cd[3]);
                *reinterpret_cast<ulonglong2*>(os) =
                    make_ulonglong2((uint64_t)(h2[0] + cs), (uint64_t)(h2[1] + cs));
                *reinterpret_cast<ulonglong2*>(os + 2) =
                    make_ulonglong2((uint64_t)(h2[2] + cs), (uint64_t)(h2[3] + cs));
                if (p.hist_out) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        p.hist_out[(size_t)im * 256 + t0 + i] = hist_keep[i];
                }
            }
            TWCYC(1);
            for (int i = tid; i < NG * 256; i += kTwThreads)
                reinterpret_cast<int*>(sm + Lay::kCorr)[i] = 0;
        } else
        {
            // 1. every thread: 2*NG (half-row, group) cells, contiguous 16-byte
            //    pieces across a warp (conflict free): read, sum the group's LG
            //    lane words (fields for W), clear
            constexpr int PER = 1024 * NG / kTwThreads;
            uint32_t va[PER], vb[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int idx = tid + kTwThreads * q;
                const int rh = idx / NG, gg = idx % NG;
                uint32_t a = 0, b = 0;
#pragma unroll
                for (int q4 = 0; q4 < LG / 4; ++q4) {
                    uint4* cell = reinterpret_cast<uint4*>(hist + rh * 128 + gg * LG * 4 + 16 * q4);
                    const uint4 v = *cell;
                    if (rh & 1) {  // W word: hist | B << 16
                        a += (v.x & 0xFFFFu) + (v.y & 0xFFFFu) + (v.z & 0xFFFFu) + (v.w & 0xFFFFu);
                        b += (v.x >> 16) + (v.y >> 16) + (v.z >> 16) + (v.w >> 16);
                    } else {
                        a += v.x + v.y + v.z + v.w;
                    }
                    *cell = make_uint4(0, 0, 0, 0);
                }
                va[q] = a;
                vb[q] = b;
            }
            __syncthreads();
            TWCYC(1);
            // 2. per-image totals into a padded scratch carved out of the (now
            //    zero) counter block: hs[s] at s + s/16, the other arrays at
            //    x + x/8 (conflict-free lane-blocked reads of warp_curve256)
            uint32_t* scr = reinterpret_cast<uint32_t*>(hist);
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int idx = tid + kTwThreads * q;
                const int rh = idx / NG, gg = idx % NG;
                const int row = rh >> 1;
                uint32_t* base = scr + gg * kTwImgWords;
                if (rh & 1) {
                    const int key = row & 255, cp = row >> 8;
                    base[kTwH + cp * 2 * kTwArr + pad8(key)] = va[q];
                    base[kTwH + cp * 2 * kTwArr + kTwArr + pad8(key)] = vb[q];
                } else {
                    base[pad16(row)] = va[q];
                }
            }
            __syncthreads();
            TWCYC(2);
            if (warp < NG && i0 + warp < p.n) {
                // 3. K3 for image i0 + warp
                const uint32_t* base = scr + warp * kTwImgWords;
                const uint32_t* h0 = base + kTwH;
                const uint32_t* b0 = h0 + kTwArr;
                const uint32_t* h1 = b0 + kTwArr;
                const uint32_t* b1 = h1 + kTwArr;
                const int* cr = reinterpret_cast<const int*>(sm + Lay::kCorr + warp * 1024);
                auto histv = [&](int v) { return (long long)h0[pad8(v)] + (long long)h1[pad8(v)]; };
                auto hs = [&](int s) { return (long long)base[pad16(s)]; };
                uint64_t card[8], sum[8];
                warp_curve256_regs(
                    [&](int t) {
                        return (long long)b0[pad8(t)] + (long long)b1[pad8(t)] - 4ll * histv(t);
                    },
                    [&](int u) -> long long {
                        if (u == 0)
                            return 0;
                        long long r2 = 4ll * histv(u - 1) - (long long)cr[u - 1] -
                                       2ll * hs(2 * u - 2) - hs(2 * u - 1);
                        if (u >= 2)
                            r2 -= hs(2 * u - 3);
                        return r2;
                    },
                    card, sum);
                const long long im = i0 + warp;
                uint64_t* os = p.sums + (size_t)im * 256 + lane * 8;
                uint64_t* oc = p.cards + (size_t)im * 256 + lane * 8;
#pragma unroll
                for (int jj = 0; jj < 8; jj += 2) {
                    *reinterpret_cast<ulonglong2*>(os + jj) = make_ulonglong2(sum[jj], sum[jj + 1]);
                    *reinterpret_cast<ulonglong2*>(oc + jj) = make_ulonglong2(card[jj], card[jj + 1]);
                }
                if (p.hist_out) {
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        p.hist_out[(size_t)im * 256 + lane * 8 + jj] = (uint32_t)histv(lane * 8 + jj);
                }
            }
            __syncthreads();
            TWCYC(3);
            // 4. clear the scratch and the border terms for the next round
            uint4* z = reinterpret_cast<uint4*>(hist);
            for (int i = tid; i < NG * kTwImgWords / 4; i += kTwThreads)
                z[i] = make_uint4(0, 0, 0, 0);
            for (int i = tid; i < NG * 256; i += kTwThreads)
                reinterpret_cast<int*>(sm + Lay::kCorr)[i] = 0;
        }
        __syncthreads();
        TWCYC(4);
        pos += (uint32_t)P;
        G = N;
    }
#ifdef KOHLER_PHASES
    if (threadIdx.x == 0 && blockIdx.x < 2048)
        for (int i = 0; i < 5; ++i)
            g_phase[blockIdx.x][i] = (unsigned long long)tw_acc[i];
#endif
#undef TWCYC
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (!waited)
        pdl_wait();
    pdl_trigger();
}

// Definition-level oracle kernel: block t scans every
// ordered 4-neighbour pair (x0 <= t < x1) of the image, like
// proj/src/direct.cpp:18-38.  Shares nothing with K1.  out: sum[256], card[256].
__global__ void __launch_bounds__(256) direct_kernel(const uint8_t* px, int w, int h, size_t pitch,
                                                     unsigned long long* out)
{
    const int t = blockIdx.x;
    unsigned long long s = 0, c = 0;
    const long long npx = (long long)w * h;
    for (long long i = threadIdx.x; i < npx; i += blockDim.x) {
        const int y = (int)(i / w), x = (int)(i - (long long)y * w);
        const int v0 = px[(size_t)y * pitch + x];
        if (v0 > t)
            continue;
        const int dx[4] = {1, -1, 0, 0};
        const int dy[4] = {0, 0, 1, -1};
        for (int d = 0; d < 4; ++d) {
            const int x1 = x + dx[d], y1 = y + dy[d];
            if (x1 < 0 || x1 >= w || y1 < 0 || y1 >= h)
                continue;
            const int v1 = px[(size_t)y1 * pitch + x1];
            if (v1 > t) {
                c += 1;
                s += (unsigned long long)min(v1 - t, t - v0);
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
        c += __shfl_xor_sync(0xFFFFFFFFu, c, off);
    }
    __shared__ unsigned long long ws[8], wc[8];
    if ((threadIdx.x & 31) == 0) {
        ws[threadIdx.x >> 5] = s;
        wc[threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long ts = 0, tc = 0;
        for (int i = 0; i < 8; ++i) {
            ts += ws[i];
            tc += wc[i];
        }
        out[t] = ts;
        out[256 + t] = tc;
    }
}

// Standalone selection: one warp per curve.  mode 0: input (sum, card);
// mode 1: input (values, defined).
struct SelectParams {
    const uint64_t* sums;
    const uint64_t* cards;
    const double* in_values;
    const uint8_t* in_defined;
    int n_curves;
    int levels;
    int k;
    int want_select;  // 0: only values/defined
    double* values;
    uint8_t* defined;
    int* t0s;
    int* topks;
    int* topk_counts;
    int* status;
};

__global__ void __launch_bounds__(32) select_kernel(const SelectParams p)
{
    extern __shared__ __align__(16) unsigned char sm[];
    // the next launch may start at once: every kernel that reads this one's
    // outputs executes griddepcontrol.wait before it does
    pdl_trigger();
    pdl_wait();  // curves may come from the preceding (PDL-overlapped) launch
    const int n = p.levels;
    const int cidx = blockIdx.x;
    double* val = reinterpret_cast<double*>(sm);
    double* rv = val + n;
    double* mv = rv + n;
    int* rt = reinterpret_cast<int*>(mv + n);
    int* mt = rt + n;
    uint8_t* def = reinterpret_cast<uint8_t*>(mt + n);
    const size_t off = (size_t)cidx * n;
    for (int t = threadIdx.x; t < n; t += 32) {
        double v;
        uint8_t d;
        if (p.sums) {
            const uint64_t cc = p.cards[off + t];
            v = cc ? (double)p.sums[off + t] / (double)cc : 0.0;
            d = cc ? 1 : 0;
        } else {
            v = p.in_values[off + t];
            d = p.in_defined[off + t] ? 1 : 0;
        }
        val[t] = v;
        def[t] = d;
        if (p.values)
            p.values[off + t] = v;
        if (p.defined)
            p.defined[off + t] = d;
    }
    __syncwarp();
    if (!p.want_select)
        return;
    SelectScratch s{rv, rt, mv, mt};
    const int st = warp_select(val, def, n, p.k, s, p.t0s ? p.t0s + cidx : nullptr,
                               p.topks ? p.topks + (size_t)cidx * p.k : nullptr,
                               p.topk_counts ? p.topk_counts + cidx : nullptr);
    if (threadIdx.x == 0 && p.status)
        p.status[cidx] = st;
}

// Standalone selection for 256-level curves: one warp per curve, 8 curves per
// CTA, lane L holding thresholds 8L..8L+7 in registers (vector loads), the
// register-resident selection of kohler_walk.cuh.
__global__ void __launch_bounds__(256) select256_kernel(const SelectParams p)
{
    __shared__ double smv[8][128];
    __shared__ int smt[8][128];
    // the next launch may start at once: every kernel that reads this one's
    // outputs executes griddepcontrol.wait before it does
    pdl_trigger();
    pdl_wait();  // curves may come from the preceding (PDL-overlapped) launch
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const long long cidx = (long long)blockIdx.x * 8 + wq;
    if (cidx >= p.n_curves)
        return;
    const size_t off = (size_t)cidx * 256 + 8 * lane;
    double v[8];
    bool d[8];
    if (p.sums) {
        uint64_t s[8], c[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(p.sums + off + j);
            const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(p.cards + off + j);
            s[j] = a.x;
            s[j + 1] = a.y;
            c[j] = b.x;
            c[j + 1] = b.y;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            d[j] = c[j] != 0;
            v[j] = d[j] ? (double)s[j] / (double)c[j] : 0.0;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = p.in_values[off + j];
            d[j] = p.in_defined[off + j] != 0;
        }
    }
    if (p.values) {
#pragma unroll
        for (int j = 0; j < 8; j += 2)
            *reinterpret_cast<double2*>(p.values + off + j) = make_double2(v[j], v[j + 1]);
    }
    if (p.defined) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            lo |= (d[j] ? 1u : 0u) << (8 * j);
            hi |= (d[j + 4] ? 1u : 0u) << (8 * j);
        }
        *reinterpret_cast<uint2*>(p.defined + off) = make_uint2(lo, hi);
    }
    if (!p.want_select)
        return;
    const int st = kohler_walk::warp_select256_regs(
        v, d, p.k, smv[wq], smt[wq], p.t0s ? p.t0s + cidx : nullptr,
        p.topks ? p.topks + (size_t)cidx * p.k : nullptr, p.topk_counts ? p.topk_counts + cidx : nullptr);
    if (lane == 0 && p.status)
        p.status[cidx] = st;
}

// ---------------------------------------------------------------------------
// Segmentation: classify / quantize
// (proj/src/threshold.cpp:84-126) and the per-frame video pipeline
// (proj/src/bench.cpp:266-281).  hist_kernel: pixel histogram per image
// (lane-striped shared counters, only needed when no K1 ran); map_kernel:
// per image a 256-entry LUT (label = #thresholds < v, or the class mean
// rounded half up from the histogram, or identity for a frame without
// boundary), then one pass out = LUT[in].
// ---------------------------------------------------------------------------
struct MapParams {
    const uint8_t* px;
    size_t pitch, image_stride;
    uint8_t* out;
    size_t out_pitch, out_stride;
    int n, w, h;
    int mode;                 // 0 classify, 1 quantize
    const int* thresholds;    // [n][ts_stride]; or a single shared set (ts_stride == 0)
    int ts_stride;
    const int* ts_counts;     // [n] or null (then ts_count for all)
    int ts_count;
    const int* status;        // [n] or null: 1 = no boundary -> pass through
    const uint32_t* hist;     // [n][256] (quantize)
    int units_per_image;      // row ranges per image, one warp each
    int flat;                 // rows dense (pitch == out_pitch == w, w % 16 == 0), 16-aligned
    uint32_t seg_magic;       // floor(2^32 / segments per row) + 1
    int* counts_out;          // [n] or null: thresholds applied per image (0 if passed through)
};

// q = i / d for 0 <= i < 2^31 / d via multiply-high (magic = floor(2^32 / d) + 1)
__device__ __forceinline__ uint32_t div_magic(uint32_t i, uint32_t magic, uint32_t d)
{
    return d == 1 ? i : __umulhi(i, magic);
}

__global__ void __launch_bounds__(512) hist_kernel(const uint8_t* px, size_t pitch,
                                                   size_t image_stride, int w, int h,
                                                   int blocks_per_image, uint32_t magic,
                                                   uint32_t* hist)
{
    __shared__ uint32_t sh[256 * 32];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 256 * 32; i += 512)
        sh[i] = 0;
    __syncthreads();
    const int img = blockIdx.x / blocks_per_image, b = blockIdx.x % blocks_per_image;
    const int y0 = (int)((long long)h * b / blocks_per_image);
    const int y1 = (int)((long long)h * (b + 1) / blocks_per_image);
    const uint8_t* base = px + (size_t)img * image_stride;
    const uint32_t segs = (uint32_t)(w + 15) / 16;
    const uint32_t total = (uint32_t)(y1 - y0) * segs;
    for (uint32_t i = tid; i < total; i += 512) {
        const uint32_t q = div_magic(i, magic, segs);
        const int y = y0 + (int)q, s = (int)(i - q * segs);
        const uint8_t* rp = base + (size_t)y * pitch + 16 * s;
        const int nb = min(16, w - 16 * s);
        if (nb == 16 && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0)) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(rp));
            const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 16; ++j)
                atomicAdd(&sh[((wd[j >> 2] >> (8 * (j & 3))) & 0xFFu) * 32 + lane], 1u);
        } else {
            for (int j = 0; j < nb; ++j)
                atomicAdd(&sh[(uint32_t)rp[j] * 32 + lane], 1u);
        }
    }
    __syncthreads();
    if (tid < 256) {
        uint32_t s = 0;
        for (int l = 0; l < 32; ++l)
            s += sh[tid * 32 + ((l + tid) & 31)];
        if (s)
            atomicAdd(hist + (size_t)img * 256 + tid, s);
    }
}

// One warp per unit (an image, or a row range of a large one): the warp builds
// its image's LUT from the histogram with shuffles (no block barriers), then
// streams its rows with kMapUnroll 16-byte loads in flight per lane.
constexpr int kMapWarps = 8, kMapThreads = 32 * kMapWarps, kMapUnroll = 8;

struct MapLut {
    uint32_t y7, ny;      // threshold + 1 replicated per byte: low 7 bits; complement
    uint32_t m0, mx;      // class-0 byte replicated, class-0 ^ class-1
    const uint8_t* lut;   // 256 entries (shared)
};

// KIND 1: two classes, out = v > t ? m1 : m0 per byte (SWAR: borrow-free low-7
// compare, majority with the top bits, sign-replicating PRMT, select);
// KIND 2: identity; KIND 0: LUT
template <int KIND>
__device__ __forceinline__ uint32_t map_word(uint32_t x, const MapLut& m)
{
    if (KIND == 2)
        return x;
    if (KIND == 1) {
        const uint32_t d = (x | 0x80808080u) - m.y7;
        uint32_t ge, mask;
        asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(ge) : "r"(x), "r"(m.ny), "r"(d));
        asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(mask) : "r"(ge));
        return m.m0 ^ (mask & m.mx);
    }
    return (uint32_t)m.lut[x & 0xFFu] | ((uint32_t)m.lut[(x >> 8) & 0xFFu] << 8) |
           ((uint32_t)m.lut[(x >> 16) & 0xFFu] << 16) | ((uint32_t)m.lut[x >> 24] << 24);
}

template <int KIND>
__device__ __forceinline__ uint4 map16(uint4 v, const MapLut& m)
{
    return make_uint4(map_word<KIND>(v.x, m), map_word<KIND>(v.y, m), map_word<KIND>(v.z, m),
                      map_word<KIND>(v.w, m));
}

// rows [y0, y1) of one image by one warp
template <int KIND>
__device__ __forceinline__ void map_rows(const MapParams& p, const uint8_t* src, uint8_t* dst,
                                         int y0, int y1, const MapLut& m, int lane)
{
    if (p.flat) {
        // dense 16-aligned rows: one contiguous range, immediate-offset loads
        const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)y0 * p.w);
        uint4* d = reinterpret_cast<uint4*>(dst + (size_t)y0 * p.w);
        const uint32_t nv = (uint32_t)((size_t)(y1 - y0) * p.w / 16);
        uint32_t i = lane;
        for (; i + 32 * (kMapUnroll - 1) < nv; i += 32 * kMapUnroll) {
            uint4 v[kMapUnroll];
#pragma unroll
            for (int u = 0; u < kMapUnroll; ++u)
                v[u] = __ldg(s + i + 32 * u);
#pragma unroll
            for (int u = 0; u < kMapUnroll; ++u)
                d[i + 32 * u] = map16<KIND>(v[u], m);
        }
        for (; i < nv; i += 32)
            d[i] = map16<KIND>(__ldg(s + i), m);
        return;
    }
    const uint32_t segs = (uint32_t)(p.w + 15) / 16;
    const uint32_t total = (uint32_t)(y1 - y0) * segs;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | p.pitch |
                       reinterpret_cast<uintptr_t>(dst) | p.out_pitch) & 15) == 0;
    for (uint32_t i = lane; i < total; i += 32) {
        const uint32_t q = div_magic(i, p.seg_magic, segs);
        const int y = y0 + (int)q, s = (int)(i - q * segs);
        const uint8_t* rp = src + (size_t)y * p.pitch + 16 * s;
        uint8_t* wp = dst + (size_t)y * p.out_pitch + 16 * s;
        const int nb = min(16, p.w - 16 * s);
        if (nb == 16 && vec)
            *reinterpret_cast<uint4*>(wp) = map16<KIND>(__ldg(reinterpret_cast<const uint4*>(rp)), m);
        else
            for (int j = 0; j < nb; ++j)
                wp[j] = m.lut[rp[j]];
    }
}

__global__ void __launch_bounds__(kMapThreads) map_kernel(const MapParams p)
{
    __shared__ unsigned long long pre[kMapWarps][2][256];  // per-warp prefix sums (count, sum)
    __shared__ uint8_t luts[kMapWarps][256], cmeans[kMapWarps][256];
    pdl_wait();  // thresholds / histograms come from the preceding launches
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long unit = (long long)blockIdx.x * kMapWarps + wid;
    if (unit >= (long long)p.n * p.units_per_image)
        return;  // whole warp; only __syncwarp below
    const int img = (int)(unit / p.units_per_image), part = (int)(unit % p.units_per_image);
    uint8_t* lut = luts[wid];
    const int* ts = p.thresholds + (size_t)img * p.ts_stride;
    const bool pass = p.status && p.status[img] != 0;
    const int nts = pass ? 0 : p.ts_counts ? p.ts_counts[img] : p.ts_count;
    if (p.counts_out && part == 0 && lane == 0)
        p.counts_out[img] = nts;
    // label(v) = number of thresholds strictly below v (lower_bound on the
    // sorted set); class l holds the grey levels (ts[l-1], ts[l]]
    int label[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        label[j] = 0;
    for (int i = 0; i < nts; ++i) {
        const int t = ts[i];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            label[j] += t < lane * 8 + j;
    }
    if (pass || p.mode == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            lut[lane * 8 + j] = (uint8_t)(pass ? lane * 8 + j : label[j]);
    } else {
        const uint4* hp = reinterpret_cast<const uint4*>(p.hist + (size_t)img * 256 + lane * 8);
        const uint4 h0 = hp[0], h1 = hp[1];
        const uint32_t hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        unsigned long long pc[8], ps[8], c = 0, s = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c += hv[j];
            s += (unsigned long long)hv[j] * (unsigned)(lane * 8 + j);
            pc[j] = c;
            ps[j] = s;
        }
        unsigned long long ic = c, is = s;  // inclusive warp scan of the lane totals
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long yc = __shfl_up_sync(0xFFFFFFFFu, ic, off);
            const unsigned long long ys = __shfl_up_sync(0xFFFFFFFFu, is, off);
            if (lane >= off) {
                ic += yc;
                is += ys;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            pre[wid][0][lane * 8 + j] = pc[j] + ic - c;
            pre[wid][1][lane * 8 + j] = ps[j] + is - s;
        }
        __syncwarp();
        for (int l = lane; l <= nts; l += 32) {  // one class mean per lane
            const int lo = l == 0 ? -1 : min(max(ts[l - 1], -1), 255);
            const int hi = l == nts ? 255 : min(max(ts[l], -1), 255);
            unsigned long long cs = 0, cc = 0;
            if (hi > lo) {
                cc = pre[wid][0][hi] - (lo >= 0 ? pre[wid][0][lo] : 0ull);
                cs = pre[wid][1][hi] - (lo >= 0 ? pre[wid][1][lo] : 0ull);
            }
            cmeans[wid][l] = cc ? (uint8_t)((2 * cs + cc) / (2 * cc)) : 0;  // round half up
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
            lut[lane * 8 + j] = cmeans[wid][label[j]];
    }
    __syncwarp();
    MapLut m;
    m.lut = lut;
    // two classes: lut[0] / lut[255] are the class values (equal when the
    // threshold lies outside 0..254, so the compare result does not matter)
    const int y = min(max((nts >= 1 ? ts[0] : 0) + 1, 0), 255);
    m.y7 = (uint32_t)(y & 0x7F) * 0x01010101u;
    m.ny = ~((uint32_t)y * 0x01010101u);
    m.m0 = (uint32_t)lut[0] * 0x01010101u;
    m.mx = m.m0 ^ ((uint32_t)lut[255] * 0x01010101u);
    const int y0 = (int)((long long)p.h * part / p.units_per_image);
    const int y1 = (int)((long long)p.h * (part + 1) / p.units_per_image);
    const uint8_t* src = p.px + (size_t)img * p.image_stride;
    uint8_t* dst = p.out + (size_t)img * p.out_stride;
    if (pass)
        map_rows<2>(p, src, dst, y0, y1, m, lane);
    else if (nts == 1)
        map_rows<1>(p, src, dst, y0, y1, m, lane);
    else
        map_rows<0>(p, src, dst, y0, y1, m, lane);
}

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

// ---------------------------------------------------------------------------
// Colour ingest: Rec. 601 integer luma of interleaved
// RGB, exactly the reference's luma601 (proj/src/pnm.cpp:63-68), used by
// read_pnm for P6/P3 input (:110-136):
//     v = min((299 r + 587 g + 114 b + 500) / 1000, 255)
// HBM-bound (3 B read + 1 B written per pixel).  One thread converts 16
// pixels: three 16-byte loads, the weighted sums by two DP2A per pixel
// (16-bit weights x 8-bit samples, FMA pipe), the division by 1000 as one
// IMAD.HI with ceil(2^32 / 1000) (exact for t < 2^18: 704 t < 2^32), one
// 16-byte store.  Ragged row ends / unaligned buffers take a per-pixel loop.
// ---------------------------------------------------------------------------
struct LumaParams {
    const uint8_t* rgb;
    size_t rpitch, rstride;   // bytes between rows / images of the RGB input
    uint8_t* gray;
    size_t gpitch, gstride;
    int w, rows, n;
    int vec;                  // all bases / pitches / strides 16-byte aligned
    long long items;          // n * rows * ceil(w / 16)
    int nchunk;
};

constexpr uint32_t kLumaMagic = 4294968u;  // ceil(2^32 / 1000)

__device__ __forceinline__ uint32_t luma_div(uint32_t t) { return __umulhi(t, kLumaMagic); }

__device__ __forceinline__ uint32_t luma1(uint32_t r, uint32_t g, uint32_t b)
{
    return luma_div(299u * r + 587u * g + 114u * b + 500u);
}

// four pixels from three words r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3 -> packed bytes
__device__ __forceinline__ uint32_t luma4(uint32_t w0, uint32_t w1, uint32_t w2)
{
    constexpr uint32_t A = 299u | 587u << 16, B = 114u, C = 299u << 16, D = 587u | 114u << 16;
    const uint32_t p0 = luma_div(__dp2a_hi(B, w0, __dp2a_lo(A, w0, 500u)));
    const uint32_t p1 = luma_div(__dp2a_lo(D, w1, __dp2a_hi(C, w0, 500u)));
    const uint32_t p2 = luma_div(__dp2a_lo(B, w2, __dp2a_hi(A, w1, 500u)));
    const uint32_t p3 = luma_div(__dp2a_hi(D, w2, __dp2a_lo(C, w2, 500u)));
    return __byte_perm(p0 | p1 << 8, p2 | p3 << 8, 0x5410);
}

__global__ void __launch_bounds__(256) luma_kernel(const LumaParams p)
{
    for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < p.items;
         it += (long long)gridDim.x * blockDim.x) {
        const long long rowi = it / p.nchunk;
        const int c = (int)(it - rowi * p.nchunk);
        const int img = (int)(rowi / p.rows), y = (int)(rowi - (long long)img * p.rows);
        const uint8_t* src = p.rgb + (size_t)img * p.rstride + (size_t)y * p.rpitch + (size_t)c * 48;
        uint8_t* dst = p.gray + (size_t)img * p.gstride + (size_t)y * p.gpitch + (size_t)c * 16;
        const int x0 = c * 16;
        if (p.vec && x0 + 16 <= p.w) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
            const uint4 b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
            const uint4 d = __ldg(reinterpret_cast<const uint4*>(src) + 2);
            uint4 o;
            o.x = luma4(a.x, a.y, a.z);
            o.y = luma4(a.w, b.x, b.y);
            o.z = luma4(b.z, b.w, d.x);
            o.w = luma4(d.y, d.z, d.w);
            *reinterpret_cast<uint4*>(dst) = o;
        } else {
            const int e = min(16, p.w - x0);
            for (int i = 0; i < e; ++i)
                dst[i] = (uint8_t)luma1(src[3 * i], src[3 * i + 1], src[3 * i + 2]);
        }
    }
}

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
    bool wide_attr_set = false;
    bool select_attr_set = false;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev)
            cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

struct BatchOut {
    uint64_t* sums;
    uint64_t* cards;
    double* values;
    uint8_t* defined;
    int* t0s;
    int* topks;
    int* topk_counts;
    int* status;
};

int launch_luma(kohler_cuda_ctx* ctx, const uint8_t* rgb, int n, int w, int rows, size_t rpitch,
                size_t rstride, uint8_t* gray, size_t gpitch, size_t gstride, cudaStream_t st)
{
    if (n <= 0 || rows <= 0)
        return KOHLER_OK;
    LumaParams lp{};
    lp.rgb = rgb;
    lp.rpitch = rpitch;
    lp.rstride = rstride;
    lp.gray = gray;
    lp.gpitch = gpitch;
    lp.gstride = gstride;
    lp.w = w;
    lp.rows = rows;
    lp.n = n;
    lp.nchunk = (w + 15) / 16;
    lp.items = (long long)n * rows * lp.nchunk;
    auto al = [](uintptr_t x) { return x % 16 == 0; };
    lp.vec = al((uintptr_t)rgb) && al(rpitch) && (n == 1 || al(rstride)) && al((uintptr_t)gray) &&
             al(gpitch) && (n == 1 || al(gstride));
    const long long blocks = std::min<long long>((lp.items + 255) / 256, (long long)ctx->sm_count * 8);
    luma_kernel<<<(unsigned)blocks, 256, 0, st>>>(lp);
    KC_CUDA(cudaGetLastError());
    ctx->last_launches += 1;
    return KOHLER_OK;
}

int check_rgb(int n, int w, int h, size_t pitch, size_t stride)
{
    if (n < 0)
        return fail(KOHLER_INVALID_ARGUMENT, "image count must be >= 0");
    if (w < 1 || h < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "GrayImage: dimensions must be at least 1x1");
    if (pitch < 3 * (size_t)w)
        return fail(KOHLER_INVALID_ARGUMENT, "RGB row pitch must be >= 3 * width");
    if (n > 1 && stride < pitch * (size_t)h)
        return fail(KOHLER_INVALID_ARGUMENT, "image stride smaller than one image");
    return KOHLER_OK;
}

int check_image(int n, int w, int h, size_t pitch)
{
    if (n < 0)
        return fail(KOHLER_INVALID_ARGUMENT, "image count must be >= 0");
    if (w < 1 || h < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "GrayImage: dimensions must be at least 1x1");
    if (pitch < (size_t)w)
        return fail(KOHLER_INVALID_ARGUMENT, "row pitch must be >= width");
    return KOHLER_OK;
}

template <class Kern, class Arg>
cudaError_t launch_pdl(Kern kernel, unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                       const Arg& arg)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, arg);
}

// Launch K1 over n images whose buffers hold band_rows own rows (+ halo).
#ifndef KOHLER_SINGLE_W
#define KOHLER_SINGLE_W 0
#endif
constexpr bool kSingleW = KOHLER_SINGLE_W != 0;

int launch_wide(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int band_rows,
                int h_total, int r0, size_t pitch, size_t image_stride, int k, int select,
                const BatchOut& o, cudaStream_t stream, int no_finish = 0,
                uint32_t* hist_out = nullptr)
{
    if (n == 0)
        return KOHLER_OK;
    if (pitch >= (1ull << 31) / 64)
        return fail(KOHLER_INVALID_ARGUMENT, "row pitch too large");
    const int nseg = (w + 15) / 16;
    // Pipeline depth d > 1 (finishing launches only): each K1 takes 1/d of
    // the SMs (one more per launch for its finish_kernel) and triggers its
    // successor at once, so d consecutive launches run side by side and each
    // one's prologue / zeroing / flush / launch gap hides under the others'
    // walks.  One accumulator buffer suffices: a launch's flush REDGs only
    // after its griddepcontrol.wait, i.e. after the previous launch's
    // finish_kernel has read and reset the buffer.
    const int depth = no_finish ? 1 : std::max(1, ctx->depth);
    const int G_max = depth > 1 ? std::max(1, (ctx->sm_count - depth) / depth) : std::max(1, ctx->sm_count - 1);
    // Rows per column walk R: a walk's rows past the band end still cost
    // their steps, so prefer R dividing the band height; longer walks
    // amortise the per-segment prime row.
    long long R = 64;
    {
        double best = 1e30;
        for (long long r = 16; r <= 64; ++r) {
            const long long ch = (band_rows + r - 1) / r;
            const double waste = (double)(ch * r - band_rows) / band_rows + 0.5 / r;
            if (waste < best - 1e-12) {
                best = waste;
                R = r;
            }
        }
        R = std::min<long long>(R, std::max(1, band_rows));
    }
    const long long chunks = (band_rows + R - 1) / R;
    const long long T = chunks * nseg;
    const long long gpi = (T + 31) / 32;
    const long long upi = gpi * R;
    const long long U = upi * n;
    // One CTA per SM, leaving one SM free: with programmatic dependent launch
    // the next launch's CTAs then never wait for this launch's serial tail.
    // Small jobs: at least ~4 rows per warp.
    long long G = std::max(1ll, std::min<long long>((U + 4 * kWalkWarps - 1) / (4 * kWalkWarps), G_max));
    const int copies = n == 1 ? kAccCopiesSingle : 1;
    int rc = ctx->acc.ensure((size_t)n * copies * 512 * sizeof(unsigned long long), true);
    if (rc)
        return rc;
    rc = ctx->tickets.ensure((size_t)n * sizeof(unsigned), true);
    if (rc)
        return rc;

    WideParams p{};
    p.px = px;
    p.pitch = pitch;
    p.image_stride = image_stride;
    p.n = n;
    p.w = w;
    p.band_rows = band_rows;
    p.buf_rows = band_rows + (r0 + band_rows < h_total ? 1 : 0);
    p.h_total = h_total;
    p.r0 = r0;
    p.nseg = nseg;
    p.R = (int)R;
    p.T = T;
    p.gpi = gpi;
    p.upi = upi;
    p.total_units = U;
    // Events into one W lane word per epoch of E units (rows), split over
    // the warps in contiguous runs of k_w segments (k_w <= units_w / R + 2):
    // copy 0 takes ceil(L/2) rows per segment plus <= 1 halo row per
    // segment, 16 pixels each: <= 16 (E/2 + 1.5 (E/R + 2 W)) <= kMaxEvents.
    // One W copy (all positions, plus the halo rows): <= 16 (E + E/R + 2 W);
    // used when every CTA's range fits one such epoch (no spill at all), which
    // saves a quarter of the counter block's zeroing and flushing.
    bool two_w;
    {
        const double cap2 = (double)kohler_walk::kMaxEventsPerWord / 16.0 - 3.0 * kWalkWarps;
        const double cap1 = (double)kohler_walk::kMaxEventsPerWord / 16.0 - 2.0 * kWalkWarps;
        const long long e1 = (long long)std::max(1.0, std::floor(cap1 / (1.0 + 1.0 / (double)R)));
        const long long range = U / G + (U % G ? 1 : 0);
        // measured (r01 phase probe): one copy shortens zeroing / flushing by
        // 0.5 us but back-to-back same-word atomics slow the walk as much, so
        // two copies stay the default; one copy remains for ablation
        two_w = !kSingleW || range > e1;
        p.epoch = two_w ? (int)std::max(1.0, std::floor(cap2 / (0.5 + 1.5 / (double)R))) : (int)e1;
    }
    p.acc = static_cast<unsigned long long*>(ctx->acc.p);
    p.early_trigger = depth > 1 ? 1 : 0;
    p.copies = copies;
    p.tickets = static_cast<unsigned*>(ctx->tickets.p);
    p.cta_q = U / G;
    p.cta_r = U % G;
    p.seg_magic = nseg > 1 ? (unsigned long long)((((unsigned __int128)1) << 64) / (unsigned)nseg) + 1ull
                           : 0ull;
    p.k = k;
    p.select = select;
    p.no_finish = no_finish;
    p.hist_out = hist_out;
    p.sums = o.sums;
    p.cards = o.cards;
    p.values = o.values;
    p.defined = o.defined;
    p.t0s = o.t0s;
    p.topks = o.topks;
    p.topk_counts = o.topk_counts;
    p.status = o.status;

    const bool vec = (reinterpret_cast<uintptr_t>(px) % 16 == 0) && (pitch % 16 == 0) &&
                     (n == 1 || image_stride % 16 == 0);
    if (!vec) {
        // K1 reads 16-byte segments with cp.async: stage unaligned inputs
        const size_t dpitch = round_up((size_t)w, 16);
        const size_t dstride = dpitch * (size_t)p.buf_rows;
        rc = ctx->stage.ensure(dstride * (size_t)n);
        if (rc)
            return rc;
        uint8_t* d = static_cast<uint8_t*>(ctx->stage.p);
        if (n == 1 || image_stride == pitch * (size_t)p.buf_rows) {
            KC_CUDA(cudaMemcpy2DAsync(d, dpitch, px, pitch, (size_t)w, (size_t)p.buf_rows * n,
                                      cudaMemcpyDeviceToDevice, stream));
        } else {
            for (int i = 0; i < n; ++i)
                KC_CUDA(cudaMemcpy2DAsync(d + dstride * i, dpitch, px + image_stride * i, pitch,
                                          (size_t)w, (size_t)p.buf_rows, cudaMemcpyDeviceToDevice,
                                          stream));
        }
        p.px = d;
        p.pitch = dpitch;
        p.image_stride = dstride;
    }
    // the smem opt-in is per device; remember it per context
    if (!ctx->wide_attr_set) {
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<false, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        ctx->wide_attr_set = true;
    }
    ctx->last_grid = (int)G;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kWalkThreads);
    cfg.dynamicSmemBytes = kSmWideBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (w % 16 == 0)
        KC_CUDA(two_w ? cudaLaunchKernelEx(&cfg, walk_kernel<true, true>, p)
                      : cudaLaunchKernelEx(&cfg, walk_kernel<true, false>, p));
    else
        KC_CUDA(two_w ? cudaLaunchKernelEx(&cfg, walk_kernel<false, true>, p)
                      : cudaLaunchKernelEx(&cfg, walk_kernel<false, false>, p));
    ctx->last_launches += 1;
    if (!no_finish) {
        FinishParams fp{};
        fp.acc = p.acc;
        fp.copies = copies;
        fp.k = k;
        fp.select = select;
        fp.sums = o.sums;
        fp.cards = o.cards;
        fp.values = o.values;
        fp.defined = o.defined;
        fp.t0s = o.t0s;
        fp.topks = o.topks;
        fp.topk_counts = o.topk_counts;
        fp.status = o.status;
        KC_CUDA(launch_pdl(finish_kernel, (unsigned)n, 256, 0, stream, fp));
        ctx->last_launches += 1;
    }
    KC_CUDA(cudaGetLastError());
    return KOHLER_OK;
}


int launch_select(kohler_cuda_ctx* ctx, const SelectParams& sp, cudaStream_t stream)
{
    if (sp.n_curves == 0)
        return KOHLER_OK;
    if (sp.levels == 256) {
        KC_CUDA(launch_pdl(select256_kernel, (unsigned)((sp.n_curves + 7) / 8), 256, 0, stream, sp));
        ctx->last_launches += 1;
        return KOHLER_OK;
    }
    const size_t smem = (size_t)sp.levels * (8 * 3 + 4 * 2 + 1);
    if (!ctx->select_attr_set) {
        KC_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(kMaxSelectLevels * (8 * 3 + 4 * 2 + 1))));
        ctx->select_attr_set = true;
    }
    KC_CUDA(launch_pdl(select_kernel, (unsigned)sp.n_curves, 32, smem, stream, sp));
    ctx->last_launches += 1;
    return KOHLER_OK;
}

template <bool ALIGNED, int LG>
int launch_twalk_t(const TwParams& tp, unsigned G, cudaStream_t stream)
{
    static bool attr_set = false;  // per process; the attribute is per function
    if (!attr_set) {
        KC_CUDA(cudaFuncSetAttribute(twalk_kernel<ALIGNED, LG>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        attr_set = true;
    }
    KC_CUDA(launch_pdl(twalk_kernel<ALIGNED, LG>, G, kTwThreads, kSmWideBytes, stream, tp));
    return KOHLER_OK;
}

// K5 geometry for a batch of n w x h images: the smallest lane group LG (most
// images per round) whose 16 * LG walkers cover the image with walks of
// R <= 62 rows (a W lane word takes <= 16 warps * (R/2 + 1) * 16 <= 8191
// events per round).  Returns false when no LG fits (K1 is used instead).
bool twalk_geometry(int n, int w, int h, int& lg, int& R, int& C)
{
    const int S = (w + 15) / 16;
    for (int cand = 4; cand <= 32; cand *= 2) {
        if (32 / cand > n && cand < 32)
            continue;  // fewer images than groups: use bigger groups
        const int walkers = kTwWarps * cand;
        if (S > walkers)
            continue;
        const int c = walkers / S;
        const int r = (h + c - 1) / c;
        if (r > 62)
            continue;
        lg = cand;
        R = r;
        C = (h + r - 1) / r;
        return true;
    }
    return false;
}

// Batches of small images: K5 twalk_kernel (curves) + select_kernel (K4).
int launch_tile(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h, size_t pitch,
                size_t image_stride, int k, int select, const BatchOut& o, cudaStream_t stream,
                uint32_t* hist_out = nullptr)
{
    int lg = 0, R = 0, C = 0;
    if (!twalk_geometry(n, w, h, lg, R, C))
        return launch_wide(ctx, px, n, w, h, h, 0, pitch, image_stride, k, select, o, stream, 0,
                           hist_out);
    TwParams tp{};
    tp.px = px;
    tp.pitch = pitch;
    tp.image_stride = image_stride;
    tp.n = n;
    tp.w = w;
    tp.h = h;
    tp.S = (w + 15) / 16;
    tp.R = R;
    tp.C = C;
    tp.sums = o.sums;
    tp.cards = o.cards;
    tp.hist_out = hist_out;
    if (!tp.sums) {
        int rc = ctx->curves.ensure((size_t)n * 512 * sizeof(uint64_t));
        if (rc)
            return rc;
        tp.sums = static_cast<uint64_t*>(ctx->curves.p);
        tp.cards = tp.sums + (size_t)n * 256;
    }
    const bool vec = (reinterpret_cast<uintptr_t>(px) % 16 == 0) && (pitch % 16 == 0) &&
                     (image_stride % 16 == 0);
    if (!vec) {
        // cp.async reads 16-byte segments: stage unaligned inputs
        const size_t dpitch = round_up((size_t)w, 16);
        const size_t dstride = dpitch * (size_t)h;
        int rc = ctx->stage.ensure(dstride * (size_t)n);
        if (rc)
            return rc;
        uint8_t* d = static_cast<uint8_t*>(ctx->stage.p);
        if (image_stride == pitch * (size_t)h) {
            KC_CUDA(cudaMemcpy2DAsync(d, dpitch, px, pitch, (size_t)w, (size_t)h * n,
                                      cudaMemcpyDeviceToDevice, stream));
        } else {
            for (int i = 0; i < n; ++i)
                KC_CUDA(cudaMemcpy2DAsync(d + dstride * i, dpitch, px + image_stride * i, pitch,
                                          (size_t)w, (size_t)h, cudaMemcpyDeviceToDevice, stream));
        }
        tp.px = d;
        tp.pitch = dpitch;
        tp.image_stride = dstride;
    }
    const int ng = 32 / lg;
    const long long rounds = (n + ng - 1) / ng;
    const unsigned G = (unsigned)std::max(1ll, std::min<long long>(rounds, ctx->sm_count - 1));
    const bool aligned = w % 16 == 0;
    int rc = KOHLER_OK;
    switch (lg * 2 + (aligned ? 1 : 0)) {
    case 4 * 2 + 1: rc = launch_twalk_t<true, 4>(tp, G, stream); break;
    case 4 * 2: rc = launch_twalk_t<false, 4>(tp, G, stream); break;
    case 8 * 2 + 1: rc = launch_twalk_t<true, 8>(tp, G, stream); break;
    case 8 * 2: rc = launch_twalk_t<false, 8>(tp, G, stream); break;
    case 16 * 2 + 1: rc = launch_twalk_t<true, 16>(tp, G, stream); break;
    case 16 * 2: rc = launch_twalk_t<false, 16>(tp, G, stream); break;
    case 32 * 2 + 1: rc = launch_twalk_t<true, 32>(tp, G, stream); break;
    default: rc = launch_twalk_t<false, 32>(tp, G, stream); break;
    }
    if (rc)
        return rc;
    ctx->last_launches += 1;
    if (select || o.values || o.defined) {
        SelectParams sp{};
        sp.sums = tp.sums;
        sp.cards = tp.cards;
        sp.n_curves = n;
        sp.levels = 256;
        sp.k = k;
        sp.want_select = select;
        sp.values = o.values;
        sp.defined = o.defined;
        sp.t0s = o.t0s;
        sp.topks = o.topks;
        sp.topk_counts = o.topk_counts;
        sp.status = o.status;
        rc = launch_select(ctx, sp, stream);
    }
    return rc;
}

// Small images in batches go to K5, everything else to K1.
bool use_tile(int n, int w, int h) { return n >= 2 && (long long)w * h <= 65536; }

// Stage a host batch into the device, run, copy results back.
//
// The upload goes in two chunks on the context's copy stream, each followed
// (on the compute stream, after an event) by the launch that consumes it:
// the first ~90 % of the bytes, whose accumulation (~1 B/ns on the device)
// hides under the PCIe transfer (~0.05 B/ns) of the last ~10 %, then that
// tail.  Each extra DMA costs ~4 us of gap, so more chunks only lose.  A
// single large image is cut into two row bands (each launch accumulates into
// the image's accumulator; only the last one finishes the curve), a batch
// into two contiguous image ranges.  Small results come back in ONE
// device-to-host copy.
int host_batch(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h, size_t pitch,
               size_t image_stride, int k, int select, const BatchOut& host, int channels = 1)
{
    const size_t dpitch = round_up((size_t)w, 16);
    const size_t dstride = dpitch * (size_t)h;
    int rc = ctx->img.ensure(std::max<size_t>(dstride * (size_t)n, 16));
    if (rc)
        return rc;
    uint8_t* dimg = static_cast<uint8_t*>(ctx->img.p);
    // uploads land in dimg (grey) or, for RGB input, in the RGB staging
    // buffer, converted per chunk by luma_kernel into dimg
    const size_t wb = (size_t)w * channels;
    const size_t upitch = channels == 1 ? dpitch : round_up(wb, 16);
    const size_t ustride = upitch * (size_t)h;
    if (channels != 1) {
        rc = ctx->rgb.ensure(std::max<size_t>(ustride * (size_t)n, 16));
        if (rc)
            return rc;
    }
    uint8_t* dup = channels == 1 ? dimg : static_cast<uint8_t*>(ctx->rgb.p);
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    // device outputs, packed: sums | cards | values | defined | t0 | count | status | topk
    const size_t n256 = (size_t)n * 256;
    const size_t tail_off = round_up(n256 * 25, 16);
    const size_t bytes = tail_off + (size_t)n * 4 * 3 + (size_t)n * k * 4;
    rc = ctx->out.ensure(bytes + 64);
    if (rc)
        return rc;
    char* b = static_cast<char*>(ctx->out.p);
    BatchOut d{};
    const bool want_curve = true;  // curves always land in the packed block
    d.sums = want_curve ? reinterpret_cast<uint64_t*>(b) : nullptr;
    d.cards = want_curve ? reinterpret_cast<uint64_t*>(b + n256 * 8) : nullptr;
    d.values = host.values ? reinterpret_cast<double*>(b + n256 * 16) : nullptr;
    d.defined = host.defined ? reinterpret_cast<uint8_t*>(b + n256 * 24) : nullptr;
    d.t0s = reinterpret_cast<int*>(b + tail_off);
    d.topk_counts = d.t0s + n;
    d.status = d.topk_counts + n;
    d.topks = d.status + n;
    ctx->last_launches = 0;

    auto upload = [&](int i0, int i1, int y0, int y1) -> int {
        // images [i0, i1), rows [y0, y1) of each
        const size_t rows = (size_t)(y1 - y0);
        if (pitch == upitch && (i1 - i0 == 1 || image_stride == pitch * (size_t)h)) {
            const size_t off = (size_t)i0 * ustride + (size_t)y0 * upitch;
            const size_t len = (i1 - i0 == 1) ? rows * upitch : (size_t)(i1 - i0) * ustride;
            KC_CUDA(cudaMemcpyAsync(dup + off, px + (size_t)i0 * image_stride + (size_t)y0 * pitch,
                                    len, cudaMemcpyHostToDevice, cs));
        } else if (image_stride == pitch * (size_t)h && y0 == 0 && y1 == h) {
            KC_CUDA(cudaMemcpy2DAsync(dup + (size_t)i0 * ustride, upitch,
                                      px + (size_t)i0 * image_stride, pitch, wb,
                                      (size_t)h * (i1 - i0), cudaMemcpyHostToDevice, cs));
        } else {
            for (int i = i0; i < i1; ++i)
                KC_CUDA(cudaMemcpy2DAsync(dup + ustride * i + (size_t)y0 * upitch, upitch,
                                          px + image_stride * i + (size_t)y0 * pitch, pitch,
                                          wb, rows, cudaMemcpyHostToDevice, cs));
        }
        return KOHLER_OK;
    };
    auto to_gray = [&](int i0, int i1, int y0, int y1) -> int {
        if (channels == 1)
            return KOHLER_OK;
        return launch_luma(ctx, dup + (size_t)i0 * ustride + (size_t)y0 * upitch, i1 - i0, w,
                           y1 - y0, upitch, ustride, dimg + (size_t)i0 * dstride + (size_t)y0 * dpitch,
                           dpitch, dstride, st);
    };
    auto sub = [&](int i0) {
        BatchOut s = d;
        if (s.sums) {
            s.sums += (size_t)i0 * 256;
            s.cards += (size_t)i0 * 256;
        }
        if (s.values)
            s.values += (size_t)i0 * 256;
        if (s.defined)
            s.defined += (size_t)i0 * 256;
        s.t0s += i0;
        s.topk_counts += i0;
        s.status += i0;
        s.topks += (size_t)i0 * k;
        return s;
    };
    const bool tile = use_tile(n, w, h);
    const size_t total = (size_t)w * h * n;
    // split point (rows of the image, or images of the batch): 9/10
    const int units = n == 1 ? h : n;
    const int cut = total >= (4u << 20) && units >= 2 ? std::max(1, (int)((long long)units * 9 / 10)) : units;
    const int chunks = cut < units ? 2 : 1;
    const int bound[3] = {0, cut, units};
    for (int c = 0; c < chunks; ++c) {
        if (n == 1) {
            const int a = bound[c], e = bound[c + 1];
            rc = upload(0, 1, a, std::min(e + 1, h));  // + the band's halo row
            if (rc)
                return rc;
            KC_CUDA(cudaEventRecord(ctx->chunk_ev[c], cs));
            KC_CUDA(cudaStreamWaitEvent(st, ctx->chunk_ev[c], 0));
            rc = to_gray(0, 1, a, std::min(e + 1, h));
            if (rc)
                return rc;
            rc = launch_wide(ctx, dimg + (size_t)a * dpitch, 1, w, e - a, h, a, dpitch, dstride, k,
                             select, d, st, c + 1 < chunks ? 1 : 0);
        } else {
            const int i0 = bound[c], i1 = bound[c + 1];
            rc = upload(i0, i1, 0, h);
            if (rc)
                return rc;
            KC_CUDA(cudaEventRecord(ctx->chunk_ev[c], cs));
            KC_CUDA(cudaStreamWaitEvent(st, ctx->chunk_ev[c], 0));
            rc = to_gray(i0, i1, 0, h);
            if (rc)
                return rc;
            const uint8_t* src = dimg + (size_t)i0 * dstride;
            rc = tile ? launch_tile(ctx, src, i1 - i0, w, h, dpitch, dstride, k, select, sub(i0), st)
                      : launch_wide(ctx, src, i1 - i0, w, h, h, 0, dpitch, dstride, k, select,
                                    sub(i0), st);
        }
        if (rc)
            return rc;
    }
    if (bytes <= (64u << 10)) {
        // one packed copy back, then scatter on the host
        rc = ctx->hout.ensure(bytes);
        if (rc)
            return rc;
        KC_CUDA(cudaMemcpyAsync(ctx->hout.p, b, bytes, cudaMemcpyDeviceToHost, st));
        KC_CUDA(cudaStreamSynchronize(st));
        const char* hb = static_cast<const char*>(ctx->hout.p);
        if (host.sums)
            std::memcpy(host.sums, hb, n256 * 8);
        if (host.cards)
            std::memcpy(host.cards, hb + n256 * 8, n256 * 8);
        if (host.values)
            std::memcpy(host.values, hb + n256 * 16, n256 * 8);
        if (host.defined)
            std::memcpy(host.defined, hb + n256 * 24, n256);
        if (select) {
            const int* ht = reinterpret_cast<const int*>(hb + tail_off);
            if (host.t0s)
                std::memcpy(host.t0s, ht, (size_t)n * 4);
            if (host.topk_counts)
                std::memcpy(host.topk_counts, ht + n, (size_t)n * 4);
            if (host.status)
                std::memcpy(host.status, ht + 2 * n, (size_t)n * 4);
            if (host.topks)
                std::memcpy(host.topks, ht + 3 * n, (size_t)n * k * 4);
        }
        return KOHLER_OK;
    }
    if (host.sums)
        KC_CUDA(cudaMemcpyAsync(host.sums, d.sums, n256 * 8, cudaMemcpyDeviceToHost, st));
    if (host.cards)
        KC_CUDA(cudaMemcpyAsync(host.cards, d.cards, n256 * 8, cudaMemcpyDeviceToHost, st));
    if (host.values)
        KC_CUDA(cudaMemcpyAsync(host.values, d.values, n256 * 8, cudaMemcpyDeviceToHost, st));
    if (host.defined)
        KC_CUDA(cudaMemcpyAsync(host.defined, d.defined, n256, cudaMemcpyDeviceToHost, st));
    if (select) {
        if (host.t0s)
            KC_CUDA(cudaMemcpyAsync(host.t0s, d.t0s, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        if (host.topk_counts)
            KC_CUDA(cudaMemcpyAsync(host.topk_counts, d.topk_counts, (size_t)n * 4,
                                    cudaMemcpyDeviceToHost, st));
        if (host.status)
            KC_CUDA(cudaMemcpyAsync(host.status, d.status, (size_t)n * 4,
                                    cudaMemcpyDeviceToHost, st));
        if (host.topks)
            KC_CUDA(cudaMemcpyAsync(host.topks, d.topks, (size_t)n * k * 4,
                                    cudaMemcpyDeviceToHost, st));
    }
    KC_CUDA(cudaStreamSynchronize(st));
    return KOHLER_OK;
}

// Segmentation host side: map_kernel over n images (one LUT per image).
int launch_map(kohler_cuda_ctx* ctx, const MapParams& mp0, cudaStream_t stream)
{
    MapParams mp = mp0;
    // unit = one warp's rows: about total / (SMs * 32 warps), 4..32 KB, never
    // across images, so enough warps are in flight at any size
    const long long px_per_image = (long long)mp.w * mp.h;
    const long long target = std::min(32768ll, std::max(4096ll, px_per_image * mp.n / (ctx->sm_count * 32ll)));
    mp.units_per_image = (int)std::max(1ll, std::min<long long>(mp.h, (px_per_image + target - 1) / target));
    const uint32_t segs = (uint32_t)(mp.w + 15) / 16;
    mp.seg_magic = (uint32_t)((1ull << 32) / segs + 1);
    const long long units = (long long)mp.units_per_image * mp.n;
    mp.flat = mp.pitch == (size_t)mp.w && mp.out_pitch == (size_t)mp.w && mp.w % 16 == 0 &&
              ((reinterpret_cast<uintptr_t>(mp.px) | reinterpret_cast<uintptr_t>(mp.out) |
                mp.image_stride | mp.out_stride) & 15) == 0;
    dim3 grid((unsigned)((units + kMapWarps - 1) / kMapWarps));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kMapThreads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KC_CUDA(cudaLaunchKernelEx(&cfg, map_kernel, mp));
    ctx->last_launches += 1;
    return KOHLER_OK;
}

int launch_hist(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h, size_t pitch,
                size_t image_stride, uint32_t* hist, cudaStream_t stream)
{
    KC_CUDA(cudaMemsetAsync(hist, 0, (size_t)n * 256 * sizeof(uint32_t), stream));
    const long long px_per_image = (long long)w * h;
    const int bpi = (int)std::max(1ll, std::min<long long>(h, (px_per_image + 65535) / 65536));
    const uint32_t segs = (uint32_t)(w + 15) / 16;
    hist_kernel<<<dim3((unsigned)((long long)bpi * n)), 512, 0, stream>>>(
        px, pitch, image_stride, w, h, bpi, (uint32_t)((1ull << 32) / segs + 1), hist);
    KC_CUDA(cudaGetLastError());
    ctx->last_launches += 1;
    return KOHLER_OK;
}

// classify (mode 0) / quantize (mode 1) of one host image with a given set
int host_classify_quantize(kohler_cuda_ctx* ctx, const uint8_t* px, int w, int h, size_t pitch,
                           const int* ts, int nts, uint8_t* out, int mode)
{
    const size_t dpitch = round_up((size_t)w, 16);
    const size_t bytes = dpitch * (size_t)h;
    int rc = ctx->img.ensure(std::max<size_t>(2 * bytes + 256 * 4 + (size_t)nts * 4 + 64, 64));
    if (rc)
        return rc;
    uint8_t* din = static_cast<uint8_t*>(ctx->img.p);
    uint8_t* dout = din + bytes;
    uint32_t* dhist = reinterpret_cast<uint32_t*>(round_up(reinterpret_cast<uintptr_t>(dout + bytes), 16));
    int* dts = reinterpret_cast<int*>(dhist + 256);
    cudaStream_t st = ctx->stream;
    ctx->last_launches = 0;
    KC_CUDA(cudaMemcpy2DAsync(din, dpitch, px, pitch, (size_t)w, (size_t)h, cudaMemcpyHostToDevice, st));
    if (nts)
        KC_CUDA(cudaMemcpyAsync(dts, ts, (size_t)nts * 4, cudaMemcpyHostToDevice, st));
    if (mode == 1) {
        rc = launch_hist(ctx, din, 1, w, h, dpitch, bytes, dhist, st);
        if (rc)
            return rc;
    }
    MapParams mp{};
    mp.px = din;
    mp.pitch = dpitch;
    mp.image_stride = bytes;
    mp.out = dout;
    mp.out_pitch = dpitch;
    mp.out_stride = bytes;
    mp.n = 1;
    mp.w = w;
    mp.h = h;
    mp.mode = mode;
    mp.thresholds = dts;
    mp.ts_stride = 0;
    mp.ts_count = nts;
    mp.hist = dhist;
    rc = launch_map(ctx, mp, st);
    if (rc)
        return rc;
    KC_CUDA(cudaMemcpy2DAsync(out, (size_t)w, dout, dpitch, (size_t)w, (size_t)h, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    return KOHLER_OK;
}

// curve -> thresholds -> quantize for a device batch (K1 / K5 export the
// pixel histograms, so the map is the only extra pass)
int segment_device(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int h, size_t pitch,
                   size_t image_stride, int k, uint8_t* out, size_t out_pitch, size_t out_stride,
                   int* thresholds, int* ts_counts, int* status, cudaStream_t stream)
{
    if (n == 0)
        return KOHLER_OK;
    const int kk = std::max(k, 1);
    // scratch: hist [n][256] u32, t0 / topk / counts for the mode not returned
    const size_t hist_bytes = (size_t)n * 256 * 4;
    const size_t scr_bytes = (size_t)n * 4 * 2 + (size_t)n * kk * 4;
    int rc = ctx->seg.ensure(hist_bytes + scr_bytes + 64);
    if (rc)
        return rc;
    uint32_t* hist = static_cast<uint32_t*>(ctx->seg.p);
    int* scr = reinterpret_cast<int*>(hist + (size_t)n * 256);
    BatchOut o{};
    if (k == 0) {
        o.t0s = thresholds;
        o.topks = scr + 2 * (size_t)n;
        o.topk_counts = scr;
    } else {
        o.t0s = scr;
        o.topks = thresholds;
        o.topk_counts = ts_counts;
    }
    o.status = status;
    const bool tile = use_tile(n, w, h);
    if (!tile)
        KC_CUDA(cudaMemsetAsync(hist, 0, hist_bytes, stream));
    rc = tile ? launch_tile(ctx, px, n, w, h, pitch, image_stride, kk, 1, o, stream, hist)
              : launch_wide(ctx, px, n, w, h, h, 0, pitch, image_stride, kk, 1, o, stream, 0, hist);
    if (rc)
        return rc;
    MapParams mp{};
    mp.px = px;
    mp.pitch = pitch;
    mp.image_stride = image_stride;
    mp.out = out;
    mp.out_pitch = out_pitch;
    mp.out_stride = out_stride;
    mp.n = n;
    mp.w = w;
    mp.h = h;
    mp.mode = 1;
    mp.thresholds = thresholds;
    mp.ts_stride = kk;
    mp.ts_counts = k == 0 ? nullptr : ts_counts;
    mp.ts_count = 1;
    mp.status = status;
    mp.hist = hist;
    mp.counts_out = k == 0 ? ts_counts : nullptr;  // 1 per frame with a boundary, else 0
    return launch_map(ctx, mp, stream);
}

} // namespace

extern "C" {

int kohler_cuda_abi_version(void) { return 101; }

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
    if (n == 0)
        return KOHLER_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    ctx->last_launches = 0;
    const size_t dp = round_up((size_t)w, 16), ds = dp * (size_t)h;
    rc = ctx->gray.ensure(ds * (size_t)n);
    if (rc)
        return rc;
    uint8_t* dg = static_cast<uint8_t*>(ctx->gray.p);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    rc = launch_luma(ctx, rgb, n, w, h, rgb_pitch, rgb_stride, dg, dp, ds, st);
    if (rc)
        return rc;
    BatchOut o{sums, cards, values, defined, t0s, topks, topk_counts, status};
    const bool select = t0s || topks || topk_counts || status;
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
    int st = 0, t0 = -1;
    const int rc =
        host_select(ctx, nullptr, nullptr, values, defined, n, k, nullptr, nullptr, &t0, out, count, &st);
    if (rc)
        return rc;
    return st ? KOHLER_NO_BOUNDARY : KOHLER_OK;
}

} // extern "C"

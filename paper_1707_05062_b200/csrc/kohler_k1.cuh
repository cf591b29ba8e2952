// kohler_k1.cuh — K1 accumulation (walk_kernel) and K3/K4 finish_kernel.
// Part of the single translation unit kohler_kernels.cu (included there,
// in this order, after the shared constants and parameter blocks).
#pragma once

namespace {

#ifdef KOHLER_CHECKED
using kohler_walk::chk_g;
using kohler_walk::chk_sm;
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
        if (p.sums)
            p.sums[(size_t)img * 256 + tid] = cs;
        if (p.cards)
            p.cards[(size_t)img * 256 + tid] = cc;
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

// K3 + K4 inside K1 for single-image launches, from the image's 512 exact
// combinations in shared memory (sval, at kSmVal; the scratch aliases the
// idle row ring).  Same arithmetic as finish_kernel.  Called by every thread
// of one CTA.  Waits for the previous launch (griddepcontrol.wait) right
// before the first output store only: calls reusing the output buffers stay
// in stream order, everything before the stores overlaps the predecessor.
__device__ void finish_from_vals(const WideParams& p, int img, unsigned char* sm)
{
    const int tid = threadIdx.x;
    long long* sval = reinterpret_cast<long long*>(sm + kSmVal);
    uint64_t* ccard = reinterpret_cast<uint64_t*>(sm + kSmCurve);
    uint64_t* csum = ccard + 256;
    double* mean = reinterpret_cast<double*>(sm + kSmMean);
    uint8_t* def = sm + kSmDef;
    unsigned char* scr = sm + kSmScratch;                           // block_select256: 3136 B
    long long* tmp = reinterpret_cast<long long*>(scr + 3200);      // [256]
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
        const uint64_t cs = csum[tid], cc = ccard[tid];
        mean[tid] = cc ? (double)cs / (double)cc : 0.0;
        def[tid] = cc ? 1 : 0;
    }
    __syncthreads();
    // the selection runs before the wait too, into shared memory (<= 128
    // maxima exist); only the stores follow the previous launch
    int* s_ints = reinterpret_cast<int*>(scr + 5248);  // t0, count, status, -, topk[128]
    if (p.select && tid < 256) {
        const int st = block_select256(mean, def, p.k, scr, 1, s_ints, s_ints + 4, s_ints + 1);
        if (tid == 0)
            s_ints[2] = st;
    }
    __syncthreads();
    pdl_wait();
    if (tid < 256) {
        const uint64_t cs = csum[tid], cc = ccard[tid];
        if (p.sums)
            p.sums[(size_t)img * 256 + tid] = cs;
        if (p.cards)
            p.cards[(size_t)img * 256 + tid] = cc;
        if (p.values)
            p.values[(size_t)img * 256 + tid] = mean[tid];
        if (p.defined)
            p.defined[(size_t)img * 256 + tid] = def[tid];
    }
    if (p.select) {
        const int cnt = s_ints[1];
        if (tid == 0) {
            if (p.t0s)
                p.t0s[img] = s_ints[0];
            if (p.topk_counts)
                p.topk_counts[img] = cnt;
            if (p.status)
                p.status[img] = s_ints[2];
        }
        if (p.topks && tid < cnt)
            p.topks[(size_t)img * p.k + tid] = s_ints[4 + tid];
    }
    __syncthreads();
}

// Ticket variant (self_finish): the CTA whose flush landed last reads the
// image's accumulator copies (summed, reset: self-cleaning), then K3 + K4.
__device__ void finish_in_cta(const WideParams& p, int img, unsigned char* sm)
{
    long long* sval = reinterpret_cast<long long*>(sm + kSmVal);
    for (int r = threadIdx.x; r < 512; r += kWalkThreads) {
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
    if (threadIdx.x == 0)
        p.tickets[img] = 0u;  // self-cleaning for the next call
    __syncthreads();
    finish_from_vals(p, img, sm);
}

// Cluster variant (small single images: the grid is one thread-block
// cluster, <= 8 CTAs): every CTA left its 512 combinations in its own
// shared memory (kSmVal); CTA rank 0 sums them over distributed shared
// memory and finishes.  No global accumulator, no ticket, no dependency on
// the previous launch until the output stores.
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ void finish_cluster(const WideParams& p, int img, unsigned char* sm)
{
    cluster_sync_all();  // every CTA's combinations are in its shared memory
    unsigned rank, nranks;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nranks));
    long long* sval = reinterpret_cast<long long*>(sm + kSmVal);
    if (rank == 0) {
        for (int t = threadIdx.x; t < 512; t += kWalkThreads) {
            const uint32_t la = (uint32_t)__cvta_generic_to_shared(sval + t);
            long long s = sval[t];
            for (unsigned r = 1; r < nranks; ++r) {
                uint32_t ra;
                long long v;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
                asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
                s += v;
            }
            sval[t] = s;
        }
    }
    cluster_sync_all();  // the peers' shared memory stays valid until rank 0 has read it
    if (rank == 0) {
        __syncthreads();
        finish_from_vals(p, img, sm);
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
        KCHK({
            chk_sm(dst + r * kBorderRow + 16 * ci, 16);
            chk_g(src, 16, p.px, p.px + (size_t)(p.n - 1) * p.image_stride + (size_t)p.buf_rows * p.pitch);
        });
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

template <bool RGB>
__device__ __forceinline__ int border_px(const uint8_t* row, int x)
{
    if constexpr (RGB)
        return (int)luma1(row[3 * x], row[3 * x + 1], row[3 * x + 2]);
    else
        return row[x];
}

template <bool RGB>
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
        const int v0 = pre ? pre[o] : border_px<RGB>(base, x);
        const int c = pre ? pre[kBorderRow + o] : border_px<RGB>(rl, x);
        KCYC(1);
        atomicAdd(&corr_tot[v0], 1);
        if (img_last) {
            atomicAdd(&corr_tot[c], -1);
        } else {
            const int d = pre ? pre[2 * kBorderRow + o] : border_px<RGB>(rl + p.pitch, x);
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
template <bool RGB>
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
    border_pass<RGB>(p, img, first ? *reinterpret_cast<const BorderSlice*>(sm + kSmBslice) : border_slice(p, img),
                prefetched ? sm + kSmBorder : nullptr, hb, corr_tot);
    KCYC(5);
    __syncthreads();
    KCYC(6);
    phase(9);
    // the accumulators may still be read / reset by the previous finish_kernel
    // (cluster mode: no shared workspace, the finishing CTA waits before its
    // output stores instead)
    if (!p.cluster)
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
        if (p.cluster) {
            reinterpret_cast<long long*>(sm + kSmVal)[t] = val;
        } else if (val != 0) {
            const int copy = blockIdx.x % p.copies;
            unsigned long long* dst = p.acc + ((size_t)img * p.copies + copy) * 512 + t;
            if (p.acc_sys)  // the group's shared accumulator on the first GPU, over NVLink
                atomicAdd_system(dst, (unsigned long long)val);
            else
                atomicAdd(dst, (unsigned long long)val);
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
#ifdef KOHLER_CHECKED
    const uint8_t* g_lo;  // the input buffer (checked builds)
    const uint8_t* g_hi;
#endif
};

template <bool RGB>
__device__ __forceinline__ LaneGeo lane_geo(const WideParams& p, const uint8_t* base, long long g,
                                            int lane)
{
    using F = K1Fmt<RGB>;
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
#ifdef KOHLER_CHECKED
        L.jcl += p.inject;  // the negative control: one row past the buffer
#endif
    } else {
        L.y0 = 1;  // a valid address (row 0), never used
        L.nrows = 0;
        L.jlo = 0;
        L.jcl = 0;
    }
    L.p = base + ((long long)L.y0 - 1) * (long long)p.pitch + (long long)L.x0 * F::bpp;
    L.pd = lane == 0 ? -16 : (int)F::seg;
    L.pds = lane == 0 ? (int)F::lpad : (int)(F::rpad - F::seg * 31);
    L.pad = ((lane == 0) & (L.x0 > 0)) | ((lane == 31) & (L.e > 15)) ? 1u : 0u;
#ifdef KOHLER_CHECKED
    L.g_lo = p.px;
    L.g_hi = p.px + (size_t)(p.n - 1) * p.image_stride + (size_t)p.buf_rows * p.pitch;
#endif
    return L;
}

// Issue the copies of ring position j of a lane's walk into ring slot `dst`
// (shared address of this lane's 16-byte segment in the slot): the segment,
// from a clamped valid row, and for lane 0 / lane 31 the 16 bytes left /
// right of it where that neighbour exists.  One cp.async group per position.
template <bool RGB>
__device__ __forceinline__ void fetch_row(const LaneGeo& L, int j, uint32_t pitch, uint32_t dst)
{
    // 64-bit row offset (once per segment start: no cost in the walk)
    const uint8_t* src = L.p + (size_t)(uint32_t)min(max(j, L.jlo), L.jcl) * pitch;
    KCHK({
        chk_sm(dst, K1Fmt<RGB>::seg);
        chk_g(src, K1Fmt<RGB>::seg, L.g_lo, L.g_hi);
        if (L.pad) {
            chk_sm(dst + L.pds, 16);
            chk_g(src + L.pd, 16, L.g_lo, L.g_hi);
        }
    });
    if constexpr (RGB) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
            "cp.async.cg.shared.global [%0], [%1], 16;\n\t"
            "cp.async.cg.shared.global [%0+16], [%1+16], 16;\n\t"
            "cp.async.cg.shared.global [%0+32], [%1+32], 16;\n\t"
            "@p cp.async.cg.shared.global [%3], [%4], 16;\n\t"
            "cp.async.commit_group;\n\t}" ::"r"(dst),
            "l"(src), "r"(L.pad), "r"(dst + L.pds), "l"(src + L.pd)
            : "memory");
        return;
    }
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
#ifdef KOHLER_CHECKED
    const uint8_t* g_lo;
    const uint8_t* g_hi;
#endif
};

__device__ __forceinline__ FetchStream fetch_stream(const LaneGeo& L, int j, uint32_t pitch,
                                                    int lane)
{
    FetchStream f;
    const int jj = min(j, L.jcl);  // j >= 3 > jlo
    f.src = L.p + (size_t)(uint32_t)jj * pitch;
    f.left = L.jcl - j;
    f.pl = L.pad && lane == 0;
    f.pr = L.pad && lane == 31;
#ifdef KOHLER_CHECKED
    f.g_lo = L.g_lo;
    f.g_hi = L.g_hi;
#endif
    return f;
}

template <bool RGB>
__device__ __forceinline__ void fetch_next(FetchStream& f, uint32_t pitch, uint32_t dst)
{
    KCHK({
        chk_sm(dst, K1Fmt<RGB>::seg);
        chk_g(f.src, K1Fmt<RGB>::seg, f.g_lo, f.g_hi);
        if (f.pl) {
            chk_sm(dst + (RGB ? 1536u : 512u), 16);
            chk_g(f.src - 16, 16, f.g_lo, f.g_hi);
        }
        if (f.pr) {
            chk_sm(dst + (RGB ? 64u : 32u), 16);
            chk_g(f.src + (RGB ? 48 : 16), 16, f.g_lo, f.g_hi);
        }
    });
    if constexpr (RGB) {
        // segment = 3 chunks; left pad: slot + lpad <- src - 16 (lane 0 at
        // slot + 0); right pad: slot + rpad = lane 31's segment + 64 <- src + 48
        asm volatile(
            "{\n\t.reg .pred pl, pr;\n\tsetp.ne.u32 pl, %2, 0;\n\tsetp.ne.u32 pr, %3, 0;\n\t"
            "cp.async.cg.shared.global [%0], [%1], 16;\n\t"
            "cp.async.cg.shared.global [%0+16], [%1+16], 16;\n\t"
            "cp.async.cg.shared.global [%0+32], [%1+32], 16;\n\t"
            "@pl cp.async.cg.shared.global [%0+1536], [%1+-16], 16;\n\t"
            "@pr cp.async.cg.shared.global [%0+64], [%1+48], 16;\n\t"
            "cp.async.commit_group;\n\t}" ::"r"(dst),
            "l"(f.src), "r"(f.pl), "r"(f.pr)
            : "memory");
        f.src += f.left > 0 ? pitch : 0u;
        --f.left;
        return;
    }
    asm volatile(
        "{\n\t.reg .pred pl, pr;\n\tsetp.ne.u32 pl, %2, 0;\n\tsetp.ne.u32 pr, %3, 0;\n\t"
#ifndef KOHLER_PROBE_NO_ROWLOADS
        "cp.async.cg.shared.global [%0], [%1], 16;\n\t"
#endif
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
    uint32_t pad_off;  // shared offset of this lane's pad byte (RGB: word) from its segment
    uint32_t pad_sh;   // RGB: right shift of the pad word to its pixel's bytes
    bool pad;          // lane reads a pad byte
    bool l_own, l_pad;
    bool r_own, r_pad;
};

template <bool RGB>
__device__ __forceinline__ void read_row_shfl(kohler_walk::Row& r, uint32_t seg, const NbrSel& n)
{
    KCHK({
        chk_sm(seg, RGB ? 48u : 16u);
        if (n.pad)
            chk_sm(seg + n.pad_off, RGB ? 4u : 1u);
    });
    uint32_t pb = 0;
    if constexpr (RGB) {
        // 48 bytes of interleaved RGB -> 16 luma bytes (the reference's luma601);
        // the pad pixel's three bytes are one aligned word (lane 0: bytes 1..3
        // of the left pad's last word; lane 31: bytes 0..2 of the right pad)
        uint32_t c[12];
#pragma unroll
        for (int q = 0; q < 3; ++q)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(c[4 * q]), "=r"(c[4 * q + 1]), "=r"(c[4 * q + 2]), "=r"(c[4 * q + 3])
                         : "r"(seg + 16u * q)
                         : "memory");
        uint32_t pw = 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
                     "@p ld.shared.u32 %0, [%2];\n\t}"
                     : "+r"(pw)
                     : "r"((uint32_t)n.pad), "r"(seg + n.pad_off)
                     : "memory");
#pragma unroll
        for (int j = 0; j < 4; ++j)
            r.w[j] = luma4(c[3 * j], c[3 * j + 1], c[3 * j + 2]);
        pw >>= n.pad_sh;
        pb = luma_div(__dp2a_hi(114u, pw, __dp2a_lo(299u | 587u << 16, pw, 500u)));
    } else {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                     : "r"(seg)
                     : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
                     "@p ld.shared.u8 %0, [%2];\n\t}"
                     : "+r"(pb)
                     : "r"((uint32_t)n.pad), "r"(seg + n.pad_off)
                     : "memory");
    }
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
// prefetched 3 positions ahead (RGB: 2) across segment boundaries.  The W copy
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

template <bool ALIGNED, bool TWO_W, bool RGB, bool CL>
__device__ __forceinline__ void walk_range(const WideParams& p, unsigned char* sm,
                                           unsigned char* hist, uint32_t smbase,
                                           const uint8_t* base, long long ua, long long ub,
                                           bool zero_first)
{
    using namespace kohler_walk;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane4 = (uint32_t)lane * 4u;
    // cluster launches: every .shared::cta address carries the CTA rank in
    // bits 24+ (as cvta returns it); the counter addresses get it from the
    // per-lane byte source of the address PRMT (absorb), so the fixed
    // immediates stay
    const uint32_t rbits = CL ? (smbase & 0xFF000000u) : 0u;
    const uint32_t lane_ra = lane4 | rbits;
    using F = K1Fmt<RGB>;
    constexpr uint32_t HA = F::hist_abs;
    const uint32_t kneg = HA - lane4 - rbits;  // pair event at A_a + A_b + kneg
    const uint32_t dummy = HA + kDummy + lane4 + rbits;
    // corr[v] of a pixel with W address A: corr_base + (A >> 6)
    // (A >> 6 = (rbits >> 6) + 4v + (lane4 >> 6); smbase carries rbits)
    const uint32_t corr_base = smbase + F::shift + kSmCorr - (lane4 >> 6) - (rbits >> 6);
    const int R = p.R;
    const uint32_t pitch = (uint32_t)p.pitch;  // < 2^32 (checked by the host)
    const bool any = ua < ub;
    // this lane's segment in slot 0 of the warp's ring; slot s is + s * kSlotBytes
    const uint32_t ring = (smbase + kSmRing + 127u) & ~127u;
    constexpr int AH = F::ahead;  // positions in flight (ring slots - 1)
    const uint32_t seg0 = ring + (uint32_t)warp * (F::slots * F::slot) + (uint32_t)lane * F::seg;

    // current segment: group g, rows [r0, r1) of its walks; next segment
    long long g = 0;
    int r0 = 0, r1 = 0;
    LaneGeo G{};
    if (any) {
        g = ua / R;
        r0 = (int)(ua - g * R);
        r1 = (int)(ub - g * R < (long long)R ? (int)(ub - g * R) : R);
        G = lane_geo<RGB>(p, base, g, lane);
        // positions 0, 1, 2 of the first segment (rows r0 - 1, r0, r0 + 1 of the walk)
        fetch_row<RGB>(G, r0, pitch, seg0);
        fetch_row<RGB>(G, r0 + 1, pitch, seg0 + F::slot);
        if (AH > 2)
            fetch_row<RGB>(G, r0 + 2, pitch, seg0 + 2 * F::slot);
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
    const uint32_t slot_end = seg0 + F::slots * F::slot;
    uint32_t sl_cur = seg0, sl_prev = seg0 + (F::slots - 1) * F::slot;
    for (;;) {
        const int L = r1 - r0;
        const int P = L + 2;
        FetchStream fs = fetch_stream(G, r0 + AH, pitch, lane);
        const long long gn = g + 1;
        const bool has_next = gn * R < ub;
        const int nr1 = has_next ? (int)(ub - gn * R < (long long)R ? (int)(ub - gn * R) : R) : 0;
        const LaneGeo N = has_next ? lane_geo<RGB>(p, base, gn, lane) : G;
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
        nb.pad_off = RGB ? (lane == 0 ? F::lpad + 12u : F::rpad - F::seg * 31u)
                         : (lane == 0 ? F::lpad + 15u : F::rpad - F::seg * 31u);
        nb.pad_sh = lane == 0 ? 8u : 0u;

        // One ring position j: prefetch position j + 3 (of this segment or,
        // past its end, of the next), absorb row r0 - 1 + j into D and
        // process row r0 - 2 + j (C) against it.
        auto step = [&](Car& D, Car& C, int j, auto kind, auto wc, auto cross) {
            constexpr int KIND = decltype(kind)::value;  // 0 absorb, 1 prime, 2 process
            constexpr bool CROSS = decltype(cross)::value;  // prefetch may cross into the next segment
            constexpr int WC = decltype(wc)::value;
            constexpr uint32_t kOffW = (WC && TWO_W) ? kOffW1 : kOffW0;
            // slot q & 3 was committed 3 groups ago; <= 2 younger groups may pend
            if (AH > 2)
                asm volatile("cp.async.wait_group 2;" ::: "memory");
            else
                asm volatile("cp.async.wait_group 1;" ::: "memory");
#ifndef KOHLER_NO_RING_SYNCWARP
            // all lanes' copies into slot q & 3 are visible, and all lanes have
            // read slot (q - 1) & 3 (the previous position), which is refilled now
            __syncwarp();
#endif
            // read this position's row first: the prefetch issue below
            // covers the LDS latency before the unpack needs the data
            Row r;
            read_row_shfl<RGB>(r, sl_cur, nb);
            const uint32_t pref = sl_prev;
            sl_prev = sl_cur;
            sl_cur = sl_cur + F::slot == slot_end ? seg0 : sl_cur + F::slot;
            if (!CROSS || j + AH < P)
                fetch_next<RGB>(fs, pitch, pref);
            else if (has_next)
                fetch_row<RGB>(N, j + AH - P, pitch, pref);
            else
                asm volatile("cp.async.commit_group;" ::: "memory");
            absorb<ALIGNED>(D, r, lane_ra, G.e);
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
            const uint32_t Arn = __byte_perm(C.rn, lane_ra, 0x7604);
            if (ALIGNED || !F.ragged) {
                if (live) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        red_add_imm<HA + kOffW>(C.A[i], b_of(Be, Bo, i));
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
                    red_add_imm<HA + kOffW>(C.A[i], real ? b_of(Be, Bo, i) : 0u);
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
        if (P > AH + 1) {
            step(X, Y, 0, K0{}, W0{}, NC{});
            step(Y, X, 1, K1{}, W1{}, NC{});
        } else {
            step(X, Y, 0, K0{}, W0{}, CR{});
            step(Y, X, 1, K1{}, W1{}, CR{});
        }
        int j = 2;
        for (; j + AH + 1 < P; j += 2) {
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

template <bool ALIGNED, bool TWO_W, bool RGB, bool CL = false>
__global__ void __launch_bounds__(kWalkThreads, 1) walk_kernel(const __grid_constant__ WideParams p)
{
    using F = K1Fmt<RGB>;
    extern __shared__ __align__(16) unsigned char sm_dyn[];
    // Shared address of the dynamic block.  In a cluster launch it carries the
    // CTA rank in bits 24+ (measured: rank r -> (r << 24) | 0x400, for
    // cvta.to.shared and cvta.to.shared::cta alike), and every .shared::cta
    // access must too (walk_range adds the rank bits to the counter
    // addresses); smloc is the offset inside the CTA's window.
    const uint32_t smbase = (uint32_t)__cvta_generic_to_shared(sm_dyn);
    const uint32_t smloc = smbase & 0x00FFFFFFu;
    if (smloc + F::shift + kSmMiscEnd > F::hist_abs ||
        F::hist_abs + kohler_walk::kHistBytes > smloc + F::smem)
        __trap();  // the fixed counter address would overlap the scratch (never seen)
    unsigned char* hist = sm_dyn + (F::hist_abs - smloc);
    // the scratch block (all kSm* offsets below), above the ring
    unsigned char* sm = sm_dyn + F::shift;
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
        // (RGB: the border pass reads its rows from global memory)
        const bool prefetched = !RGB && bs.xb - bs.xa <= kBorderPx;
        if (prefetched)
            border_prefetch(p, i_first, bs, smbase + F::shift + kSmBorder);
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
                walk_range<ALIGNED, TWO_W, RGB, CL>(p, sm, hist, smbase, base, wa, wb, !zeroed);
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
            flush_image<RGB>(ps, img, sm, hist, img < i_last, TWO_W, prefetched && img == i_first, img == i_first);
            // (the last image: no re-zeroing)
            flushed = true;
            if (CL) {
                finish_cluster(ps, img, sm);
            } else if (ps.self_finish) {
                // ticket: the CTA whose REDGs land last finishes the image
                __threadfence();
                __syncthreads();
                int* flag = reinterpret_cast<int*>(sm + kSmFlag);
                if (tid == 0)
                    *flag = atomicAdd(ps.tickets + img, 1u) == gridDim.x - 1u;
                __syncthreads();
                if (*flag) {
                    __threadfence();
                    finish_in_cta(ps, img, sm);
                }
            }
        }
    }
    if (!flushed)
        pdl_trigger();
    phase(7);
}

} // namespace

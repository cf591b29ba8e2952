// kohler_launch.cuh — host-side launchers (grid / parameter choice, chunked
// host path, segmentation drivers) used by the C ABI in kohler_kernels.cu.
// Part of the single translation unit kohler_kernels.cu.
#pragma once

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

// K1 over RGB directly (no grey image): whole 16-pixel segments, 16-byte
// aligned rows and images, and an image large enough for K1 (small images
// go through luma_kernel + K5)
bool use_tile(int n, int w, int h);
bool rgb_fused_ok(const kohler_cuda_ctx* ctx, const uint8_t* rgb, int n, int w, int h, size_t pitch,
                  size_t stride)
{
    return ctx->rgb_fused && w % 16 == 0 && reinterpret_cast<uintptr_t>(rgb) % 16 == 0 &&
           pitch % 16 == 0 && pitch < (1ull << 32) && (n == 1 || stride % 16 == 0) &&
           !use_tile(n, w, h);
}

// Device output arrays are written (and the curves of the selection kernels
// read) with vector accesses: sums / cards / values 16-byte, defined 8-byte,
// the int arrays 4-byte aligned.  A misaligned pointer would raise a sticky
// cudaErrorMisalignedAddress, so it is refused up front.
int check_out_align(const void* sums, const void* cards, const void* values, const void* defined,
                    const void* t0s, const void* topks, const void* counts, const void* status)
{
    auto mis = [](const void* p, uintptr_t a) { return p && reinterpret_cast<uintptr_t>(p) % a; };
    if (mis(sums, 16) || mis(cards, 16) || mis(values, 16))
        return fail(KOHLER_INVALID_ARGUMENT,
                    "device sums / cards / values must be 16-byte aligned");
    if (mis(defined, 8))
        return fail(KOHLER_INVALID_ARGUMENT, "device defined array must be 8-byte aligned");
    if (mis(t0s, 4) || mis(topks, 4) || mis(counts, 4) || mis(status, 4))
        return fail(KOHLER_INVALID_ARGUMENT, "device int outputs must be 4-byte aligned");
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
constexpr long long kClusterMax = 8;     // portable cluster size
constexpr long long kSelfFinishMax = 24;

int launch_wide(kohler_cuda_ctx* ctx, const uint8_t* px, int n, int w, int band_rows,
                int h_total, int r0, size_t pitch, size_t image_stride, int k, int select,
                const BatchOut& o, cudaStream_t stream, int no_finish = 0,
                uint32_t* hist_out = nullptr, bool rgb = false,
                unsigned long long* acc_ext = nullptr)
{
    // acc_ext (device groups, peer mode; one image, no_finish): the flush adds
    // into this accumulator -- [kAccCopiesSingle][512] on the group's first
    // GPU, reached over NVLink -- instead of the context's own
    if (n == 0)
        return KOHLER_OK;
    // rgb: px is interleaved RGB (3 bytes per pixel) and K1 computes the
    // luma itself; the caller guarantees rgb_fused_ok()
    // the walk advances its row pointers by a 32-bit pitch (row offsets
    // themselves are 64-bit): any row below 4 GiB
    if (pitch >= (1ull << 32))
        return fail(KOHLER_INVALID_ARGUMENT, "row pitch must be below 2^32 bytes");
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
        // up to 144 rows per walk (128 measured against 64: C2 +1.3 %, C4 +2.6 %,
        // C3 +0.4 %; the prime positions per walk amortise over more rows.  144
        // lets C2's 3456 rows split into 24 x 144 with 243 full groups and C3's
        // 1080 into 8 x 135 with 30: C2 +0.3 %, C3 +0.5 % over a cap of 128)
        for (long long r = 16; r <= kMaxWalkRows; ++r) {
            const long long ch = (band_rows + r - 1) / r;
            // idle lanes of the image's last 32-walk group count like wasted rows
            // (C3: 1080 rows x 120 segments -> R = 90 fills 45 groups exactly;
            // R = 120 leaves 24 of the 34th group's lanes idle, 2.2 %)
            const long long tasks = ch * nseg, lanes = (tasks + 31) / 32 * 32;
            const double waste = (double)(ch * r - band_rows) / band_rows + 0.5 / r +
                                 (double)(lanes - tasks) / (double)tasks;
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
    p.acc = acc_ext ? acc_ext : static_cast<unsigned long long*>(ctx->acc.p);
    p.acc_sys = acc_ext ? 1 : 0;
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
    // One image per launch: small grids (<= 8 CTAs) run as ONE thread-block
    // cluster whose rank-0 CTA sums the CTAs' combinations over distributed
    // shared memory and finishes (no global accumulator, so consecutive
    // launches share no workspace and overlap freely, stream order kept by the
    // griddepcontrol.wait before the output stores); mid-size grids let the
    // CTA whose flush lands last finish (ticket); larger ones keep
    // finish_kernel, which runs on the SM the pipelined K1s leave free.
    const bool single = n == 1 && !no_finish;
    // (two W copies: the cluster kernels are instantiated for that layout only)
    p.cluster = (single && G <= kClusterMax && !ctx->no_cluster && !rgb && two_w) ? 1 : 0;
    if (p.cluster && ctx->cluster_ok < 0) {
        // can a cluster of kClusterMax K1 CTAs (one SM each, 194 KiB) be
        // co-scheduled at all on this device / partition?  If not, the ticket
        // form runs instead (same results).
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        cudaLaunchConfig_t oc = {};
        oc.gridDim = dim3((unsigned)kClusterMax);
        oc.blockDim = dim3(kWalkThreads);
        oc.dynamicSmemBytes = kSmWideBytes;
        cudaLaunchAttribute ca[1];
        ca[0].id = cudaLaunchAttributeClusterDimension;
        ca[0].val.clusterDim.x = (unsigned)kClusterMax;
        ca[0].val.clusterDim.y = 1;
        ca[0].val.clusterDim.z = 1;
        oc.attrs = ca;
        oc.numAttrs = 1;
        int nclusters = 0;
        const cudaError_t oe =
            cudaOccupancyMaxActiveClusters(&nclusters, walk_kernel<true, true, false, true>, &oc);
        ctx->cluster_ok = (oe == cudaSuccess && nclusters > 0) ? 1 : 0;
        if (oe != cudaSuccess)
            (void)cudaGetLastError();  // not sticky; clear it
    }
    if (ctx->cluster_ok == 0)
        p.cluster = 0;
    p.self_finish = (single && !p.cluster && G <= kSelfFinishMax) ? 1 : 0;
    if (p.cluster)
        p.early_trigger = 1;

    p.hist_out = hist_out;
#ifdef KOHLER_CHECKED
    p.inject = ctx->inject ? 1 : 0;
#endif
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
    if (rgb && (!vec || w % 16 != 0 || hist_out))
        return fail(KOHLER_INVALID_ARGUMENT, "K1 over RGB needs 16-byte aligned rows of whole segments");
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
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, true, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<false, true, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, false, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<false, false, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytesRgb));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytesRgb));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<true, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        KC_CUDA(cudaFuncSetAttribute(walk_kernel<false, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmWideBytes));
        ctx->wide_attr_set = true;
    }
    ctx->last_grid = (int)G;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kWalkThreads);
    cfg.dynamicSmemBytes = rgb ? kSmWideBytesRgb : kSmWideBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)G;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.cluster ? 2 : 1;
    if (p.cluster)
        KC_CUDA(w % 16 == 0 ? cudaLaunchKernelEx(&cfg, walk_kernel<true, true, false, true>, p)
                            : cudaLaunchKernelEx(&cfg, walk_kernel<false, true, false, true>, p));
    else if (rgb)
        KC_CUDA(two_w ? cudaLaunchKernelEx(&cfg, walk_kernel<true, true, true>, p)
                      : cudaLaunchKernelEx(&cfg, walk_kernel<true, false, true>, p));
    else if (w % 16 == 0)
        KC_CUDA(two_w ? cudaLaunchKernelEx(&cfg, walk_kernel<true, true, false>, p)
                      : cudaLaunchKernelEx(&cfg, walk_kernel<true, false, false>, p));
    else
        KC_CUDA(two_w ? cudaLaunchKernelEx(&cfg, walk_kernel<false, true, false>, p)
                      : cudaLaunchKernelEx(&cfg, walk_kernel<false, false, false>, p));
    ctx->last_launches += 1;
    if (!no_finish && !p.self_finish && !p.cluster) {
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
        // persistent: every warp strides over the curves (kohler_select.cuh)
        if (!ctx->select256_attr_set) {
            KC_CUDA(cudaFuncSetAttribute(select256_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSel256Smem));
            KC_CUDA(cudaFuncSetAttribute(select256_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared));
            ctx->select256_attr_set = true;
        }
        const long long ctas = std::min<long long>((sp.n_curves + kSel256Warps - 1) / kSel256Warps,
                                                   (long long)ctx->sm_count * kSel256CtasPerSm);
        KC_CUDA(launch_pdl(select256_kernel, (unsigned)ctas, 32 * kSel256Warps, kSel256Smem, stream, sp));
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
// events per round with two W copies; LG = 4 keeps one W copy, so R <= 31
// there: 16 * 31 * 16 <= 8191).  Returns false when no LG fits (K1 is used
// instead).
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
        if (r > (cand == 4 ? 31 : 62))
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
    if (!tp.sums || !tp.cards) {
        // K5 writes both curves (the selection reads them): a missing one
        // goes to the workspace
        int rc = ctx->curves.ensure((size_t)n * 512 * sizeof(uint64_t));
        if (rc)
            return rc;
        uint64_t* ws = static_cast<uint64_t*>(ctx->curves.p);
        if (!tp.sums)
            tp.sums = ws;
        if (!tp.cards)
            tp.cards = ws + (size_t)n * 256;
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
    // RGB on the 16-pixel grid: K1 walks the uploaded RGB rows itself
    const bool fused = channels == 3 && rgb_fused_ok(ctx, dup, n, w, h, upitch, ustride);
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    // device outputs, packed: sums | cards | values | defined | t0 | count | status | topk
    const size_t n256 = (size_t)n * 256;
    const size_t tail_off = round_up(n256 * 25, 16);
    const size_t bytes = tail_off + (size_t)n * 4 * 3 + (size_t)n * k * 4;
    // small results (<= 64 KiB): the kernels write them straight into the
    // pinned host staging block (mapped, unified addressing), so no separate
    // device-to-host copy sits at the end of the call
    const bool small = bytes <= (64u << 10);
    rc = small ? ctx->hout.ensure(bytes + 64) : ctx->out.ensure(bytes + 64);
    if (rc)
        return rc;
    char* b = static_cast<char*>(small ? ctx->hout.p : ctx->out.p);
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
        if (channels == 1 || fused)
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
            // + the band's halo row; a later chunk starts one row down (its
            // first row is the previous chunk's halo, which that chunk's
            // kernels may still be reading: never rewrite it)
            const int a_up = c ? a + 1 : a;
            rc = a_up < std::min(e + 1, h) ? upload(0, 1, a_up, std::min(e + 1, h)) : KOHLER_OK;
            if (rc)
                return rc;
            KC_CUDA(cudaEventRecord(ctx->chunk_ev[c], cs));
            KC_CUDA(cudaStreamWaitEvent(st, ctx->chunk_ev[c], 0));
            rc = a_up < std::min(e + 1, h) ? to_gray(0, 1, a_up, std::min(e + 1, h)) : KOHLER_OK;
            if (rc)
                return rc;
            rc = fused ? launch_wide(ctx, dup + (size_t)a * upitch, 1, w, e - a, h, a, upitch, ustride,
                                     k, select, d, st, c + 1 < chunks ? 1 : 0, nullptr, true)
                       : launch_wide(ctx, dimg + (size_t)a * dpitch, 1, w, e - a, h, a, dpitch,
                                     dstride, k, select, d, st, c + 1 < chunks ? 1 : 0);
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
            if (fused)
                rc = launch_wide(ctx, dup + (size_t)i0 * ustride, i1 - i0, w, h, h, 0, upitch, ustride,
                                 k, select, sub(i0), st, 0, nullptr, true);
            else
                rc = tile ? launch_tile(ctx, src, i1 - i0, w, h, dpitch, dstride, k, select, sub(i0), st)
                      : launch_wide(ctx, src, i1 - i0, w, h, h, 0, dpitch, dstride, k, select,
                                    sub(i0), st);
        }
        if (rc)
            return rc;
    }
    if (small) {
        // the results are already in the pinned block: wait, then scatter
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

// kohler_segment.cuh — segmentation kernels (hist_kernel, map_kernel: classify / quantize).
// Part of the single translation unit kohler_kernels.cu (included there,
// in this order, after the shared constants and parameter blocks).
#pragma once

namespace {

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

} // namespace

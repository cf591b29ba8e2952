// kohler_select.cuh — direct_kernel and the selection kernels (K4 on given curves).
// Part of the single translation unit kohler_kernels.cu (included there,
// in this order, after the shared constants and parameter blocks).
#pragma once

namespace {

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

// Standalone selection for 256-level curves: one warp per curve, lane L
// holding thresholds 8L..8L+7 in registers, the register-resident selection
// of kohler_walk.cuh.  Persistent: 4 CTAs of 10 warps per SM, every warp
// strides over the curves and, for (sum, card) input, keeps the NEXT curve's
// 4 KiB in flight (cp.async into its own shared buffer, issued right after
// the current curve moved from the buffer into registers), so no warp waits
// on HBM between curves: on C5 the one-curve-per-warp form spent 7 of 12
// warp-cycles per issue on the loads' scoreboard at 3.0 TB/s
// (profiles/r02h).  Buffer layout: 16-byte chunk g of [sums | cards] at slot
// g ^ ((g >> 3) & 3), which makes the lanes' LDS.128 of chunks 4L + q
// conflict free.
constexpr int kSel256Warps = 10;   // 55 KiB of shared memory per CTA, 4 CTAs = 40 warps per SM
constexpr int kSel256CtasPerSm = 4;
constexpr uint32_t kSel256Buf = 4096;  // per warp: sums[256] | cards[256]
constexpr uint32_t kSel256PerWarp = kSel256Buf + 128 * 8 + 128 * 4;
constexpr uint32_t kSel256Smem = kSel256Warps * kSel256PerWarp;

__device__ __forceinline__ uint32_t sel256_slot(uint32_t g)
{
    return ((g & 127u) ^ ((g >> 3) & 3u)) | (g & 128u);  // sums: chunks 0..127, cards: 128..255
}

__global__ void __launch_bounds__(32 * kSel256Warps, kSel256CtasPerSm)
select256_kernel(const SelectParams p)
{
    // dynamic (kSel256Smem > 48 KiB): per warp the curve buffer, then the maxima keys and thresholds
    extern __shared__ __align__(16) unsigned char sel_sm[];
    unsigned char* const wsm = sel_sm + (threadIdx.x >> 5) * kSel256PerWarp;
    unsigned char* const sbuf_w = wsm;
    unsigned long long* const smv_w = reinterpret_cast<unsigned long long*>(wsm + kSel256Buf);
    int* const smt_w = reinterpret_cast<int*>(wsm + kSel256Buf + 128 * 8);
    // the next launch may start at once: every kernel that reads this one's
    // outputs executes griddepcontrol.wait before it does
    pdl_trigger();
    pdl_wait();  // curves may come from the preceding (PDL-overlapped) launch
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const long long stride = (long long)gridDim.x * kSel256Warps;
    long long cidx = (long long)blockIdx.x * kSel256Warps + wq;
    const uint32_t buf = (uint32_t)__cvta_generic_to_shared(sbuf_w);
    const bool staged = p.sums != nullptr;
    // copy curve c's sums and cards (2 x 128 chunks of 16 bytes) into the buffer
    auto prefetch = [&](long long c) {
        if (c < p.n_curves) {
            const unsigned char* gs = reinterpret_cast<const unsigned char*>(p.sums + (size_t)c * 256);
            const unsigned char* gc = reinterpret_cast<const unsigned char*>(p.cards + (size_t)c * 256);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t g = (uint32_t)lane + 32u * i;
                KCHK({
                    kohler_walk::chk_sm(buf + 16u * sel256_slot(g), 16);
                    kohler_walk::chk_sm(buf + 16u * sel256_slot(g + 128u), 16);
                    kohler_walk::chk_g(gs + 16u * g, 16, reinterpret_cast<const uint8_t*>(p.sums),
                                       reinterpret_cast<const uint8_t*>(p.sums + (size_t)p.n_curves * 256));
                    kohler_walk::chk_g(gc + 16u * g, 16, reinterpret_cast<const uint8_t*>(p.cards),
                                       reinterpret_cast<const uint8_t*>(p.cards + (size_t)p.n_curves * 256));
                });
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(buf + 16u * sel256_slot(g)),
                             "l"(gs + 16u * g)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(buf + 16u * sel256_slot(g + 128u)),
                             "l"(gc + 16u * g)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (staged)
        prefetch(cidx);
    for (; cidx < p.n_curves; cidx += stride) {
        const size_t off = (size_t)cidx * 256 + 8 * lane;
        double v[8];
        bool d[8];
        if (staged) {
            uint64_t s[8], c[8];
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                KCHK({
                    kohler_walk::chk_sm(buf + 16u * sel256_slot(4u * lane + q), 16);
                    kohler_walk::chk_sm(buf + 16u * sel256_slot(4u * lane + q + 128u), 16);
                });
                const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(
                    sbuf_w + 16u * sel256_slot(4u * lane + q));
                const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(
                    sbuf_w + 16u * sel256_slot(4u * lane + q + 128u));
                s[2 * q] = a.x;
                s[2 * q + 1] = a.y;
                c[2 * q] = b.x;
                c[2 * q + 1] = b.y;
            }
            __syncwarp();  // every lane has read the buffer: refill it
            prefetch(cidx + stride);
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
            continue;
        const int st = kohler_walk::warp_select256_regs(
            v, d, p.k, smv_w, smt_w, p.t0s ? p.t0s + cidx : nullptr,
            p.topks ? p.topks + (size_t)cidx * p.k : nullptr, p.topk_counts ? p.topk_counts + cidx : nullptr);
        if (lane == 0 && p.status)
            p.status[cidx] = st;
        __syncwarp();  // the maxima scratch is reused by the next curve
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

} // namespace

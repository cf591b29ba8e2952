// kohler_device.cuh — device helpers shared by the sm_100a kernels:
// the int64 prefix scans that rebuild a curve from its 512 combinations
// (card first differences, sum second differences; DESIGN.md §2 and the
// derivation in kohler_walk.cuh) and the K4 selection (mean contrast,
// optimal threshold, top-k local maxima; proj/src/threshold.cpp:9-82)
// used by finish_kernel, K5's flush and the select kernels.  The
// accumulation itself lives in kohler_walk.cuh / kohler_k1.cuh / kohler_k5.cuh.
#pragma once

#include <cstdint>

namespace kohler_dev {

// ---- exact reconstruction ------------------------------------------------

// Inclusive prefix over 256 int64 values by one warp (lane owns 8 entries).
__device__ __forceinline__ void warp_prefix256(const long long* in, long long* out)
{
    const int lane = threadIdx.x & 31;
    long long a[8];
    long long run = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        run += in[lane * 8 + j];
        a[j] = run;
    }
    long long x = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long yv = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off)
            x += yv;
    }
    const long long excl = x - run;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        out[lane * 8 + j] = a[j] + excl;
}

// Count and sum of one curve from its 512 combinations, by one warp, lane
// owning thresholds [8*lane, 8*lane+8): card = prefix(cd), sum =
// prefix(prefix(h2)); cd(t) / h2(u) are functors.  Each lane's 8 (card, sum)
// are returned in registers.
template <class CD, class H2>
__device__ __forceinline__ void warp_curve256_regs(CD cd, H2 h2, uint64_t (&card)[8],
                                                   uint64_t (&sum)[8])
{
    const int lane = threadIdx.x & 31;
    long long a[8], g[8];
    long long ra = 0, rg = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        ra += cd(lane * 8 + j);
        a[j] = ra;
        rg += h2(lane * 8 + j);
        g[j] = rg;
    }
    long long xa = ra, xg = rg;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long ya = __shfl_up_sync(0xFFFFFFFFu, xa, off);
        const long long yg = __shfl_up_sync(0xFFFFFFFFu, xg, off);
        if (lane >= off) {
            xa += ya;
            xg += yg;
        }
    }
    const long long ea = xa - ra, eg = xg - rg;
    long long rs = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        card[j] = (uint64_t)(a[j] + ea);
        rs += g[j] + eg;
        g[j] = rs;
    }
    long long xs = rs;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long ys = __shfl_up_sync(0xFFFFFFFFu, xs, off);
        if (lane >= off)
            xs += ys;
    }
    const long long es = xs - rs;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        sum[j] = (uint64_t)(g[j] + es);
}

// ---- selection (K4): mean contrast, optimal threshold, top-k maxima ------

struct SelectScratch {
    double* rv;  // run values      [n]
    int* rt;     // run first t     [n]
    double* mv;  // maxima values   [n]
    int* mt;     // maxima t        [n]
};

__device__ __forceinline__ unsigned lanemask_lt()
{
    return (1u << (threadIdx.x & 31)) - 1u;
}

// One warp selects on a curve held in shared (or global) memory.
// Restates proj/src/threshold.cpp:25-82 exactly (for non-NaN values):
// optimal_threshold = argmax with ties to the smallest t; top_k_local_maxima
// collapses equal-valued runs of the defined subsequence to their first t,
// keeps runs strictly above both neighbouring runs (one-sided at the ends),
// ranks by (value desc, t asc), keeps k, outputs ascending.
// Returns 1 (no boundary) when nothing is defined, else 0.
__device__ int warp_select(const double* val, const uint8_t* def, int n, int k,
                           const SelectScratch& s, int* out_t0, int* out_topk, int* out_count)
{
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();

    double bv = 0.0;
    int bt = -1;
    for (int t = lane; t < n; t += 32) {
        if (def[t]) {
            const double v = val[t];
            if (bt < 0 || v > bv) {
                bv = v;
                bt = t;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, off);
        const int ot = __shfl_xor_sync(0xFFFFFFFFu, bt, off);
        if (ot >= 0 && (bt < 0 || ov > bv || (ov == bv && ot < bt))) {
            bv = ov;
            bt = ot;
        }
    }

    bool carry_has = false;
    double carry_v = 0.0;
    int nr = 0;
    for (int c0 = 0; c0 < n; c0 += 32) {
        const int t = c0 + lane;
        const bool d = t < n && def[t];
        const double v = d ? val[t] : 0.0;
        const unsigned dm = __ballot_sync(0xFFFFFFFFu, d);
        const unsigned before = dm & lt;
        const int src = before ? 31 - __clz(before) : lane;
        const double pv_lane = __shfl_sync(0xFFFFFFFFu, v, src);
        const bool has_prev = before != 0 || carry_has;
        const double pv = before ? pv_lane : carry_v;
        const bool start = d && (!has_prev || v != pv);
        const unsigned sm = __ballot_sync(0xFFFFFFFFu, start);
        if (start) {
            const int pos = nr + __popc(sm & lt);
            s.rv[pos] = v;
            s.rt[pos] = t;
        }
        nr += __popc(sm);
        if (dm) {
            carry_v = __shfl_sync(0xFFFFFFFFu, v, 31 - __clz(dm));
            carry_has = true;
        }
    }
    __syncwarp();
    if (nr == 0) {
        if (lane == 0) {
            if (out_t0)
                *out_t0 = -1;
            if (out_count)
                *out_count = 0;
        }
        return 1;
    }

    int nm = 0;
    for (int r0 = 0; r0 < nr; r0 += 32) {
        const int r = r0 + lane;
        bool m = false;
        double v = 0.0;
        int t = 0;
        if (r < nr) {
            v = s.rv[r];
            t = s.rt[r];
            m = (r == 0 || v > s.rv[r - 1]) && (r == nr - 1 || v > s.rv[r + 1]);
        }
        const unsigned mm = __ballot_sync(0xFFFFFFFFu, m);
        if (m) {
            const int pos = nm + __popc(mm & lt);
            s.mv[pos] = v;
            s.mt[pos] = t;
        }
        nm += __popc(mm);
    }
    __syncwarp();

    // Top-k by k rounds of a warp argmax over the unselected maxima
    // (value desc, t asc), then emit the selected ones in t order (the maxima
    // array is already sorted by t).  Lane L owns maxima L, L+32, ... and
    // tracks them in a 64-bit mask (nm <= n/2+1 <= 2049 for n <= 4096).
    unsigned long long selmask = 0ull;
    const int rounds = k < nm ? k : nm;
    if (rounds == nm) {
        selmask = ~0ull;
    } else {
        for (int r = 0; r < rounds; ++r) {
            double lv = 0.0;
            int lbt = -1, lj = -1;
            for (int j = 0, i = lane; i < nm; ++j, i += 32) {
                if ((selmask >> j) & 1ull)
                    continue;
                const double v = s.mv[i];
                const int t = s.mt[i];
                if (lbt < 0 || v > lv || (v == lv && t < lbt)) {
                    lv = v;
                    lbt = t;
                    lj = j;
                }
            }
            double bvv = lv;
            int btt = lbt, bl = lane;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xFFFFFFFFu, bvv, off);
                const int ot = __shfl_xor_sync(0xFFFFFFFFu, btt, off);
                const int ol = __shfl_xor_sync(0xFFFFFFFFu, bl, off);
                if (ot >= 0 && (btt < 0 || ov > bvv || (ov == bvv && ot < btt))) {
                    bvv = ov;
                    btt = ot;
                    bl = ol;
                }
            }
            if (lane == bl && lj >= 0)
                selmask |= 1ull << lj;
        }
    }
    int cnt = 0;
    for (int j = 0, i0 = 0; i0 < nm; ++j, i0 += 32) {
        const int i = i0 + lane;
        const bool sel = i < nm && ((selmask >> j) & 1ull);
        const unsigned sb = __ballot_sync(0xFFFFFFFFu, sel);
        if (sel && out_topk)
            out_topk[cnt + __popc(sb & lt)] = s.mt[i];
        cnt += __popc(sb);
    }
    if (lane == 0) {
        if (out_t0)
            *out_t0 = bt;
        if (out_count)
            *out_count = cnt;
    }
    return 0;
}

// Block-parallel selection for 256-level curves: 256 threads, thread t owns
// threshold t.  Same rules as warp_select (proj/src/threshold.cpp:25-82), but
// every step is a block-wide scan/reduction instead of one warp's serial loop,
// which keeps the per-image tail short.  `val`/`def` are in shared memory;
// `scr` needs 256*(8+4) + 64 bytes.  Must be called by all 256 threads of a
// group of 8 warps that can barrier with bar.sync `bar_id` (256 threads).
// Returns (to every thread) 1 for no boundary, else 0.
__device__ __forceinline__ void bar256(int id)
{
    asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}

__device__ int block_select256(const double* val, const uint8_t* def, int k, unsigned char* scr,
                               int bar_id, int* out_t0, int* out_topk, int* out_count)
{
    const int t = threadIdx.x & 255;
    const int lane = t & 31, wp = t >> 5;
    const unsigned lt = lanemask_lt();
    double* mv = reinterpret_cast<double*>(scr);             // [256] maxima values
    int* mt = reinterpret_cast<int*>(scr + 2048);            // [256] maxima t
    int* wsum = reinterpret_cast<int*>(scr + 3072);          // [8]
    int* wmax = wsum + 8;                                    // [8]
    int* wmin = wmax + 8;                                    // [8]
    double* wbv = reinterpret_cast<double*>(scr + 3072 + 96); // [8]
    int* wbt = reinterpret_cast<int*>(scr + 3072 + 160);     // [8]

    const bool d = def[t] != 0;
    const double v = val[t];

    // argmax with ties to the smallest t
    double bv = v;
    int bt = d ? t : -1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, off);
        const int ot = __shfl_xor_sync(0xFFFFFFFFu, bt, off);
        if (ot >= 0 && (bt < 0 || ov > bv || (ov == bv && ot < bt))) {
            bv = ov;
            bt = ot;
        }
    }
    // previous defined index (max-scan of d ? t : -1), inclusive then shift
    int pd = d ? t : -1;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xFFFFFFFFu, pd, off);
        if (lane >= off && o > pd)
            pd = o;
    }
    if (lane == 31) {
        wmax[wp] = pd;
        wbv[wp] = bv;
        wbt[wp] = bt;
    }
    bar256(bar_id);
    int carry = -1;
    for (int i = 0; i < wp; ++i)
        carry = wmax[i] > carry ? wmax[i] : carry;
    const int pd_incl = pd > carry ? pd : carry;
    int prev = __shfl_up_sync(0xFFFFFFFFu, pd_incl, 1);
    if (lane == 0)
        prev = carry;
    // prev = last defined index < t (or -1)
    const bool start = d && (prev < 0 || val[prev] != v);
    // next run start after t: suffix min-scan of (start ? t : 256)
    int ns = start ? t : 256;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_down_sync(0xFFFFFFFFu, ns, off);
        if (lane + off < 32 && o < ns)
            ns = o;
    }
    if (lane == 0)
        wmin[wp] = ns;
    // block argmax result
    double gbv = 0.0;
    int gbt = -1;
    for (int i = 0; i < 8; ++i) {
        const double ov = wbv[i];
        const int ot = wbt[i];
        if (ot >= 0 && (gbt < 0 || ov > gbv || (ov == gbv && ot < gbt))) {
            gbv = ov;
            gbt = ot;
        }
    }
    bar256(bar_id);
    int carry_n = 256;
    for (int i = wp + 1; i < 8; ++i)
        carry_n = wmin[i] < carry_n ? wmin[i] : carry_n;
    const int ns_incl = ns < carry_n ? ns : carry_n;
    int nxt = __shfl_down_sync(0xFFFFFFFFu, ns_incl, 1);
    if (lane == 31)
        nxt = carry_n;
    // nxt = first run start > t (or 256)
    const bool is_max = start && (prev < 0 || v > val[prev]) && (nxt >= 256 || v > val[nxt]);
    // any run at all? (a defined entry exists iff the argmax exists)
    const bool any = gbt >= 0;

    // compact maxima in t order
    const unsigned mb = __ballot_sync(0xFFFFFFFFu, is_max);
    if (lane == 0)
        wsum[wp] = __popc(mb);
    bar256(bar_id);
    int base = 0, nm = 0;
    for (int i = 0; i < 8; ++i) {
        base += i < wp ? wsum[i] : 0;
        nm += wsum[i];
    }
    const int pos = base + __popc(mb & lt);
    if (is_max) {
        mv[pos] = v;
        mt[pos] = t;
    }
    bar256(bar_id);
    // rank by (value desc, t asc); keep rank < k
    bool sel = false;
    if (is_max) {
        if (k >= nm) {
            sel = true;
        } else {
            // independent loads, 8 per trip (mv/mt are padded to 256)
            int rank = 0;
            for (int j0 = 0; j0 < nm && rank < k; j0 += 8) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int j = j0 + q;
                    const double u = mv[j];
                    rank += (j < nm) && ((u > v) || (u == v && mt[j] < t));
                }
            }
            sel = rank < k;
        }
    }
    const unsigned sb = __ballot_sync(0xFFFFFFFFu, sel);
    if (lane == 0)
        wsum[8 + wp] = __popc(sb);  // wmax area is free now
    bar256(bar_id);
    int sbase = 0, cnt = 0;
    for (int i = 0; i < 8; ++i) {
        sbase += i < wp ? wsum[8 + i] : 0;
        cnt += wsum[8 + i];
    }
    if (sel && out_topk)
        out_topk[sbase + __popc(sb & lt)] = t;
    if (t == 0) {
        if (out_t0)
            *out_t0 = any ? gbt : -1;
        if (out_count)
            *out_count = any ? cnt : 0;
    }
    return any ? 0 : 1;
}

} // namespace kohler_dev

// kohler_device.cuh — device building blocks of the sm_100a Köhler path.
//
// Accumulation ("K1").  Every unordered 4-neighbour pair (a,b)
// with lo = min, hi = max, s = a + b is reduced to O(1) integer updates:
//     H_hi[hi] += 1, H_s[s] += 1            (per pair; equal pairs included)
//     hist[a]  += 1                          (per pixel, as the 'cur' row)
// The curve is rebuilt exactly from these:
//     P      = 4*hist - corr                 (degree-weighted pixel histogram)
//     card[t]= sum_{v<=t} (P[v] - 2 H_hi[v])
//     sum[t] = sum_{u<=t} sum_{u'<=u} ( P[u'-1] - H_s[2u'-3] - 2 H_s[2u'-2] - H_s[2u'-1] )
// because the tent min(hi-t, t-lo) on [lo,hi) (proj/src/kernels/pair_tent.hpp:12-18)
// has second difference +1 at lo+1 and hi+1 and -1 at floor(s/2)+1 and
// ceil(s/2)+1, and equal pairs cancel exactly.  `corr` holds the border
// terms (missing neighbours) and the compensation for the equal "fake" pairs
// the universal lane path creates at row ends (see border_terms()).
//
// Histogram layout in shared memory (128 KiB, "lane-striped"): 512 rows of
// 256 bytes; word (row, half, lane) lives at row*256 + half*128 + lane*4, so
// lane L only ever touches bank L and every warp-wide update is
// bank-conflict free whatever the keys are.  half 0 of row r holds H_s[r]
// (r = 0..510), half 1 of rows 0..255 holds hist[v], half 1 of rows
// 256..511 holds H_hi[v].  The byte address (key << 8) | lane*4 is one PRMT.
#pragma once

#include <cstdint>

namespace kohler_dev {

constexpr int kLevels = 256;
constexpr uint32_t kStripedBytes = 512u * 256u;
constexpr uint32_t kOffHs = 0;             // + (s << 8) | lane4
constexpr uint32_t kOffHist = 128;         // + (v << 8) | lane4
constexpr uint32_t kOffHhi = 65536 + 128;  // + (v << 8) | lane4

__device__ __forceinline__ void inc(unsigned char* base, uint32_t off)
{
    atomicAdd(reinterpret_cast<uint32_t*>(base + off), 1u);
}

// Four pairs packed in 16-bit lanes: x = [a0, a2], y = [b0, b2] (one byte per
// 16-bit lane, upper byte zero).  Two pairs per call.
__device__ __forceinline__ void pairs2(unsigned char* sm, uint32_t x, uint32_t y, uint32_t lane4)
{
    const uint32_t hx = __vmaxu2(x, y);  // VIMNMX.U16x2
    const uint32_t sx = x + y;           // no carry between halves (<= 510)
    inc(sm + kOffHhi, __byte_perm(hx, lane4, 0x5504));
    inc(sm + kOffHhi, __byte_perm(hx, lane4, 0x5524));
    inc(sm + kOffHs, __byte_perm(sx, lane4, 0x5104));
    inc(sm + kOffHs, __byte_perm(sx, lane4, 0x5324));
}

__device__ __forceinline__ void pixels4(unsigned char* sm, uint32_t c, uint32_t lane4)
{
    inc(sm + kOffHist, __byte_perm(c, lane4, 0x5504));
    inc(sm + kOffHist, __byte_perm(c, lane4, 0x5514));
    inc(sm + kOffHist, __byte_perm(c, lane4, 0x5524));
    inc(sm + kOffHist, __byte_perm(c, lane4, 0x5534));
}

// All updates of one 16-pixel segment: 16 right pairs (the 16th against rn),
// 16 down pairs (cur vs nxt) and 16 pixels.  80 conflict-free ATOMS.
__device__ __forceinline__ void accumulate_segment(unsigned char* sm, const uint32_t (&c)[4],
                                                   const uint32_t (&n)[4], uint32_t rn,
                                                   uint32_t lane4)
{
    uint32_t ce[5];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        ce[j] = __byte_perm(c[j], 0, 0x4240);  // [b0, b2]
    ce[4] = rn & 0xFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t co = __byte_perm(c[j], 0, 0x4341);          // [b1, b3]
        const uint32_t ro = __byte_perm(ce[j], ce[j + 1], 0x1412); // [b2, next b0]
        const uint32_t ne = __byte_perm(n[j], 0, 0x4240);
        const uint32_t no = __byte_perm(n[j], 0, 0x4341);
        pairs2(sm, ce[j], co, lane4);  // right pairs (b0,b1), (b2,b3)
        pairs2(sm, co, ro, lane4);     // right pairs (b1,b2), (b3,next)
        pairs2(sm, ce[j], ne, lane4);  // down pairs, columns 0 and 2
        pairs2(sm, co, no, lane4);     // down pairs, columns 1 and 3
        pixels4(sm, c[j], lane4);
    }
}

// Byte i (compile-time index after unrolling) of a 16-byte segment.
__device__ __forceinline__ uint32_t byte_at(const uint32_t (&c)[4], int i)
{
    return (c[i >> 2] >> (8 * (i & 3))) & 0xFFu;
}

// Byte e (runtime index, 0..15) without dynamic register indexing (which
// would force the segment into local memory).
__device__ __forceinline__ uint32_t byte_dyn(const uint32_t (&c)[4], int e)
{
    const uint32_t wd = e < 4 ? c[0] : e < 8 ? c[1] : e < 12 ? c[2] : c[3];
    return (wd >> (8 * (e & 3))) & 0xFFu;
}

// Replace bytes i > e of the segment by v (row-end lanes).
__device__ __forceinline__ void fill_tail(uint32_t (&c)[4], int e, uint32_t v)
{
    const uint32_t vvvv = v * 0x01010101u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int keep = e - 4 * j + 1;  // bytes of word j to keep
        if (keep <= 0)
            c[j] = vvvv;
        else if (keep < 4) {
            const uint32_t m = 0xFFFFFFFFu << (8 * keep);
            c[j] = (c[j] & ~m) | (vvvv & m);
        }
    }
}

template <bool VEC>
__device__ __forceinline__ void load_segment(const uint8_t* row, int x0, int w, uint32_t (&c)[4])
{
    if (VEC) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + x0));
        c[0] = v.x;
        c[1] = v.y;
        c[2] = v.z;
        c[3] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int x = x0 + 4 * j + b;
                const uint32_t byte = x < w ? __ldg(row + x) : 0u;
                word |= byte << (8 * b);
            }
            c[j] = word;
        }
    }
}

// Geometry of one 16-pixel segment step, band-relative.
struct StepGeom {
    int w;         // image width
    int y;         // band-relative row of `cur`
    int band_rows; // own rows of the band
    int gy;        // global row of `cur`
    int h_total;   // global image height
    int x0;        // first column of the segment
};

// One lane's step: fix up row ends / last rows so that every lane runs the
// same predicate-free accumulate_segment, and record the border terms.
//
// Row-end lane (x0 + 16 >= w, e = w-1-x0): bytes > e of cur and nxt and the
// right neighbour are replaced by v = cur[e].  The resulting equal "fake"
// pairs cancel in the reconstruction once P counts them: the garbage pixels'
// 4*hist supplies 4(15-e), the fake pairs need 2(16-e) + 2(15-e), so corr[v]
// gets -2, plus +1 for pixel e's missing right pair: -1 in total.
// Last image row: nxt := cur, so every down pair is an equal fake pair:
// corr += 1 (missing down pair) - 2 (fake) = -1 per real pixel.
// Band-first row: +1 per real pixel (its up pair belongs to the row above /
// does not exist).  Row start: +1 (no left pair).  Halo row pixels (row r1 of
// a band with r1 < h): -1 each (their up pair is owned, P gains 1).
// `corr` is lane-striped like the histograms (word (v, lane) at
// v*128 + lane*4, 32 KiB) so its updates are bank-conflict free, and the
// per-pixel loops are branch-free (a disabled term adds 0).
__device__ __forceinline__ void corr_add(unsigned char* corr, uint32_t lane4, uint32_t v, int d)
{
    atomicAdd(reinterpret_cast<int*>(corr + (v << 7) + lane4), d);
}

struct StripedCorr {  // K1: lane-striped corr (conflict free)
    unsigned char* base;
    uint32_t lane4;
    __device__ __forceinline__ void operator()(uint32_t v, int d) const { corr_add(base, lane4, v, d); }
};

struct PlainCorr {  // K5: one 256-entry corr array per image group
    int* base;
    __device__ __forceinline__ void operator()(uint32_t v, int d) const { atomicAdd(base + v, d); }
};

template <class CorrAdd>
__device__ __forceinline__ void border_terms(const CorrAdd& corr, const StepGeom& g,
                                             uint32_t (&c)[4], uint32_t (&n)[4], uint32_t& rn,
                                             bool has_down)
{
    const int e = g.w - 1 - g.x0;  // index of the last real pixel if < 16
    if (g.x0 == 0)
        corr(c[0] & 0xFFu, 1);
    // +1 (band-first row: no owned up pair), -1 (last image row: missing down
    // pair +1, fake equal down pair -2); both at once cancel.
    const int dcur = (g.y == 0 ? 1 : 0) - (has_down ? 0 : 1);
    if (dcur != 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            corr(byte_at(c, i), i <= e ? dcur : 0);
    }
    if (has_down && g.y + 1 == g.band_rows) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            corr(byte_at(n, i), i <= e ? -1 : 0);
    }
    if (e <= 15) {
        const uint32_t v = byte_dyn(c, e);
        fill_tail(c, e, v);
        if (has_down)
            fill_tail(n, e, v);
        rn = v;
        corr(v, -1);
    }
    if (!has_down) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            n[j] = c[j];
    }
}

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
// prefix(prefix(h2)).  cd(t)/h2(u) are functors; results go to card[]/sum[].
template <class CD, class H2>
__device__ __forceinline__ void warp_curve256(CD cd, H2 h2, uint64_t* card, uint64_t* sum)
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
        a[j] += ea;
        g[j] += eg;
        rs += g[j];
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
    for (int j = 0; j < 8; ++j) {
        card[lane * 8 + j] = (uint64_t)a[j];
        sum[lane * 8 + j] = (uint64_t)(g[j] + es);
    }
}

// Same as warp_curve256 but returns each lane's 8 (card, sum) in registers.
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

// The 512 linear combinations one partial contributes: cd[v] (count first
// difference) in [0,256) and h2[u] (sum second difference) in [256,512).
// hist(v), hhi(v), hs(s) read the partial's reduced histograms.
template <class Hist, class Hhi, class Hs, class Corr>
__device__ __forceinline__ long long combo(int t, Hist hist, Hhi hhi, Hs hs, Corr corr)
{
    if (t < 256) {
        const long long p = 4ll * (long long)hist(t) - (long long)corr(t);
        return p - 2ll * (long long)hhi(t);
    }
    const int u = t - 256;
    if (u == 0)
        return 0;
    const long long p = 4ll * (long long)hist(u - 1) - (long long)corr(u - 1);
    long long r = p - 2ll * (long long)hs(2 * u - 2) - (long long)hs(2 * u - 1);
    if (u >= 2)
        r -= (long long)hs(2 * u - 3);
    return r;
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

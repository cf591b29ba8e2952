// kohler_walk.cuh — K1 accumulation, "three events per pixel".
//
// Every lane walks DOWN a column of one 16-pixel segment, so each pixel's
// four neighbour relations are available without re-reading anything:
// the right pair (within the lane's registers + one neighbour byte), the
// down pair (the next row, loaded ahead) and, carried from the previous
// row, the up pair.  Per pixel x with value v it emits
//
//   W[v]      += B(x) << 16 | 1          (packed: sign sum, pixel count)
//   Hs[v + r] += 1                       (right pair midpoint event)
//   Hs[v + d] += 1                       (down pair midpoint event)
//
// with B(x) = sum over the 4 neighbour slots of (1 + sign(n - v)) in [0, 8]
// (a missing / fake neighbour counts as an equal one).  That is 3 shared
// atomics per pixel instead of the 5 of the marginal-histogram form
// (hist + H_hi + H_s per pair), which is what bounds this kernel.
//
// Reconstruction (SURVEY.md Appendix A restated on these counters): with
// hist = sum of the low fields, Bs = sum of the high fields, P = 4 hist - corr,
//     card'[v] = Bs[v] - 4 hist[v]          (= sum_x sum_n sign(n - v): +1 at lo, -1 at hi)
//     sum''[u] = P[u-1] - Hs[2u-3] - 2 Hs[2u-2] - Hs[2u-1]
// because the tent min(hi - t, t - lo) (proj/src/kernels/pair_tent.hpp:12-18)
// has second difference +1 at lo+1 and hi+1 and -1 at floor(s/2)+1,
// ceil(s/2)+1.  `corr` fixes P at borders: P must count, for every pixel,
// its incidences among the EMITTED pairs, with an emitted equal "fake" pair
// counted twice.  Row start / first band row (pair missing or not owned):
// corr +1.  Row end / last image row (fake equal pair emitted): corr -1.
// Halo pixel (one owned up pair, emitted as a W event): corr +3.
//
// The per-pair sign step q(a -> b) = 1 + sign(b - a) is computed two pairs
// at a time in 16-bit SIMD lanes (qstep below).  Only differences of q enter
// B, so B needs no per-pair offsets.  The work is split between the integer
// ALU pipe and the FMA pipe (IMAD), which on sm_100 each retire half a warp
// instruction per cycle per scheduler; the ALU pipe, not the shared atomics,
// is what bounds this loop.
//
// Shared memory (lane-striped: lane L only touches bank L, so every warp-wide
// update is conflict free for any data):
//   rows of 256 B, word (row, half, lane) at row*256 + half*128 + lane*4
//   half 0, rows 0..510 : Hs[s];  row 511: dummy (neutralised events)
//   half 1, rows 0..255 : W copy 0 (even rows);  rows 256..511: W copy 1 (odd rows)
// A pixel's W address is A = (v << 8) | lane*4 (one PRMT; bytes 2 and 3 come
// from the same byte source as lane*4: the CTA rank bits of a cluster
// launch, else 0); a pair's Hs address is A_a + A_b - lane*4 - rank bits =
// (a + b) << 8 | lane*4 | rank bits (one IADD3).
#pragma once

#include <cstdint>

namespace kohler_walk {

constexpr uint32_t kHistBytes = 512u * 256u;       // Hs / dummy / W0 / W1
constexpr uint32_t kOffW0 = 128;
constexpr uint32_t kOffW1 = 65536 + 128;
constexpr uint32_t kDummy = 511u << 8;
// W word = Bsum << 16 | hist.  A W lane word takes at most this many pixel
// events between spills, so hist and Bsum <= 8 * it fit 16 bits each.
constexpr int kMaxEventsPerWord = 8191;
constexpr uint32_t kTo = 0x02020202u;              // unpack fill: lanes b + 512 ("to" form)
constexpr uint32_t kNeutral = 0x00010001u;         // q of an equal pair, both lanes

// Constants ptxas must not see through: the integer ALU pipe
// (PRMT / IADD3 / LOP3 / LEA / VIADDMNMX) is the saturated math pipe of the
// walk and the FMA pipe (IMAD) is half idle, but ptxas strength-reduces every
// multiply by a KNOWN power of two or by -1 back into an ALU instruction
// (LEA, LEA.HI, IADD3).  A __constant__ word is a run-time value to the
// compiler, so x * c + y stays an IMAD with a constant-bank operand.
#ifndef KOHLER_FMA_SHIFT
#define KOHLER_FMA_SHIFT 4
#endif
__constant__ uint32_t kOpaque[4] = {1u << 24, 0xFFFFFFFFu, 65536u, 0u};

struct Row {  // one prefetched 16-pixel row segment + its neighbour bytes
    uint32_t w[4];
    uint32_t ln, rn;
};

struct Car {  // a row segment in the form the accumulation uses
    uint32_t A[16];      // (v << 8) | lane*4 per pixel
    uint32_t e[4], o[4]; // 16-bit lanes b + 512: e[j] = (b4j, b4j+2), o[j] = (b4j+1, b4j+3)
    uint32_t ue[4], uo[4];  // q(up -> this) per pixel, same lane layout
    uint32_t ln, rn;     // left / right neighbour byte (fixed up at borders)
};

// The sign step q(from -> to) = 1 + sign(to - from) in {0, 1, 2} per 16-bit
// lane, by ONE VIADDMNMX.S16x2.RELU: relu(min(to + nf, 2)) lanewise.
// Unpacked lanes are kept in "to" form x'' = b + 512 (the unpack PRMT's fill
// byte); a "from" operand is nf = 1 - x'' per lane, made by one subtract from
// 0x00020001: the low lane always borrows exactly once (x'' >= 512), which
// the high half of the constant pre-pays.  to + nf = to - from + 1.
__device__ __forceinline__ uint32_t qfrom(uint32_t to_form)
{
#if KOHLER_FMA_SHIFT & 2
    return to_form * kOpaque[1] + 0x00020001u;
#else
    return 0x00020001u - to_form;
#endif
}

__device__ __forceinline__ uint32_t qstep(uint32_t nf, uint32_t to_form)
{
    return __vimin_s16x2_relu(__vadd2(to_form, nf), 0x00020002u);
}

// ---- checked builds (-DKOHLER_CHECKED, lib/libkohler_cuda_checked.so) ----
// compute-sanitizer is not available on the GPU pool, so the checked build
// asserts its own bounds: every shared-memory counter event inside the
// counter block, every other shared access inside the CTA's dynamic window,
// every cp.async source inside the input buffer.  A violation prints where
// and traps (the call then fails with a CUDA error).  Each kernel sets the
// ranges once per CTA (chk_init) before its first access.
#ifdef KOHLER_CHECKED
// The ranges come from the hardware, not from shared state: the dynamic
// window [cvta(dyn), + %dynamic_smem_size) (carrying the cluster rank bits
// like every access), counter events at or above kCtrLo inside it; the
// global source range travels in LaneGeo / FetchStream (g_lo, g_hi).
constexpr uint32_t kCtrLo = 0x10000;  // lowest counter-block address of any kernel
__device__ __noinline__ void chk_fail(int code, uint32_t a)
{
    printf("KOHLER_CHECKED violation %d at 0x%x (block %d thread %d)\n", code, a, (int)blockIdx.x,
           (int)threadIdx.x);
    __trap();
}
__device__ __forceinline__ void chk_window(uint32_t& lo, uint32_t& hi)
{
    extern __shared__ __align__(16) unsigned char kohler_dyn_smem[];
    uint32_t sz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sz));
    lo = (uint32_t)__cvta_generic_to_shared(kohler_dyn_smem);
    hi = lo + sz;
}
__device__ __forceinline__ void chk_sm(uint32_t a, uint32_t bytes)
{
    uint32_t lo, hi;
    chk_window(lo, hi);
    if (a < lo || a + bytes > hi || (a & (bytes >= 4 ? 3 : 0)))
        chk_fail(2, a);
}
__device__ __forceinline__ void chk_ctr(uint32_t a)
{
    chk_sm(a, 4);
    if ((a & 0x00FFFFFFu) < kCtrLo)
        chk_fail(1, a);
}
__device__ __forceinline__ void chk_g(const void* p, uint32_t bytes, const uint8_t* g_lo,
                                      const uint8_t* g_hi)
{
    const uint8_t* q = static_cast<const uint8_t*>(p);
    if (q < g_lo || q + bytes > g_hi)
        chk_fail(3, (uint32_t)(uintptr_t)q);
}
#define KCHK(x) x
#else
#define KCHK(x) do { } while (0)
#endif

__device__ __forceinline__ void red_inc(uint32_t saddr)
{
    KCHK(chk_ctr(saddr));
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(saddr));
}

template <uint32_t OFF>
__device__ __forceinline__ void red_add_imm(uint32_t saddr, uint32_t v)
{
    KCHK(chk_ctr(saddr + OFF));
    asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(saddr), "r"(v), "n"(OFF));
}

__device__ __forceinline__ void red_add(uint32_t saddr, uint32_t v)
{
    KCHK(chk_sm(saddr, 4));
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v));
}

// Unpack a loaded row into Y.  The loads already applied the border rule for
// aligned segments (a row start's left neighbour and a row end's right
// neighbour are the pixel itself: equal => neutral); a ragged segment (row
// end inside it, index e < 15) gets its bytes past the row end replaced by
// the last real pixel, which is also its right neighbour.
template <bool ALIGNED>
__device__ __forceinline__ void absorb(Car& Y, const Row& r0, uint32_t lane4, int e)
{
    Row r = r0;
    if (!ALIGNED && e < 15) {
        const uint32_t wd = e < 4 ? r.w[0] : e < 8 ? r.w[1] : e < 12 ? r.w[2] : r.w[3];
        const uint32_t v = (wd >> (8 * (e & 3))) & 0xFFu;
        const uint32_t vvvv = v * 0x01010101u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int keep = e - 4 * j + 1;  // bytes of word j to keep
            if (keep <= 0)
                r.w[j] = vvvv;
            else if (keep < 4) {
                const uint32_t m = 0xFFFFFFFFu << (8 * keep);
                r.w[j] = (r.w[j] & ~m) | (vvvv & m);
            }
        }
        r.rn = v;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        Y.e[j] = __byte_perm(r.w[j], kTo, 0x4240);
        Y.o[j] = __byte_perm(r.w[j], kTo, 0x4341);
#if KOHLER_FMA_SHIFT & 1
        // the high 16-bit lanes (pixels 4j+2, 4j+3) on the FMA pipe:
        // e >> 8 = (b2 + 512) << 8 | (b0 + 512) >> 8 = (b2 << 8) + 0x20002
        Y.A[4 * j + 0] = __byte_perm(r.w[j], lane4, 0x7604);
        Y.A[4 * j + 1] = __byte_perm(r.w[j], lane4, 0x7614);
        Y.A[4 * j + 2] = __umulhi(Y.e[j], kOpaque[0]) + (lane4 - 0x20002u);
        Y.A[4 * j + 3] = __umulhi(Y.o[j], kOpaque[0]) + (lane4 - 0x20002u);
#else
#pragma unroll
        for (int k = 0; k < 4; ++k)
            Y.A[4 * j + k] = __byte_perm(r.w[j], lane4, 0x7604 | (k << 4));
#endif
    }
    Y.ln = r.ln;
    Y.rn = r.rn;
}

// q of the four pair families of the current row X against the down row
// (De, Do).  qre/qro: right pairs of even/odd pixels; qde/qdo: down pairs.
__device__ __forceinline__ void pair_q(const Car& X, const uint32_t (&De)[4],
                                       const uint32_t (&Do)[4], uint32_t (&qre)[4],
                                       uint32_t (&qro)[4], uint32_t (&qde)[4], uint32_t (&qdo)[4])
{
    const uint32_t rn_to = X.rn | 0x0200u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t ro = __byte_perm(X.e[j], j < 3 ? X.e[j + 1] : rn_to, 0x5432);
        const uint32_t fe = qfrom(X.e[j]), fo = qfrom(X.o[j]);
        qre[j] = qstep(fe, X.o[j]);
        qro[j] = qstep(fo, ro);
        qde[j] = qstep(fe, De[j]);
        qdo[j] = qstep(fo, Do[j]);
    }
}

// B(x) for the 16 pixels, exact in 16-bit lanes: Be[j] = (B(4j), B(4j+2)),
// Bo[j] = (B(4j+1), B(4j+3)).
__device__ __forceinline__ void b_terms(const Car& X, const uint32_t (&qre)[4],
                                        const uint32_t (&qro)[4], const uint32_t (&qde)[4],
                                        const uint32_t (&qdo)[4], uint32_t (&Be)[4],
                                        uint32_t (&Bo)[4])
{
    // low lane: q(left neighbour -> b0), nf = 1 - (ln + 512)
    const uint32_t qL = qstep(0xFFFFFE01u - X.ln, X.e[0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t qrl = j == 0 ? __byte_perm(qL, qro[0], 0x5410)
                                    : __byte_perm(qro[j - 1], qro[j], 0x5432);
        Be[j] = 0x00040004u + qre[j] - qrl + qde[j] - X.ue[j];
        Bo[j] = 0x00040004u + qro[j] - qre[j] + qdo[j] - X.uo[j];
    }
}

// Increment of pixel i's W word, B(i) << 16 | 1: the low lane by one IMAD
// (the high lane shifts out), the high lane by one LOP3.
__device__ __forceinline__ uint32_t inc_of(uint32_t lanes, int hi)
{
    if (!hi)
#if KOHLER_FMA_SHIFT & 4
        return lanes * kOpaque[2] + 1u;
#else
        return lanes * 65536u + 1u;
#endif
    uint32_t r;
    asm("lop3.b32 %0, %1, 0xFFFF0000, %2, 0xEA;" : "=r"(r) : "r"(lanes), "r"(1u));  // (a & b) | c
    return r;
}

__device__ __forceinline__ uint32_t b_of(const uint32_t (&Be)[4], const uint32_t (&Bo)[4], int i)
{
    return inc_of((i & 1) ? Bo[i >> 2] : Be[i >> 2], i & 2);
}

} // namespace kohler_walk

// ---- single-warp finish for 256-level curves (K3 + K4) --------------------
//
// One warp, lane L owning thresholds t = 8L .. 8L+7 in registers, restates
// proj/src/threshold.cpp exactly (for finite values):
//   mean_contrast (:9-23)       values[t] = (double)sum / (double)card, defined iff card > 0
//   optimal_threshold (:25-37)  argmax over defined t, ties to the smallest t
//   top_k_local_maxima (:39-82) collapse equal-valued runs of the defined
//                               subsequence (first t kept), keep runs strictly
//                               above both neighbouring runs (one-sided at the
//                               ends), rank by (value desc, t asc), keep k,
//                               report ascending.
// Cross-lane information moves by warp scans of per-lane summaries:
//   prefix: the last defined value left of a lane;
//   suffix: the value of the leftmost run right of a lane and the value of
//           the run after it (a run may continue across lanes).
namespace kohler_walk {

struct RunSum {      // summary of a range of thresholds (its defined entries)
    int has;         // any defined entry
    double lv;       // leftmost run value
    int lnext_has;   // a second run exists
    double lnext;    // value of the run after the leftmost run
};

__device__ __forceinline__ RunSum runsum_combine(const RunSum& A, const RunSum& B)
{
    // A left of B
    if (!A.has)
        return B;
    if (!B.has)
        return A;
    RunSum r;
    r.has = 1;
    r.lv = A.lv;
    if (A.lnext_has) {
        r.lnext_has = 1;
        r.lnext = A.lnext;
    } else if (A.lv == B.lv) {  // A is one run continuing into B's leftmost run
        r.lnext_has = B.lnext_has;
        r.lnext = B.lnext;
    } else {
        r.lnext_has = 1;
        r.lnext = B.lv;
    }
    return r;
}

__device__ __forceinline__ RunSum runsum_shfl_down(const RunSum& x, int off)
{
    RunSum y;
    y.has = __shfl_down_sync(0xFFFFFFFFu, x.has, off);
    y.lv = __shfl_down_sync(0xFFFFFFFFu, x.lv, off);
    y.lnext_has = __shfl_down_sync(0xFFFFFFFFu, x.lnext_has, off);
    y.lnext = __shfl_down_sync(0xFFFFFFFFu, x.lnext, off);
    return y;
}

// better (value desc, t asc) of two candidates; t < 0 = none
__device__ __forceinline__ void best_of(double& bv, int& bt, double ov, int ot)
{
    if (ot >= 0 && (bt < 0 || ov > bv || (ov == bv && ot < bt))) {
        bv = ov;
        bt = ot;
    }
}

// v/d: this lane's 8 values / defined flags (t = 8 lane + j).  mv/mt: smem
// scratch for the maxima (>= 128 entries).  Returns 1 (no boundary) or 0.
__device__ int warp_select256_regs(const double (&v)[8], const bool (&d)[8], int k, double* mv,
                                   int* mt, int* out_t0, int* out_topk, int* out_count)
{
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // optimal threshold
    double bv = 0.0;
    int bt = -1;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (d[j] && (bt < 0 || v[j] > bv)) {
            bv = v[j];
            bt = 8 * lane + j;
        }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, off);
        const int ot = __shfl_xor_sync(0xFFFFFFFFu, bt, off);
        best_of(bv, bt, ov, ot);
    }
    if (bt < 0) {  // nothing defined: NoBoundaryError
        if (lane == 0) {
            if (out_t0)
                *out_t0 = -1;
            if (out_count)
                *out_count = 0;
        }
        return 1;
    }
    // prefix: last defined value strictly left of this lane
    int ph = 0;
    double pv = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (d[j]) {
            ph = 1;
            pv = v[j];
        }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int oh = __shfl_up_sync(0xFFFFFFFFu, ph, off);
        const double ov = __shfl_up_sync(0xFFFFFFFFu, pv, off);
        if (lane >= off && !ph) {
            ph = oh;
            pv = ov;
        }
    }
    int cin_h = __shfl_up_sync(0xFFFFFFFFu, ph, 1);
    double cin_v = __shfl_up_sync(0xFFFFFFFFu, pv, 1);
    if (lane == 0)
        cin_h = 0;
    // suffix: run summary of everything right of this lane
    RunSum mine{0, 0.0, 0, 0.0};
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        if (d[j]) {
            RunSum e{1, v[j], 0, 0.0};
            mine = runsum_combine(e, mine);
        }
    }
    RunSum suf = mine;  // inclusive suffix over lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const RunSum o = runsum_shfl_down(suf, off);
        if (lane + off < 32)
            suf = runsum_combine(suf, o);
    }
    RunSum right = runsum_shfl_down(suf, 1);  // lanes > lane
    if (lane == 31)
        right.has = 0;
    // per entry, right to left: value of the next run after the entry's run
    // (nr_has/nr), tracking the run the entry belongs to (cur)
    bool is_start[8];
    double nxt[8];
    bool nxt_has[8];
    {
        int ch = right.has;
        double cv = right.lv;                 // value of the run right of here
        int nh = right.lnext_has;
        double nv = right.lnext;              // and the run after it
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            if (d[j]) {
                if (!ch) {
                    ch = 1;
                    cv = v[j];
                    nh = 0;
                } else if (v[j] != cv) {
                    nh = 1;
                    nv = cv;
                    cv = v[j];
                }
                nxt_has[j] = nh;
                nxt[j] = nv;
            } else {
                nxt_has[j] = false;
                nxt[j] = 0.0;
            }
        }
    }
    // left to right: run starts and their maxima
    unsigned maxmask = 0;
    {
        int hh = cin_h;
        double hv = cin_v;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            is_start[j] = false;
            if (d[j]) {
                is_start[j] = !hh || v[j] != hv;
                if (is_start[j] && (!hh || hv < v[j]) && (!nxt_has[j] || nxt[j] < v[j]))
                    maxmask |= 1u << j;
                hh = 1;
                hv = v[j];
            }
        }
    }
    // compact the maxima in t order
    const int myn = __popc(maxmask);
    int pre = myn;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xFFFFFFFFu, pre, off);
        if (lane >= off)
            pre += o;
    }
    const int nm = __shfl_sync(0xFFFFFFFFu, pre, 31);
    int pos = pre - myn;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (maxmask & (1u << j)) {
            mv[pos] = v[j];
            mt[pos] = 8 * lane + j;
            ++pos;
        }
    __syncwarp();
    // top-k: k rounds of warp argmax over the maxima (<= 128: 4 per lane)
    double cv[4];
    int ct[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        ct[q] = i < nm ? mt[i] : -1;
        cv[q] = i < nm ? mv[i] : 0.0;
    }
    unsigned sel = 0;  // bit q: candidate lane + 32 q selected
    if (k >= nm) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (ct[q] >= 0)
                sel |= 1u << q;
    } else {
        for (int r = 0; r < k; ++r) {
            double lv = 0.0;
            int ltt = -1;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!(sel & (1u << q)))
                    best_of(lv, ltt, cv[q], ct[q]);
            double gv = lv;
            int gt = ltt;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xFFFFFFFFu, gv, off);
                const int ot = __shfl_xor_sync(0xFFFFFFFFu, gt, off);
                best_of(gv, gt, ov, ot);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (ct[q] == gt)
                    sel |= 1u << q;
        }
    }
    // report ascending t: candidates are in t order (index lane + 32 q)
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const bool s = (sel >> q) & 1u;
        const unsigned b = __ballot_sync(0xFFFFFFFFu, s);
        if (s && out_topk)
            out_topk[cnt + __popc(b & lt)] = ct[q];
        cnt += __popc(b);
    }
    if (lane == 0) {
        if (out_t0)
            *out_t0 = bt;
        if (out_count)
            *out_count = cnt;
    }
    return 0;
}

} // namespace kohler_walk

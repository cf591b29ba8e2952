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
// Cross-lane information moves by warp votes and indexed shuffles (see
// warp_select256_regs).
namespace kohler_walk {


// Order-preserving 64-bit key of a finite double (-0.0 counts as +0.0, like
// the IEEE comparison): a > b  <=>  key(a) > key(b),  a == b  <=>  equal keys.
// Every finite value has a key > 0, so 0 stands for "no value".
__device__ __forceinline__ unsigned long long order_key(double x)
{
    const long long b = __double_as_longlong(x + 0.0);
    return b < 0 ? ~(unsigned long long)b : (unsigned long long)b | 0x8000000000000000ull;
}

__device__ __forceinline__ double shfl_f64(double x, int src)
{
    return __shfl_sync(0xFFFFFFFFu, x, src);
}

// v/d: this lane's 8 values / defined flags (t = 8 lane + j).  mk/mt: smem
// scratch for the maxima (>= 128 entries: keys and thresholds).  Returns 1
// (no boundary) or 0.
//
// The rules only compare each defined value with the previous defined one,
// so a lane reduces its 8 entries to three bit masks -- S: a run starts here
// (first defined value, or it differs from the previous one), U: it is a
// rise (or nothing precedes it), F: it is a fall -- in straight-line
// predicated code, and a run start is a local maximum iff it is a rise and
// the NEXT run start, wherever it is, is a fall or does not exist.  Across
// lanes that takes one indexed shuffle (the last defined value left of the
// lane) and votes (which lanes hold a run start, and whether their first one
// is a fall); the earlier forms moved whole run summaries by log-step scans
// (~165 dependent SHFL and ~1180 instructions per curve; now 2 SHFL, ~12
// votes / REDUX).  Then:
//   compaction prefix sums of the per-lane maxima counts by votes per bit;
//   top-k      rank of every local maximum among all of them (value desc,
//              t asc) from the shared-memory list, keep rank < k;
//   optimum    the rank-0 maximum (the first threshold of the first run with
//              the largest value is always a local maximum), by REDUX.
__device__ int warp_select256_regs(const double (&v)[8], const bool (&d)[8], int k,
                                   unsigned long long* mk, int* mt, int* out_t0, int* out_topk,
                                   int* out_count)
{
    constexpr unsigned kFull = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    unsigned dm = 0;
    double lastv = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        dm |= (d[j] ? 1u : 0u) << j;
        lastv = d[j] ? v[j] : lastv;
    }
    const unsigned H = __ballot_sync(kFull, dm != 0);
    if (H == 0) {  // nothing defined: NoBoundaryError
        if (lane == 0) {
            if (out_t0)
                *out_t0 = -1;
            if (out_count)
                *out_count = 0;
        }
        return 1;
    }
    // the last defined value strictly left of this lane
    const unsigned Hl = H & lt;
    double pv = shfl_f64(lastv, Hl ? 31 - __clz(Hl) : lane);
    bool ph = Hl != 0;
    // every defined entry against the previous defined value
    unsigned S = 0, U = 0, F = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const bool gt = v[j] > pv, ne = v[j] != pv;
        const bool st = d[j] && (!ph || ne);
        const bool up = d[j] && (!ph || gt);
        const bool fl = d[j] && ph && ne && !gt;
        S |= (st ? 1u : 0u) << j;
        U |= (up ? 1u : 0u) << j;
        F |= (fl ? 1u : 0u) << j;
        pv = d[j] ? v[j] : pv;
        ph = ph || d[j];
    }
    // the first run start right of this lane: none, or a fall => a maximum may end here
    const unsigned BS = __ballot_sync(kFull, S != 0);
    const unsigned BF = __ballot_sync(kFull, (F & (S & (0u - S))) != 0);
    const unsigned BSr = BS & (0xFFFFFFFEu << lane);
    unsigned carry = BSr ? (BF >> (__ffs(BSr) - 1)) & 1u : 1u;
    unsigned ok = 0;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        const unsigned m = (S >> j) & 1u;
        ok |= (carry & m) << j;
        carry = m ? (F >> j) & 1u : carry;
    }
    const unsigned maxmask = S & U & ok;
    // compact the maxima in t order (a lane has <= 4: strict maxima are never adjacent)
    const int myn = __popc(maxmask);
    int pos = 0, nm = 0;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const unsigned m = __ballot_sync(kFull, (myn >> b) & 1);
        pos += __popc(m & lt) << b;
        nm += __popc(m) << b;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (maxmask & (1u << j)) {
            KCHK(if (pos < 0 || pos >= 128) chk_fail(4, (uint32_t)pos));  // <= 128 maxima exist
            mk[pos] = order_key(v[j]);
            mt[pos] = 8 * lane + j;
            ++pos;
        }
    __syncwarp();
    // candidates lane + 32 q (t order)
    unsigned long long ck[4];
    int ct[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        const bool in = i < nm;
        ck[q] = in ? mk[i] : 0ull;
        ct[q] = in ? mt[i] : -1;
    }
    // optimal threshold = the largest maximum, ties to the smallest t
    {
        unsigned long long key = ck[0];
        int bt = ct[0];
#pragma unroll
        for (int q = 1; q < 4; ++q)
            if (ck[q] > key) {  // later candidates have larger t: strict
                key = ck[q];
                bt = ct[q];
            }
        const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
        const unsigned mh = __reduce_max_sync(kFull, khi);
        const bool c1 = khi == mh;
        const unsigned ml = __reduce_max_sync(kFull, c1 ? klo : 0u);
        const bool c2 = c1 && klo == ml && bt >= 0;
        const unsigned t0 = __reduce_min_sync(kFull, c2 ? (unsigned)bt : 0x7FFFFFFFu);
        if (lane == 0 && out_t0)
            *out_t0 = (int)t0;
    }
    unsigned sel = 0;  // bit q: candidate lane + 32 q selected
    if (k >= nm) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (ct[q] >= 0)
                sel |= 1u << q;
    } else {
        // rank among all maxima (value desc, t asc = list index asc)
        int rank[4] = {0, 0, 0, 0};
        if (nm <= 32) {
#pragma unroll 4
            for (int j = 0; j < nm; ++j) {
                const unsigned long long x = mk[j];  // broadcast
                rank[0] += (x > ck[0] || (x == ck[0] && j < lane)) ? 1 : 0;
            }
        } else {
#pragma unroll 2
            for (int j = 0; j < nm; ++j) {
                const unsigned long long x = mk[j];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    rank[q] += (x > ck[q] || (x == ck[q] && j < lane + 32 * q)) ? 1 : 0;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (ct[q] >= 0 && rank[q] < k)
                sel |= 1u << q;
    }
    // report ascending t: candidates are in t order (index lane + 32 q)
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const bool s = (sel >> q) & 1u;
        const unsigned b = __ballot_sync(kFull, s);
        if (s && out_topk)
            out_topk[cnt + __popc(b & lt)] = ct[q];
        cnt += __popc(b);
    }
    if (lane == 0 && out_count)
        *out_count = cnt;
    return 0;
}

} // namespace kohler_walk

/*
 * kohler_oracle.c — CPU restatement of the reference's Köhler contrast-curve
 * path.  TEST INFRASTRUCTURE ONLY: this file is the checker that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA
 * product path against.  Nothing in paper_1707_05062_b200/ links, loads or
 * calls it; the product path fails loudly when its CUDA library is missing.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (1) the hand-derived constants of the reference's own tests
 *     (proj/tests/test_contrast.cpp:32-123, test_threshold.cpp:50-183,
 *      acceptance.cpp:158-202), and
 * (2) golden vectors produced by the reference library itself compiled from
 *     /root/reference (oracle/_ref/libkohler_ref.so, oracle/Makefile) and
 *     committed under tests/golden/ by tests/golden/make_golden.py.
 *
 * Every function cites the reference lines it restates.  Scalar, single
 * threaded, written for clarity rather than speed.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "kohler_oracle.h"

/* Tent update of one unordered pair, lo <= hi: every threshold t in [lo, hi)
 * gains min(hi - t, t - lo) contrast and one boundary pair.
 * Restates proj/src/kernels/pair_tent.hpp:12-18 and curve.cpp:10-14. */
void oracle_pair_contribution(int lo, int hi, uint64_t *sum, uint64_t *card)
{
    for (int t = lo; t < hi; ++t) {
        int up = t - lo, down = hi - t;
        sum[t] += (uint64_t)(up < down ? up : down);
        card[t] += 1;
    }
}

/* One run of parallel pixel pairs (cur[j], nbr[j]); equal pairs are skipped.
 * Restates proj/src/kernels/pair_scalar.cpp:12-22. */
static void pair_run(const uint8_t *cur, const uint8_t *nbr, size_t n, uint64_t *sum,
                     uint64_t *card)
{
    for (size_t j = 0; j < n; ++j) {
        int a = cur[j], b = nbr[j];
        if (a == b)
            continue;
        oracle_pair_contribution(a < b ? a : b, a < b ? b : a, sum, card);
    }
}

/* Pairs owned by rows [r0, r1) of a row-major w x h image with row pitch
 * `pitch`: the right pairs inside each row and the down pairs into the next
 * row; no padding, no wraparound.  ACCUMULATES into sum/card.
 * Restates proj/src/fast.cpp:15-32 (accumulate_rows). */
void oracle_curve_rows(const uint8_t *px, int w, int h, size_t pitch, int r0, int r1,
                       uint64_t *sum, uint64_t *card)
{
    for (int i = r0; i < r1; ++i) {
        const uint8_t *row = px + (size_t)i * pitch;
        if (w > 1)
            pair_run(row, row + 1, (size_t)w - 1, sum, card);
        if (i + 1 < h)
            pair_run(row, row + pitch, (size_t)w, sum, card);
    }
}

/* Whole-image curve with one worker; writes (zeroes first) 256 entries.
 * Restates proj/src/fast.cpp:36-48 for workers == 1 (the worker count does
 * not change the result: contrast.hpp:13-17). */
void oracle_fast_curve(const uint8_t *px, int w, int h, uint64_t *sum, uint64_t *card)
{
    memset(sum, 0, ORACLE_LEVELS * sizeof(uint64_t));
    memset(card, 0, ORACLE_LEVELS * sizeof(uint64_t));
    oracle_curve_rows(px, w, h, (size_t)w, 0, h, sum, card);
}

/* Row-block decomposition exactly as the threaded driver splits it, merged by
 * entrywise sum.  Restates proj/src/fast.cpp:42-61 + curve.cpp:16-30. */
void oracle_fast_curve_blocks(const uint8_t *px, int w, int h, unsigned blocks,
                              uint64_t *sum, uint64_t *card)
{
    uint64_t ps[ORACLE_LEVELS], pc[ORACLE_LEVELS];
    memset(sum, 0, ORACLE_LEVELS * sizeof(uint64_t));
    memset(card, 0, ORACLE_LEVELS * sizeof(uint64_t));
    if (blocks > (unsigned)h)
        blocks = (unsigned)h;
    if (blocks < 1)
        blocks = 1;
    for (unsigned b = 0; b < blocks; ++b) {
        int r0 = (int)((uint64_t)h * b / blocks);
        int r1 = (int)((uint64_t)h * (b + 1) / blocks);
        memset(ps, 0, sizeof ps);
        memset(pc, 0, sizeof pc);
        oracle_curve_rows(px, w, h, (size_t)w, r0, r1, ps, pc);
        for (int t = 0; t < ORACLE_LEVELS; ++t) {
            sum[t] += ps[t];
            card[t] += pc[t];
        }
    }
}

/* Definition-level curve: for each threshold, scan all ordered 4-neighbour
 * pairs (x0 in the lower class, x1 in the upper one).  Θ(256·4·N).
 * Restates proj/src/direct.cpp:10-43. */
void oracle_direct_curve(const uint8_t *px, int w, int h, uint64_t *sum, uint64_t *card)
{
    static const int dx[4] = {1, -1, 0, 0};
    static const int dy[4] = {0, 0, 1, -1};
    for (int t = 0; t < ORACLE_LEVELS; ++t) {
        uint64_t s = 0, c = 0;
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                int v0 = px[(size_t)y * w + x];
                if (v0 > t)
                    continue;
                for (int k = 0; k < 4; ++k) {
                    int x1 = x + dx[k], y1 = y + dy[k];
                    if (x1 < 0 || x1 >= w || y1 < 0 || y1 >= h)
                        continue;
                    int v1 = px[(size_t)y1 * w + x1];
                    if (v1 > t) {
                        c += 1;
                        s += (uint64_t)(v1 - t < t - v0 ? v1 - t : t - v0);
                    }
                }
            }
        sum[t] = s;
        card[t] = c;
    }
}

/* values[t] = sum/card as IEEE double where card > 0, else 0 and undefined.
 * Restates proj/src/threshold.cpp:9-23. */
void oracle_mean_contrast(const uint64_t *sum, const uint64_t *card, int n, double *values,
                          uint8_t *defined)
{
    for (int t = 0; t < n; ++t) {
        if (card[t] > 0) {
            values[t] = (double)sum[t] / (double)card[t];
            defined[t] = 1;
        } else {
            values[t] = 0.0;
            defined[t] = 0;
        }
    }
}

/* Argmax over defined entries, strict '>' so the smallest t wins ties;
 * returns -1 when nothing is defined (the reference throws NoBoundaryError).
 * Restates proj/src/threshold.cpp:25-37. */
int oracle_optimal_threshold(const double *values, const uint8_t *defined, int n)
{
    int best = -1;
    for (int t = 0; t < n; ++t) {
        if (!defined[t])
            continue;
        if (best < 0 || values[t] > values[best])
            best = t;
    }
    return best;
}

typedef struct {
    double value;
    int first_t;
} oracle_run;

static int run_rank_cmp(const void *pa, const void *pb)
{
    const oracle_run *a = (const oracle_run *)pa, *b = (const oracle_run *)pb;
    if (a->value != b->value)
        return a->value > b->value ? -1 : 1;
    return (a->first_t > b->first_t) - (a->first_t < b->first_t);
}

static int int_cmp(const void *pa, const void *pb)
{
    int a = *(const int *)pa, b = *(const int *)pb;
    return (a > b) - (a < b);
}

/* Top-k local maxima of the defined subsequence.  Runs of exactly equal
 * values collapse to their smallest t; a run is a maximum when strictly above
 * both neighbouring runs (one-sided at the ends); rank by value desc then t
 * asc; keep k; return ascending.  Status: 0 ok, ORACLE_NO_BOUNDARY when no
 * entry is defined, ORACLE_INVALID_K when k < 1 (checked first).
 * Restates proj/src/threshold.cpp:39-82. */
int oracle_top_k_local_maxima(const double *values, const uint8_t *defined, int n, int k,
                              int *out, int *out_count)
{
    *out_count = 0;
    if (k < 1)
        return ORACLE_INVALID_K;
    oracle_run *runs = (oracle_run *)malloc(sizeof(oracle_run) * (size_t)(n > 0 ? n : 1));
    oracle_run *maxima = (oracle_run *)malloc(sizeof(oracle_run) * (size_t)(n > 0 ? n : 1));
    int nr = 0, nm = 0;
    for (int t = 0; t < n; ++t) {
        if (!defined[t])
            continue;
        if (nr == 0 || values[t] != runs[nr - 1].value) {
            runs[nr].value = values[t];
            runs[nr].first_t = t;
            ++nr;
        }
    }
    if (nr == 0) {
        free(runs);
        free(maxima);
        return ORACLE_NO_BOUNDARY;
    }
    for (int r = 0; r < nr; ++r) {
        int above_prev = (r == 0) || runs[r].value > runs[r - 1].value;
        int above_next = (r + 1 == nr) || runs[r].value > runs[r + 1].value;
        if (above_prev && above_next)
            maxima[nm++] = runs[r];
    }
    qsort(maxima, (size_t)nm, sizeof(oracle_run), run_rank_cmp);
    if (nm > k)
        nm = k;
    for (int i = 0; i < nm; ++i)
        out[i] = maxima[i].first_t;
    qsort(out, (size_t)nm, sizeof(int), int_cmp);
    *out_count = nm;
    free(runs);
    free(maxima);
    return 0;
}

/* Σ over unordered N4 pairs of |a-b| and of floor((a-b)^2/4): the
 * total-variation and quarter-square identities the reference's tests hold
 * the curve to (proj/tests/test_support.hpp:70-102). */
void oracle_identities(const uint8_t *px, int w, int h, uint64_t *tv, uint64_t *qs)
{
    uint64_t a = 0, b = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int v = px[(size_t)y * w + x];
            if (x + 1 < w) {
                int d = abs(v - px[(size_t)y * w + x + 1]);
                a += (uint64_t)d;
                b += (uint64_t)d * (uint64_t)d / 4;
            }
            if (y + 1 < h) {
                int d = abs(v - px[(size_t)(y + 1) * w + x]);
                a += (uint64_t)d;
                b += (uint64_t)d * (uint64_t)d / 4;
            }
        }
    *tv = a;
    *qs = b;
}

/* Whole pipeline for one image: curve, mean curve, t0, top-k (the timed
 * section of proj/src/bench.cpp:174-181 plus proj/tools/kohler_main.cpp:95-105).
 * Returns 0 or ORACLE_NO_BOUNDARY (t0 = -1, no thresholds). */
int oracle_analyze(const uint8_t *px, int w, int h, int k, uint64_t *sum, uint64_t *card,
                   double *values, uint8_t *defined, int *t0, int *topk, int *topk_count)
{
    oracle_fast_curve(px, w, h, sum, card);
    oracle_mean_contrast(sum, card, ORACLE_LEVELS, values, defined);
    *t0 = oracle_optimal_threshold(values, defined, ORACLE_LEVELS);
    return oracle_top_k_local_maxima(values, defined, ORACLE_LEVELS, k, topk, topk_count);
}

/* Rec. 601 integer luma of one RGB sample, as the reference's luma601
 * (proj/src/pnm.cpp:63-68): round half up in thousandths, clamped to 255. */
uint8_t oracle_luma601(unsigned r, unsigned g, unsigned b)
{
    const unsigned v = (299u * r + 587u * g + 114u * b + 500u) / 1000u;
    return (uint8_t)(v < 255u ? v : 255u);
}

/* Colour reduction of read_pnm for P6 / P3 (proj/src/pnm.cpp:110-136):
 * interleaved RGB rows of `pitch` bytes -> w x h grey, row-major. */
void oracle_rgb_to_gray(const uint8_t *rgb, int w, int h, size_t pitch, uint8_t *out)
{
    for (int y = 0; y < h; ++y) {
        const uint8_t *row = rgb + (size_t)y * pitch;
        for (int x = 0; x < w; ++x)
            out[(size_t)y * w + x] = oracle_luma601(row[3 * x], row[3 * x + 1], row[3 * x + 2]);
    }
}

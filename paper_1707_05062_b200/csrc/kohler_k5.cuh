// kohler_k5.cuh — K5 twalk_kernel: batches of small images.
// Part of the single translation unit kohler_kernels.cu (included there,
// in this order, after the shared constants and parameter blocks).
#pragma once

namespace {

#ifdef KOHLER_CHECKED
using kohler_walk::chk_g;
using kohler_walk::chk_sm;
#endif

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

// Per-group border-term arrays int[256] at a 1040-byte stride: the 8 groups'
// arrays start in different 16-byte bank quads, so the flush's per-group
// LDS.128 reads of a quarter warp are conflict free (a 1024-byte stride made
// them 8-way conflicts, ncu r7).
constexpr uint32_t kTwCorrStride = 1040;
#ifndef KOHLER_TW_SLOTS
#define KOHLER_TW_SLOTS 3
#endif

template <int LG>
struct TwLayout {
    static constexpr int NG = 32 / LG;
    // LG = 4 (8 images per round, walks of <= 31 rows): one W copy (a lane
    // word takes <= 16 warps * 31 rows * 16 px <= 8191 events per round)
    static constexpr bool kOneW = LG == 4;
    // 32 lane segments (512 B, 128-byte aligned), then 2 pads per group
    static constexpr uint32_t kSlot = (512 + 32 * NG + 127) / 128 * 128;
    static constexpr uint32_t kRing = 0;  // + up to 127 B of alignment
    // ring slots per warp (KOHLER_TW_SLOTS, default 3: 2 rows in flight; 4
    // measured 0.4 % slower on C5)
    static constexpr int kSlots = KOHLER_TW_SLOTS;
    static constexpr int kAhead = kSlots - 1;
    static constexpr uint32_t kRingBytes = kTwWarps * kSlots * kSlot + 128;
    static constexpr uint32_t kCorr = kRingBytes;  // int[NG][260] (not with one W copy)
    static constexpr uint32_t kTot = kCorr + (kOneW ? 0u : NG * kTwCorrStride);  // i64 [3][16 warps][NG] scan carries
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
#ifdef KOHLER_CHECKED
    L.g_lo = p.px;
    L.g_hi = p.px + (size_t)(p.n - 1) * p.image_stride + (size_t)p.h * p.pitch;
#endif
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
    const uint32_t corr_g = smbase + Lay::kCorr + (uint32_t)g * kTwCorrStride;
    const uint32_t corr_base = corr_g - (lane4 >> 6);
    // border term corr[v] += d of a pixel with W address A: with one W copy
    // (LG = 4) the unused second copy is a lane-striped corr table (conflict
    // free, no address arithmetic); otherwise the per-group int arrays
    auto corr_add = [&](uint32_t A, uint32_t d) {
        if constexpr (Lay::kOneW)
            red_add_imm<kHistAbs + kOffW1>(A, d);
        else
            red_add(corr_base + (A >> 6), d);
    };
    const uint32_t pitch = (uint32_t)p.pitch;
    const int task = warp * LG + lig;
    const int P = p.R + 2;
    const uint32_t ring = (smbase + Lay::kRing + 127u) & ~127u;
    constexpr int AH = Lay::kAhead;
    const uint32_t seg0 = ring + (uint32_t)warp * (Lay::kSlots * Lay::kSlot) + (uint32_t)lane * 16u;
    const uint32_t slot_end = seg0 + Lay::kSlots * Lay::kSlot;
    uint32_t sl_cur = seg0, sl_prev = seg0 + (Lay::kSlots - 1) * Lay::kSlot;
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
#pragma unroll
    for (int f = 0; f < AH; ++f)
        fetch_row<false>(G, f, pitch, seg0 + f * Lay::kSlot);
    {
        uint4* z = reinterpret_cast<uint4*>(hist);
        for (int i = tid; i < (int)(kHistBytes / 16); i += kTwThreads)
            z[i] = make_uint4(0, 0, 0, 0);
        if constexpr (!Lay::kOneW)
            for (int i = tid; i < NG * (int)(kTwCorrStride / 4); i += kTwThreads)
                reinterpret_cast<int*>(sm + Lay::kCorr)[i] = 0;
    }
    __syncthreads();
    bool waited = false;
    Car X, Y;
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
            constexpr uint32_t kOffW = (WC && !Lay::kOneW) ? kOffW1 : kOffW0;
            if (AH > 2)
                asm volatile("cp.async.wait_group 2;" ::: "memory");
            else
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncwarp();
            Row r;  // read first: the prefetch issue covers the LDS latency
            read_row_shfl<false>(r, sl_cur, nb);
            const uint32_t pref = sl_prev;  // slot of position j + AH (j - 1's, read already)
            sl_prev = sl_cur;
            sl_cur = sl_cur + Lay::kSlot == slot_end ? seg0 : sl_cur + Lay::kSlot;
            if (!CROSS || j + AH < P)
                fetch_row<false>(G, j + AH, pitch, pref);
            else if (has_next)
                fetch_row<false>(N, j + AH - P, pitch, pref);
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
                // the image's first row (no up pairs): corr +1 per pixel, from
                // the row just absorbed (no global re-read after the walk)
                if (G.nrows > 0 && !has_up) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (ALIGNED || i <= G.e)
                            corr_add(D.A[i], 1u);
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
                    corr_add(C.A[0], 1u);
                if (row_end)
                    corr_add(Arn, 0xFFFFFFFFu);
            }
        };
        using K0 = std::integral_constant<int, 0>;
        using K1 = std::integral_constant<int, 1>;
        using K2 = std::integral_constant<int, 2>;
        using W0 = std::integral_constant<int, 0>;
        using W1 = std::integral_constant<int, 1>;
        using NC = std::false_type;
        using CR = std::true_type;
        if (P > AH + 1) {
            step(X, Y, 0, K0{}, W0{}, NC{});
            step(Y, X, 1, K1{}, W1{}, NC{});
        } else {
            if (has_next)
                N = geo(i0 + stride);
            step(X, Y, 0, K0{}, W0{}, CR{});
            step(Y, X, 1, K1{}, W1{}, CR{});
        }
        int j = 2;
        for (; j + AH + 1 < P; j += 2) {
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
        // the image's last row (its down pairs were emitted as equal fakes:
        // the down row was the row itself): corr -1 per pixel.  It was the
        // row processed at position P - 1 (C of that step: Y if P - 1 is
        // even, else X); outside the walk loop, which stays branch-free.
        if (G.nrows > 0 && G.y0 + G.nrows == p.h) {
            const Car& Cl = ((P - 1) & 1) ? X : Y;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (ALIGNED || i <= G.e)
                    corr_add(Cl.A[i], 0xFFFFFFFFu);
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
            // gi = L & 7, keys t0 .. t0 + 3 (t0 = 16 w + 4 (L >> 3)) of the W
            // table and rows 2 t0 - 1 .. 2 t0 + 6 of the Hs table.  A group's 4
            // lane words of a counter row are one 16-byte piece and the 8
            // lanes of a quarter warp (one LDS.128 wavefront) take 8 images,
            // i.e. 8 bank quads: conflict free.  Every piece has exactly one
            // reader, which clears it right after reading (no second pass).
            // No lane needs another lane's counters: the terms a lane holds
            // for the NEXT lane's first key travel with its scan total (see
            // dA below), so the flush has one barrier -- the exchange of the
            // warps' scan totals.
            const int gi = lane & 7, q4 = lane >> 3;
            const int t0 = 16 * warp + 4 * q4;
            uint32_t hh[4], bb[4];  // hist(t0 + i), B sums
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint4* c = reinterpret_cast<uint4*>(hist + (t0 + i) * 256 + 128 + gi * 16);
                const uint4 v = *c;
                *c = make_uint4(0, 0, 0, 0);
                hh[i] = (v.x & 0xFFFFu) + (v.y & 0xFFFFu) + (v.z & 0xFFFFu) + (v.w & 0xFFFFu);
                bb[i] = (v.x >> 16) + (v.y >> 16) + (v.z >> 16) + (v.w >> 16);
            }
            // Hs rows 2 t0 - 1 + i: the eight rows whose terms all fall on this
            // lane's keys t0 .. t0 + 3 or -- the last two -- on key t0 + 4 (below).
            // Row -1 does not exist; row 511 (the dummy row of neutralised
            // events) is never read, so it needs no clearing either.
            uint32_t hs[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 2 * t0 - 1 + i;
                hs[i] = 0u;
                if (r >= 0) {
                    uint4* c = reinterpret_cast<uint4*>(hist + r * 256 + gi * 16);
                    const uint4 v = *c;
                    *c = make_uint4(0, 0, 0, 0);
                    hs[i] = v.x + v.y + v.z + v.w;
                }
            }
            int crv[4];  // corr(t0 + i): the lane-striped second W copy
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint4* c = reinterpret_cast<uint4*>(hist + (256 + t0 + i) * 256 + 128 + gi * 16);
                const uint4 v = *c;
                *c = make_uint4(0, 0, 0, 0);
                crv[i] = (int)(v.x + v.y + v.z + v.w);
            }
            // h2(u) = 4 hist(u-1) - corr(u-1) - Hs(2u-3) - 2 Hs(2u-2) - Hs(2u-1).
            // With the rows above a lane holds every term of h2(t0+1 .. t0+3),
            // the Hs(2 t0 - 1) term of h2(t0), and all other terms of the NEXT
            // lane's first key, h2(t0+4) -- its "deferred" part dA.  Everything
            // downstream is a prefix scan, and a term of key t0 + 4 acts on
            // exactly the keys of the later lanes: dA joins this lane's scan
            // TOTAL but not its own elements, and no lane needs another lane's
            // counters (no hand-off, no barrier before the scans).
            long long cd[4], h2[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                cd[i] = (long long)bb[i] - 4ll * (long long)hh[i];
            h2[0] = -(long long)hs[0];
            h2[1] = 4ll * hh[0] - (long long)crv[0] - (long long)hs[0] - 2ll * hs[1] - (long long)hs[2];
            h2[2] = 4ll * hh[1] - (long long)crv[1] - (long long)hs[2] - 2ll * hs[3] - (long long)hs[4];
            h2[3] = 4ll * hh[2] - (long long)crv[2] - (long long)hs[4] - 2ll * hs[5] - (long long)hs[6];
            const long long dA = 4ll * hh[3] - (long long)crv[3] - (long long)hs[6] - 2ll * hs[7];
            // scans: lane-local, then across the image's 4 lanes (a quad);
            // `extra` counts in the lane's total only
            long long* tot = reinterpret_cast<long long*>(sm + Lay::kTot);  // [3][16][NG]
            auto quad_scan = [&](long long (&v)[4], long long extra) -> long long {
#pragma unroll
                for (int i = 1; i < 4; ++i)
                    v[i] += v[i - 1];
                const long long own = v[3] + extra;
                long long x = own;  // the image's 4 lanes are gi, gi + 8, gi + 16, gi + 24
#pragma unroll
                for (int off = 1; off < 4; off <<= 1) {
                    const long long y = __shfl_up_sync(0xFFFFFFFFu, x, 8 * off);
                    if (q4 >= off)
                        x += y;
                }
                const long long ex = x - own;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    v[i] += ex;
                return __shfl_sync(0xFFFFFFFFu, x, 24 + gi);  // the image's (= warp's) total
            };
            const long long tc = quad_scan(cd, 0);
            const long long tg = quad_scan(h2, dA);  // h2 -> g, local to the warp's 16 keys
            const long long tsl = quad_scan(h2, 0);  // g -> sum, local too (earlier warps enter below)
            if (q4 == 0) {
                tot[(0 * 16 + warp) * NG + gi] = tc;
                tot[(1 * 16 + warp) * NG + gi] = tg;
                tot[(2 * 16 + warp) * NG + gi] = tsl;
            }
            __syncthreads();
            // The earlier warps' part, from their totals alone (one exchange, no
            // third barrier): with cg = sum of earlier tg, key k of the warp has
            //   g[k]   = g_local[k] + cg
            //   sum[k] = sum_local[k] + (k + 1) cg + cs,
            //   cs     = sum over earlier warps w' of (tsl(w') + 16 cg(w'))
            //          = sum over w' < w of (tsl(w') + 16 (w - 1 - w') tg(w')).
            // The image's 4 lanes (q4) load 4 warps' totals each, independent
            // loads, then two shuffles (a serial 15-load chain made warp 15
            // the round's straggler at the final barrier).
            long long cc = 0, cg = 0, cs = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int w2 = 4 * q4 + i;
                if (w2 < warp) {
                    const long long g2 = tot[(1 * 16 + w2) * NG + gi];
                    cc += tot[(0 * 16 + w2) * NG + gi];
                    cg += g2;
                    cs += tot[(2 * 16 + w2) * NG + gi] + 16ll * (long long)(warp - 1 - w2) * g2;
                }
            }
            cc += __shfl_xor_sync(0xFFFFFFFFu, cc, 8);
            cg += __shfl_xor_sync(0xFFFFFFFFu, cg, 8);
            cs += __shfl_xor_sync(0xFFFFFFFFu, cs, 8);
            cc += __shfl_xor_sync(0xFFFFFFFFu, cc, 16);
            cg += __shfl_xor_sync(0xFFFFFFFFu, cg, 16);
            cs += __shfl_xor_sync(0xFFFFFFFFu, cs, 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                cd[i] += cc;                                      // card
                h2[i] += (long long)(4 * q4 + i + 1) * cg + cs;  // sum
            }
            const long long im = i0 + gi;
            if (im < p.n) {
                // 64-bit stores straight from the register pairs: STG.128 made
                // ptxas funnel all four through one register quad, each waiting
                // for the previous store to release it (long-scoreboard stalls)
                uint64_t* os = p.sums + (size_t)im * 256 + t0;
                uint64_t* oc = p.cards + (size_t)im * 256 + t0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    oc[i] = (uint64_t)cd[i];
                    os[i] = (uint64_t)h2[i];
                }
                if (p.hist_out) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        p.hist_out[(size_t)im * 256 + t0 + i] = hh[i];
                }
            }
            TWCYC(1);
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
            //    x + x/8 (conflict-free lane-blocked reads of warp_curve256_regs)
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
                const int* cr = reinterpret_cast<const int*>(sm + Lay::kCorr + warp * kTwCorrStride);
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
            for (int i = tid; i < NG * (int)(kTwCorrStride / 4); i += kTwThreads)
                reinterpret_cast<int*>(sm + Lay::kCorr)[i] = 0;
        }
        // LG = 4 needs no barrier here: every counter piece was cleared before
        // the totals barrier, and the next round writes the totals only behind
        // its walk-end barrier, which every warp reaches after this round's
        // last read of them; a warp done with its stores starts the next
        // round's walk while the others finish theirs
        if constexpr (LG != 4)
            __syncthreads();
        TWCYC(4);
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

} // namespace

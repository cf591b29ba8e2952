// C++ test of the drop-in (libkohler_b200.so) through the reference's own
// headers-compatible API, on the GPU: the hand-derived cases of
// proj/tests/test_contrast.cpp:32-123 and test_threshold.cpp:50-183, the
// exception contract (contrast.hpp:13-18, threshold.hpp:50-60, curve.cpp:18-19),
// worker / repeat determinism, and seeded images against the oracle's C
// restatement (oracle/kohler_oracle.c: test infrastructure, linked only here).
// Built and run by tests/test_dropin_cpp.py; prints "PASS <n>" or exits 1.
#include <cstdint>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "kohler/contrast.hpp"
#include "kohler/curve.hpp"
#include "kohler/image.hpp"
#include "kohler/stream.hpp"
#include "kohler/threshold.hpp"

extern "C" void oracle_fast_curve(const uint8_t* px, int w, int h, uint64_t* sum, uint64_t* card);

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
        }                                                                         \
    } while (0)

template <class E, class F>
static bool throws(F f)
{
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main()
{
    using namespace kohler;
    // [2, 5] column: card = 1 at t in {2,3,4}, sum = {0,1,1}
    {
        const GrayImage img(1, 2, std::vector<std::uint8_t>{2, 5});
        const ContrastCurve c = fast_contrast_curve(img, 1);
        for (int t = 0; t < 256; ++t) {
            CHECK(c.cardinality[t] == ((t >= 2 && t <= 4) ? 1u : 0u));
            CHECK(c.contrast_sum[t] == ((t == 3 || t == 4) ? 1u : 0u));
        }
        CHECK(c == direct_contrast_curve(img));
        CHECK(optimal_threshold(mean_contrast(c)) == 3);
    }
    // 2x2 checker: card 4, sum 4 min(t, 255 - t), t0 = 127
    {
        const GrayImage img(2, 2, std::vector<std::uint8_t>{0, 255, 255, 0});
        const ContrastCurve c = fast_contrast_curve(img, 2);
        for (int t = 0; t < 256; ++t) {
            CHECK(c.cardinality[t] == (t <= 254 ? 4u : 0u));
            CHECK(c.contrast_sum[t] == (t <= 254 ? 4u * (std::uint64_t)std::min(t, 255 - t) : 0u));
        }
        CHECK(c.contrast_sum[127] == 508u);
        const MeanContrastCurve mc = mean_contrast(c);
        CHECK(optimal_threshold(mc) == 127);
        CHECK(top_k_local_maxima(mc, 1).thresholds == std::vector<int>{127});
    }
    // (0, 255) pair: total 16256
    {
        ContrastCurve acc;
        pair_contribution(0, 255, acc);
        std::uint64_t tot = 0;
        for (auto v : acc.contrast_sum)
            tot += v;
        CHECK(tot == 16256u);
    }
    // empty boundary: zero curve, NoBoundaryError from both selectors
    {
        const GrayImage flat(5, 4, 100);
        const ContrastCurve c = fast_contrast_curve(flat);
        CHECK(c == ContrastCurve());
        const MeanContrastCurve mc = mean_contrast(c);
        CHECK(throws<NoBoundaryError>([&] { (void)optimal_threshold(mc); }));
        CHECK(throws<NoBoundaryError>([&] { (void)top_k_local_maxima(mc, 3); }));
    }
    // exception contract
    {
        const GrayImage img(3, 3, 7);
        CHECK(throws<std::invalid_argument>([&] { (void)fast_contrast_curve(img, 0); }));
        MeanContrastCurve mc;
        mc.values.assign(256, 1.0);
        mc.defined.assign(256, true);
        CHECK(throws<std::invalid_argument>([&] { (void)top_k_local_maxima(mc, 0); }));
        CHECK(throws<std::invalid_argument>([&] { (void)merge_accumulators({}); }));
        CHECK(throws<std::invalid_argument>([&] { (void)GrayImage(0, 3); }));
    }
    // plateau rule: equal-valued runs collapse, maxima strictly above both neighbours
    {
        MeanContrastCurve mc;
        mc.values.assign(256, 0.0);
        mc.defined.assign(256, false);
        const int ts[] = {10, 11, 12, 20, 30, 31};
        const double vs[] = {5.0, 5.0, 5.0, 3.0, 9.0, 9.0};
        for (int i = 0; i < 6; ++i) {
            mc.values[ts[i]] = vs[i];
            mc.defined[ts[i]] = true;
        }
        CHECK(optimal_threshold(mc) == 30);
        CHECK(top_k_local_maxima(mc, 5).thresholds == (std::vector<int>{10, 30}));
        CHECK(top_k_local_maxima(mc, 1).thresholds == std::vector<int>{30});
    }
    // seeded images (the reference generator's distributions) vs the oracle;
    // every workers value gives the identical curve; repeats are identical
    std::mt19937 rng(20240811);
    for (int i = 0; i < 60; ++i) {
        const int w = 1 + (int)(rng() % 97), h = 1 + (int)(rng() % 61);
        std::vector<std::uint8_t> px((std::size_t)w * h);
        const int dist = i % 4;
        const std::uint8_t a = (std::uint8_t)(rng() & 255), b = (std::uint8_t)(rng() & 255);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                std::uint8_t v;
                if (dist == 0)
                    v = (std::uint8_t)(rng() & 255);
                else if (dist == 1)
                    v = (rng() & 1) ? a : b;
                else if (dist == 2)
                    v = a;
                else
                    v = (std::uint8_t)((x * 7 + y * 3) & 255);
                px[(std::size_t)y * w + x] = v;
            }
        const GrayImage img(w, h, px);
        std::vector<std::uint64_t> s(256), c(256);
        oracle_fast_curve(px.data(), w, h, s.data(), c.data());
        const ContrastCurve g = fast_contrast_curve(img, 1 + (unsigned)(i % 5));
        CHECK(g.contrast_sum == s && g.cardinality == c);
        CHECK(fast_contrast_curve(img, 7) == g);
        CHECK(direct_contrast_curve(img) == g);
    }
    // FrameStream (two frames in flight) == the synchronous functions
    {
        std::vector<GrayImage> frames;
        for (int f = 0; f < 6; ++f) {
            const int w = 640 + 16 * f, h = 360;
            std::vector<std::uint8_t> px((std::size_t)w * h);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    px[(std::size_t)y * w + x] =
                        (std::uint8_t)(((x / (40 + f)) + (y / 30)) % 2 ? 200 : 40) + (std::uint8_t)(rng() % 7);
            frames.emplace_back(w, h, px);
        }
        frames.emplace_back(64, 48, 9);  // no boundary
        b200::FrameStream fs(6);
        std::vector<b200::FrameResult> got;
        long long prev = fs.submit(frames[0]);
        for (std::size_t f = 1; f < frames.size(); ++f) {
            const long long t = fs.submit(frames[f]);
            got.push_back(fs.collect(prev));
            prev = t;
        }
        got.push_back(fs.collect(prev));
        for (std::size_t f = 0; f < frames.size(); ++f) {
            const ContrastCurve c = fast_contrast_curve(frames[f]);
            CHECK(got[f].curve == c);
            const MeanContrastCurve mc = mean_contrast(c);
            CHECK(got[f].mean.values == mc.values && got[f].mean.defined == mc.defined);
            if (got[f].has_boundary) {
                CHECK(got[f].optimal_threshold == optimal_threshold(mc));
                CHECK(got[f].top_k == top_k_local_maxima(mc, 6));
            } else {
                CHECK(throws<NoBoundaryError>([&] { (void)optimal_threshold(mc); }));
            }
        }
        CHECK(!got.back().has_boundary);
        const long long a = fs.submit(frames[0]);
        const long long b = fs.submit(frames[1]);
        CHECK(throws<std::invalid_argument>([&] { (void)fs.submit(frames[2]); }));
        (void)fs.collect(a);
        (void)b;  // left in flight: the destructor drains it
    }
    if (g_fail) {
        std::fprintf(stderr, "%d of %d checks failed\n", g_fail, g_checks);
        return 1;
    }
    std::printf("PASS %d\n", g_checks);
    return 0;
}

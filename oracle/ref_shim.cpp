// ref_shim.cpp — C entry points over the reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  TEST INFRASTRUCTURE ONLY:
// used by tests/ to pin the oracle and the CUDA path against the reference
// itself, and by bench.py's CPU-baseline / `--impl reference` legs to time
// the reference's own fast path on the host cores.
//
// The reference is built with -Dkohler=kohler_ref so that it can share a
// process with the drop-in library, which defines kohler::fast_contrast_curve.
// Header names in #include are not macro-expanded, so "kohler/…" still
// resolves to the reference's headers.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "kohler/contrast.hpp"
#include "kohler/curve.hpp"
#include "kohler/image.hpp"
#include "kohler/kernels.hpp"
#include "kohler/pnm.hpp"
#include "kohler/threshold.hpp"

namespace {

enum Status { kOk = 0, kNoBoundary = 1, kInvalidArgument = 2, kOther = 3 };

kohler::MeanContrastCurve to_mc(const double* values, const uint8_t* defined, int n)
{
    kohler::MeanContrastCurve mc;
    mc.values.assign(values, values + n);
    mc.defined.resize(static_cast<std::size_t>(n));
    for (int t = 0; t < n; ++t)
        mc.defined[t] = defined[t] != 0;
    return mc;
}

struct PipelineOut {
    uint64_t* sum;
    uint64_t* card;
    double* values;
    uint8_t* defined;
    int* t0;
    int* topk;
    int* topk_count;
};

// The per-image timed section: curve -> mean curve -> t0 -> top-k
// (proj/src/bench.cpp:174-181 plus the O(256) selection of
// proj/tools/kohler_main.cpp:95-105).
int pipeline(const kohler::GrayImage& img, unsigned workers, int k, const PipelineOut& o)
{
    const kohler::ContrastCurve c = kohler::fast_contrast_curve(img, workers);
    const kohler::MeanContrastCurve mc = kohler::mean_contrast(c);
    if (o.sum) {
        std::memcpy(o.sum, c.contrast_sum.data(), 256 * sizeof(uint64_t));
        std::memcpy(o.card, c.cardinality.data(), 256 * sizeof(uint64_t));
    }
    if (o.values) {
        for (int t = 0; t < 256; ++t) {
            o.values[t] = mc.values[t];
            o.defined[t] = mc.defined[t] ? 1 : 0;
        }
    }
    try {
        const int t0 = kohler::optimal_threshold(mc);
        const kohler::ThresholdSet ts = kohler::top_k_local_maxima(mc, k);
        if (o.t0)
            *o.t0 = t0;
        if (o.topk) {
            *o.topk_count = static_cast<int>(ts.thresholds.size());
            std::copy(ts.thresholds.begin(), ts.thresholds.end(), o.topk);
        }
        return kOk;
    } catch (const kohler::NoBoundaryError&) {
        if (o.t0)
            *o.t0 = -1;
        if (o.topk_count)
            *o.topk_count = 0;
        return kNoBoundary;
    }
}

} // namespace

extern "C" {

const char* kref_active_kernel() { return kohler::kernels::active().name.data(); }

void* kref_image_new(const uint8_t* px, int w, int h)
{
    try {
        std::vector<std::uint8_t> v(px, px + static_cast<std::size_t>(w) * static_cast<std::size_t>(h));
        return new kohler::GrayImage(w, h, std::move(v));
    } catch (...) {
        return nullptr;
    }
}

void kref_image_free(void* img) { delete static_cast<kohler::GrayImage*>(img); }

int kref_fast_curve(const void* img, unsigned workers, uint64_t* sum, uint64_t* card)
{
    try {
        const auto c = kohler::fast_contrast_curve(*static_cast<const kohler::GrayImage*>(img), workers);
        std::memcpy(sum, c.contrast_sum.data(), 256 * sizeof(uint64_t));
        std::memcpy(card, c.cardinality.data(), 256 * sizeof(uint64_t));
        return kOk;
    } catch (const std::invalid_argument&) {
        return kInvalidArgument;
    }
}

int kref_direct_curve(const void* img, uint64_t* sum, uint64_t* card)
{
    const auto c = kohler::direct_contrast_curve(*static_cast<const kohler::GrayImage*>(img));
    std::memcpy(sum, c.contrast_sum.data(), 256 * sizeof(uint64_t));
    std::memcpy(card, c.cardinality.data(), 256 * sizeof(uint64_t));
    return kOk;
}

void kref_pair_contribution(int lo, int hi, uint64_t* sum, uint64_t* card)
{
    kohler::ContrastCurve acc;
    kohler::pair_contribution(static_cast<std::uint8_t>(lo), static_cast<std::uint8_t>(hi), acc);
    std::memcpy(sum, acc.contrast_sum.data(), 256 * sizeof(uint64_t));
    std::memcpy(card, acc.cardinality.data(), 256 * sizeof(uint64_t));
}

void kref_mean_contrast(const uint64_t* sum, const uint64_t* card, int n, double* values,
                        uint8_t* defined)
{
    kohler::ContrastCurve c(n);
    std::copy(sum, sum + n, c.contrast_sum.begin());
    std::copy(card, card + n, c.cardinality.begin());
    const auto mc = kohler::mean_contrast(c);
    for (int t = 0; t < n; ++t) {
        values[t] = mc.values[t];
        defined[t] = mc.defined[t] ? 1 : 0;
    }
}

int kref_optimal_threshold(const double* values, const uint8_t* defined, int n, int* t0)
{
    try {
        *t0 = kohler::optimal_threshold(to_mc(values, defined, n));
        return kOk;
    } catch (const kohler::NoBoundaryError&) {
        *t0 = -1;
        return kNoBoundary;
    }
}

int kref_top_k(const double* values, const uint8_t* defined, int n, int k, int* out, int* count)
{
    *count = 0;
    try {
        const auto ts = kohler::top_k_local_maxima(to_mc(values, defined, n), k);
        *count = static_cast<int>(ts.thresholds.size());
        std::copy(ts.thresholds.begin(), ts.thresholds.end(), out);
        return kOk;
    } catch (const kohler::NoBoundaryError&) {
        return kNoBoundary;
    } catch (const std::invalid_argument&) {
        return kInvalidArgument;
    }
}

int kref_pipeline(const void* img, unsigned workers, int k, uint64_t* sum, uint64_t* card,
                  double* values, uint8_t* defined, int* t0, int* topk, int* topk_count)
{
    return pipeline(*static_cast<const kohler::GrayImage*>(img), workers, k,
                    {sum, card, values, defined, t0, topk, topk_count});
}

// Batch of images.  threads == 1: "as shipped", sequential per-image calls
// with `workers` threads each (proj/src/bench.cpp:263-277).  threads > 1:
// frame-parallel, `threads` host threads pulling images, each call using
// `workers` (normally 1).  Outputs are per image (256 u64 / int per image,
// k ints of top-k); any may be null.  Returns the number of no-boundary images.
int kref_pipeline_batch(void* const* imgs, int n, unsigned workers, int threads, int k,
                        uint64_t* sums, uint64_t* cards, int* t0s, int* topks, int* topk_counts)
{
    std::atomic<int> next{0}, no_boundary{0};
    auto body = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n)
                return;
            PipelineOut o{sums ? sums + 256 * (std::size_t)i : nullptr,
                          cards ? cards + 256 * (std::size_t)i : nullptr,
                          nullptr,
                          nullptr,
                          t0s ? t0s + i : nullptr,
                          topks ? topks + (std::size_t)k * i : nullptr,
                          topk_counts ? topk_counts + i : nullptr};
            if (pipeline(*static_cast<const kohler::GrayImage*>(imgs[i]), workers, k, o) ==
                kNoBoundary)
                no_boundary.fetch_add(1);
        }
    };
    if (threads <= 1) {
        body();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back(body);
        for (auto& th : pool)
            th.join();
    }
    return no_boundary.load();
}

// Median wall time (steady_clock) of `runs` pipeline calls after `warmup`
// untimed ones — the reference bench's timing method
// (proj/src/bench.cpp:30-35,171-185).
double kref_time_pipeline(const void* img, unsigned workers, int k, int warmup, int runs)
{
    const auto& image = *static_cast<const kohler::GrayImage*>(img);
    PipelineOut o{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    for (int i = 0; i < warmup; ++i)
        pipeline(image, workers, k, o);
    std::vector<double> t;
    for (int i = 0; i < runs; ++i) {
        const auto a = std::chrono::steady_clock::now();
        pipeline(image, workers, k, o);
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    }
    std::sort(t.begin(), t.end());
    if (t.empty())
        return 0.0;
    return t.size() % 2 ? t[t.size() / 2] : 0.5 * (t[t.size() / 2 - 1] + t[t.size() / 2]);
}

} // extern "C"

extern "C" {

// classify / quantize (proj/src/threshold.cpp:84-126) with a given set of
// thresholds (sorted, as a ThresholdSet holds them).
void kref_classify(const void* img, const int* ts, int nts, uint8_t* labels)
{
    kohler::ThresholdSet s;
    s.thresholds.assign(ts, ts + nts);
    const auto l = kohler::classify(*static_cast<const kohler::GrayImage*>(img), s);
    std::copy(l.labels.begin(), l.labels.end(), labels);
}

void kref_quantize(const void* img, const int* ts, int nts, uint8_t* out)
{
    kohler::ThresholdSet s;
    s.thresholds.assign(ts, ts + nts);
    const auto q = kohler::quantize(*static_cast<const kohler::GrayImage*>(img), s);
    const auto px = q.pixels();
    std::copy(px.begin(), px.end(), out);
}

// One video frame of proj/src/bench.cpp:266-281: curve -> mean -> {t0} ->
// two-class quantize; a frame without boundary passes through unchanged.
// k > 0: the segment command's top-k thresholds (tools/kohler_main.cpp:95-103)
// instead of {t0}.  Returns 1 for a frame without boundary, else 0.
int kref_segment(const void* img, unsigned workers, int k, uint8_t* out, int* ts_out,
                 int* ts_count)
{
    const auto& im = *static_cast<const kohler::GrayImage*>(img);
    const kohler::ContrastCurve c = kohler::fast_contrast_curve(im, workers);
    *ts_count = 0;
    try {
        const kohler::MeanContrastCurve mc = kohler::mean_contrast(c);
        kohler::ThresholdSet ts;
        if (k <= 0)
            ts.thresholds.push_back(kohler::optimal_threshold(mc));
        else
            ts = kohler::top_k_local_maxima(mc, k);
        const auto q = kohler::quantize(im, ts);
        const auto px = q.pixels();
        std::copy(px.begin(), px.end(), out);
        *ts_count = static_cast<int>(ts.thresholds.size());
        std::copy(ts.thresholds.begin(), ts.thresholds.end(), ts_out);
        return 0;
    } catch (const kohler::NoBoundaryError&) {
        const auto px = im.pixels();
        std::copy(px.begin(), px.end(), out);
        return 1;
    }
}

// The reference's PNM decoder (proj/src/pnm.cpp:87-139): pins the colour
// ingest (luma601 on P6 / P3) of the CUDA path.  0 ok, 2 on a PnmError or if
// the image does not fit `cap` bytes.
int kref_read_pnm(const uint8_t* bytes, size_t n, uint8_t* out, size_t cap, int* w, int* h)
{
    try {
        const kohler::GrayImage im = kohler::read_pnm(std::span<const std::uint8_t>(bytes, n));
        const auto px = im.pixels();
        if (px.size() > cap)
            return 2;
        std::copy(px.begin(), px.end(), out);
        *w = im.width();
        *h = im.height();
        return 0;
    } catch (const std::exception&) {
        return 2;
    }
}

} // extern "C"

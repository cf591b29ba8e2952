// kohler_dropin.cpp — the C++ drop-in (libkohler_b200.so) over the C ABI.
//
// Implements the reference's hot-path API (proj/include/kohler/contrast.hpp:11,18
// and threshold.hpp:50-60) with the same signatures, argument meaning and
// exception behaviour, computing on the B200 through kohler_cuda.h:
//   fast_contrast_curve   -> kohler_cuda_curve          (ref src/fast.cpp:36-62)
//   direct_contrast_curve -> kohler_cuda_direct_curve   (ref src/direct.cpp:10-43)
//   mean_contrast         -> kohler_cuda_mean_contrast  (ref src/threshold.cpp:9-23)
//   optimal_threshold     -> kohler_cuda_optimal_threshold (ref :25-37)
//   top_k_local_maxima    -> kohler_cuda_top_k_local_maxima (ref :39-82)
//   classify              -> kohler_cuda_classify       (ref :84-101)
//   quantize              -> kohler_cuda_quantize       (ref :103-126)
// pair_contribution / merge_accumulators are the reference's tiny host
// utilities (ref src/curve.cpp:10-30) and stay on the host.
//
// One process-wide context on device $KOHLER_CUDA_DEVICE (default 0) is
// created on first use; calls are serialised on it, so concurrent callers are
// safe and get identical results.  No CPU fallback: failures throw.
//
// Multi-GPU: with $KOHLER_CUDA_DEVICES set (a comma-separated device list,
// e.g. "0,1,2,3"), fast_contrast_curve runs over that device group instead:
// the reference's row-block split over the GPUs (src/fast.cpp:42-61; one band
// per device instead of one per worker thread) with the band partials merged
// by one NCCL all-reduce (kohler_cuda_multi_curve).  The result is the same
// integer curve for any split, exactly as the reference's is for any
// `workers`.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kohler/contrast.hpp"
#include "kohler/curve.hpp"
#include "kohler/image.hpp"
#include "kohler/stream.hpp"
#include "kohler/threshold.hpp"
#include "kohler_cuda.h"

namespace kohler {

namespace {

kohler_cuda_ctx* context()
{
    static std::once_flag once;
    static kohler_cuda_ctx* ctx = nullptr;
    static std::string error;
    std::call_once(once, [] {
        int dev = 0;
        if (const char* env = std::getenv("KOHLER_CUDA_DEVICE"))
            dev = std::atoi(env);
        if (kohler_cuda_create(dev, &ctx) != KOHLER_OK) {
            error = std::string("kohler: no usable B200 device: ") + kohler_cuda_last_error();
            ctx = nullptr;
        }
    });
    if (!ctx)
        throw std::runtime_error(error);
    return ctx;
}

// The device group of $KOHLER_CUDA_DEVICES, or null when it is unset.
kohler_cuda_multi* group()
{
    static std::once_flag once;
    static kohler_cuda_multi* g = nullptr;
    static std::string error;
    std::call_once(once, [] {
        const char* env = std::getenv("KOHLER_CUDA_DEVICES");
        if (!env || !*env)
            return;
        std::vector<int> devs;
        for (const char* p = env; *p;) {
            char* end = nullptr;
            const long d = std::strtol(p, &end, 10);
            if (end == p) {
                error = std::string("kohler: bad KOHLER_CUDA_DEVICES '") + env + "'";
                return;
            }
            devs.push_back((int)d);
            p = *end == ',' ? end + 1 : end;
        }
        if (kohler_cuda_multi_create(devs.data(), (int)devs.size(), &g) != KOHLER_OK) {
            error = std::string("kohler: device group ") + env + ": " + kohler_cuda_last_error();
            g = nullptr;
        }
    });
    if (!g && !error.empty())
        throw std::runtime_error(error);
    return g;
}

// Status -> the reference's exception types.
void raise_for(int status)
{
    switch (status) {
    case KOHLER_OK:
        return;
    case KOHLER_NO_BOUNDARY:
        throw NoBoundaryError{};
    case KOHLER_INVALID_ARGUMENT:
        throw std::invalid_argument(kohler_cuda_last_error());
    default:
        throw std::runtime_error(std::string("kohler (CUDA): ") + kohler_cuda_last_error());
    }
}

struct FlatMean {
    std::vector<double> values;
    std::vector<std::uint8_t> defined;
    explicit FlatMean(const MeanContrastCurve& mc)
        : values(mc.values), defined(mc.defined.size())
    {
        for (std::size_t t = 0; t < defined.size(); ++t)
            defined[t] = mc.defined[t] ? 1 : 0;
    }
};

} // namespace

void pair_contribution(std::uint8_t lo, std::uint8_t hi, ContrastCurve& acc)
{
    for (int t = lo; t < hi; ++t) {
        const int up = t - lo, down = hi - t;
        acc.contrast_sum[t] += static_cast<std::uint64_t>(up < down ? up : down);
        acc.cardinality[t] += 1;
    }
}

ContrastCurve merge_accumulators(std::span<const ContrastCurve> parts)
{
    if (parts.empty())
        throw std::invalid_argument("merge_accumulators: no partial results");
    ContrastCurve out(parts[0].levels());
    for (const ContrastCurve& p : parts) {
        if (p.levels() != out.levels())
            throw std::invalid_argument("merge_accumulators: mismatched curve lengths");
        for (int t = 0; t < out.levels(); ++t) {
            out.contrast_sum[t] += p.contrast_sum[t];
            out.cardinality[t] += p.cardinality[t];
        }
    }
    return out;
}

ContrastCurve fast_contrast_curve(const GrayImage& img, unsigned workers)
{
    if (workers < 1)
        throw std::invalid_argument("fast_contrast_curve: workers must be at least 1");
    ContrastCurve curve;
    if (kohler_cuda_multi* g = group()) {
        raise_for(kohler_cuda_multi_curve(g, img.row(0), img.width(), img.height(),
                                          static_cast<std::size_t>(img.width()),
                                          curve.contrast_sum.data(), curve.cardinality.data()));
        return curve;
    }
    raise_for(kohler_cuda_curve(context(), img.row(0), img.width(), img.height(),
                                static_cast<std::size_t>(img.width()),
                                curve.contrast_sum.data(), curve.cardinality.data()));
    return curve;
}

ContrastCurve direct_contrast_curve(const GrayImage& img)
{
    ContrastCurve curve;
    raise_for(kohler_cuda_direct_curve(context(), img.row(0), img.width(), img.height(),
                                       static_cast<std::size_t>(img.width()),
                                       curve.contrast_sum.data(), curve.cardinality.data()));
    return curve;
}

MeanContrastCurve mean_contrast(const ContrastCurve& curve)
{
    const int n = curve.levels();
    MeanContrastCurve mc;
    mc.values.assign(static_cast<std::size_t>(n), 0.0);
    std::vector<std::uint8_t> def(static_cast<std::size_t>(n), 0);
    if (n > 0)
        raise_for(kohler_cuda_mean_contrast(context(), curve.contrast_sum.data(),
                                            curve.cardinality.data(), n, mc.values.data(),
                                            def.data()));
    mc.defined.assign(def.begin(), def.end());
    return mc;
}

int optimal_threshold(const MeanContrastCurve& mc)
{
    const FlatMean f(mc);
    if (f.values.empty())
        throw NoBoundaryError{};
    int t0 = -1;
    raise_for(kohler_cuda_optimal_threshold(context(), f.values.data(), f.defined.data(),
                                            static_cast<int>(f.values.size()), &t0));
    return t0;
}

ThresholdSet top_k_local_maxima(const MeanContrastCurve& mc, int k)
{
    if (k < 1)
        throw std::invalid_argument("top_k_local_maxima: k must be at least 1");
    const FlatMean f(mc);
    if (f.values.empty())
        throw NoBoundaryError{};
    // at most levels maxima exist: a huge k means "all of them", cheaply
    k = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(k), f.values.size()));
    std::vector<int> out(static_cast<std::size_t>(k));
    int count = 0;
    raise_for(kohler_cuda_top_k_local_maxima(context(), f.values.data(), f.defined.data(),
                                             static_cast<int>(f.values.size()), k, out.data(),
                                             &count));
    out.resize(static_cast<std::size_t>(count));
    return ThresholdSet{std::move(out)};
}

LabelImage classify(const GrayImage& img, const ThresholdSet& ts)
{
    LabelImage out{img.width(), img.height(), {}};
    out.labels.resize(img.pixel_count());
    const auto px = img.pixels();
    raise_for(kohler_cuda_classify(context(), px.data(), img.width(), img.height(),
                                   static_cast<std::size_t>(img.width()), ts.thresholds.data(),
                                   static_cast<int>(ts.thresholds.size()), out.labels.data()));
    return out;
}

GrayImage quantize(const GrayImage& img, const ThresholdSet& ts)
{
    GrayImage out(img.width(), img.height());
    const auto px = img.pixels();
    raise_for(kohler_cuda_quantize(context(), px.data(), img.width(), img.height(),
                                   static_cast<std::size_t>(img.width()), ts.thresholds.data(),
                                   static_cast<int>(ts.thresholds.size()), out.pixels().data()));
    return out;
}

namespace b200 {

// the frame a ticket borrows (kept alive by the caller until collect)
struct FrameStream::Slot {
    long long ticket;
};

FrameStream::FrameStream(int k) : k_(k)
{
    if (k < 1)
        throw std::invalid_argument("top_k_local_maxima: k must be at least 1");
}

FrameStream::~FrameStream()
{
    for (Slot* s : slots_) {  // drain what was never collected
        kohler_cuda_collect(context(), s->ticket, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, nullptr);
        delete s;
    }
}

long long FrameStream::submit(const GrayImage& frame)
{
    long long t = -1;
    raise_for(kohler_cuda_submit(context(), frame.row(0), 1, frame.width(), frame.height(),
                                 static_cast<std::size_t>(frame.width()), 0, k_, &t));
    slots_.push_back(new Slot{t});
    return t;
}

FrameResult FrameStream::collect(long long ticket)
{
    FrameResult r;
    std::vector<double> vals(256);
    std::vector<std::uint8_t> def(256);
    std::vector<int> topk(static_cast<std::size_t>(k_));
    int t0 = -1, cnt = 0, status = 0;
    raise_for(kohler_cuda_collect(context(), ticket, r.curve.contrast_sum.data(),
                                  r.curve.cardinality.data(), vals.data(), def.data(), &t0,
                                  topk.data(), &cnt, &status));
    for (std::size_t i = 0; i < slots_.size(); ++i)
        if (slots_[i]->ticket == ticket) {
            delete slots_[i];
            slots_.erase(slots_.begin() + static_cast<std::ptrdiff_t>(i));
            break;
        }
    r.mean.values = vals;
    r.mean.defined.resize(256);
    for (int t = 0; t < 256; ++t)
        r.mean.defined[t] = def[t] != 0;
    r.has_boundary = status == KOHLER_OK;
    r.optimal_threshold = r.has_boundary ? t0 : -1;
    if (r.has_boundary)
        r.top_k.thresholds.assign(topk.begin(), topk.begin() + cnt);
    return r;
}

} // namespace b200

} // namespace kohler

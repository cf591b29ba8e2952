// kohler/stream.hpp — B200 extension (no reference counterpart): a frame loop
// at PCIe speed.
//
// The reference's per-frame loops (proj/src/bench.cpp:264-284, the CLI's
// video command) call fast_contrast_curve + mean_contrast + selection once
// per frame; each call returns before the next upload starts.  FrameStream
// keeps two frames in flight on the GPU (kohler_cuda_submit /
// kohler_cuda_collect): frame i + 1 uploads while frame i's kernels and
// copy-back run, so a loop over frames runs at the host-to-device copy rate.
// Results are identical to the synchronous functions.
#pragma once

#include <cstdint>
#include <vector>

#include "kohler/curve.hpp"
#include "kohler/image.hpp"
#include "kohler/threshold.hpp"

namespace kohler::b200 {

struct FrameResult {
    ContrastCurve curve;
    MeanContrastCurve mean;
    bool has_boundary = false;  // false: no boundary (optimal_threshold would throw)
    int optimal_threshold = -1;
    ThresholdSet top_k;         // the k most significant local maxima, ascending
};

class FrameStream {
public:
    /// k: maxima per frame (>= 1, else std::invalid_argument).
    explicit FrameStream(int k = 6);
    ~FrameStream();
    FrameStream(const FrameStream&) = delete;
    FrameStream& operator=(const FrameStream&) = delete;

    /// Enqueue a frame (borrowed until the matching collect()); returns its
    /// ticket.  At most two frames may be in flight: a third submit throws
    /// std::invalid_argument until the oldest has been collected.
    long long submit(const GrayImage& frame);
    /// Wait for `ticket` and return its results.
    FrameResult collect(long long ticket);

private:
    int k_;
    struct Slot;
    std::vector<Slot*> slots_;
};

} // namespace kohler::b200

// kohler/contrast.hpp — B200 drop-in: whole-image contrast curves.
//
// Source-compatible with proj/include/kohler/contrast.hpp:8-18.  Both
// functions run on the GPU through the C ABI in kohler_cuda.h; there is no
// CPU fallback (a missing or unusable GPU raises std::runtime_error).
#pragma once

#include "kohler/curve.hpp"
#include "kohler/image.hpp"

namespace kohler {

/// Definition-level curve: a naive GPU kernel scanning all ordered
/// 4-neighbour pairs once per threshold (shares no code with the fast path).
ContrastCurve direct_contrast_curve(const GrayImage& img);

/// The fast curve: one pass over the image on the GPU (sm_100a), exact.
/// `workers` is validated like the reference (0 throws std::invalid_argument)
/// and otherwise ignored: the result is identical for every worker count.
ContrastCurve fast_contrast_curve(const GrayImage& img, unsigned workers = 1);

} // namespace kohler

"""B200-native Köhler boundary-contrast curve (arXiv 1707.05062 hot path).

The product is the CUDA library ``lib/libkohler_cuda.so`` (C ABI in
``include/kohler_cuda.h``) and the C++ drop-in ``lib/libkohler_b200.so``
(headers under ``include/kohler/``).  This package is the Python host layer
over the same C ABI.
"""
from .api import (BatchResult, ContrastCurve, Context, DeviceGroup, GrayImage, LabelImage, MeanContrastCurve,
                  NoBoundaryError, ThresholdSet, analyze_batch, classify, default_context,
                  direct_contrast_curve, fast_contrast_curve, mean_contrast, merge_accumulators,
                  optimal_threshold, pair_contribution, quantize, top_k_local_maxima)

__all__ = [
    "BatchResult", "ContrastCurve", "Context", "DeviceGroup", "GrayImage", "LabelImage", "MeanContrastCurve",
    "NoBoundaryError", "ThresholdSet", "analyze_batch", "classify", "default_context",
    "direct_contrast_curve", "fast_contrast_curve", "mean_contrast", "merge_accumulators",
    "optimal_threshold", "pair_contribution", "quantize", "top_k_local_maxima",
]

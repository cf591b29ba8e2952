"""Python mirror of the reference's hot-path API, computed on the B200.

Same names, argument meaning and error behaviour as the reference's C++ API
(proj/include/kohler/{image,curve,contrast,threshold}.hpp):

=========================  =============================================  ======================
Python (this module)       reference                                      C ABI
=========================  =============================================  ======================
GrayImage                  image.hpp:15-63                                (host array)
ContrastCurve              curve.hpp:14-27                                256 x u64 x 2
pair_contribution          curve.hpp:32 / curve.cpp:10-14                 (host utility)
merge_accumulators         curve.hpp:37 / curve.cpp:16-30                 (host utility)
fast_contrast_curve        contrast.hpp:18 / fast.cpp:36-62               kohler_cuda_curve
direct_contrast_curve      contrast.hpp:11 / direct.cpp:10-43             kohler_cuda_direct_curve
mean_contrast              threshold.hpp:50 / threshold.cpp:9-23          kohler_cuda_mean_contrast
optimal_threshold          threshold.hpp:54 / threshold.cpp:25-37         kohler_cuda_optimal_threshold
top_k_local_maxima         threshold.hpp:60 / threshold.cpp:39-82         kohler_cuda_top_k_local_maxima
NoBoundaryError            threshold.hpp:14-20                            KOHLER_NO_BOUNDARY
LabelImage                 threshold.hpp:40-48                            (host array)
classify                   threshold.hpp:62-64 / threshold.cpp:84-101     kohler_cuda_classify
quantize                   threshold.hpp:66-67 / threshold.cpp:103-126    kohler_cuda_quantize
=========================  =============================================  ======================

Plus the batched / device-resident entry points of the B200 build
(:class:`Context`).  Everything runs through libkohler_cuda.so; there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib

LEVELS = _lib.LEVELS


class NoBoundaryError(RuntimeError):
    """No threshold has a boundary (reference: kohler::NoBoundaryError)."""

    def __init__(self, msg: str = "no boundary: the contrast curve is undefined at every threshold"):
        super().__init__(msg)


def _raise_for(status: int) -> None:
    if status == _lib.KOHLER_OK:
        return
    if status == _lib.KOHLER_NO_BOUNDARY:
        raise NoBoundaryError()
    msg = _lib.last_error()
    if status == _lib.KOHLER_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _lib.KOHLER_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(f"kohler (CUDA): {msg}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class GrayImage:
    """Row-major 8-bit image (reference GrayImage, image.hpp:15-63)."""

    def __init__(self, width: int, height: int, pixels=0):
        if width < 1 or height < 1:
            raise ValueError("GrayImage: dimensions must be at least 1x1")
        if np.isscalar(pixels):
            arr = np.full((height, width), int(pixels), dtype=np.uint8)
        else:
            arr = np.ascontiguousarray(np.asarray(pixels, dtype=np.uint8))
            if arr.size != width * height:
                raise ValueError("GrayImage: pixel count does not match dimensions")
            arr = arr.reshape(height, width)
        self._px = arr

    @classmethod
    def from_array(cls, a: np.ndarray) -> "GrayImage":
        a = np.asarray(a, dtype=np.uint8)
        if a.ndim != 2:
            raise ValueError("GrayImage.from_array expects a 2-D array")
        return cls(a.shape[1], a.shape[0], a)

    def width(self) -> int:
        return self._px.shape[1]

    def height(self) -> int:
        return self._px.shape[0]

    def pixel_count(self) -> int:
        return self._px.size

    def __call__(self, x: int, y: int) -> int:
        return int(self._px[y, x])

    def pixels(self) -> np.ndarray:
        return self._px

    def __eq__(self, other) -> bool:
        return isinstance(other, GrayImage) and np.array_equal(self._px, other._px)


class ContrastCurve:
    """contrast_sum / cardinality accumulators (reference curve.hpp:14-27)."""

    def __init__(self, levels: int = LEVELS):
        self.contrast_sum = np.zeros(levels, dtype=np.uint64)
        self.cardinality = np.zeros(levels, dtype=np.uint64)

    def levels(self) -> int:
        return int(self.cardinality.shape[0])

    def __eq__(self, other) -> bool:
        return (isinstance(other, ContrastCurve) and np.array_equal(self.contrast_sum, other.contrast_sum)
                and np.array_equal(self.cardinality, other.cardinality))

    def __repr__(self) -> str:
        return f"ContrastCurve(levels={self.levels()}, pairs={int(self.cardinality.sum())})"


@dataclass
class MeanContrastCurve:
    values: np.ndarray   # float64[levels]
    defined: np.ndarray  # bool[levels]

    def levels(self) -> int:
        return int(self.values.shape[0])


@dataclass
class ThresholdSet:
    thresholds: list

    def size(self) -> int:
        return len(self.thresholds)

    def __eq__(self, other) -> bool:
        return isinstance(other, ThresholdSet) and list(self.thresholds) == list(other.thresholds)


@dataclass
class BatchResult:
    sums: Optional[np.ndarray]       # (n, 256) u64
    cards: Optional[np.ndarray]      # (n, 256) u64
    values: Optional[np.ndarray]     # (n, 256) f64
    defined: Optional[np.ndarray]    # (n, 256) u8
    t0: np.ndarray                   # (n,) int32, -1 = no boundary
    topk: np.ndarray                 # (n, k) int32, valid prefix topk_count[i]
    topk_count: np.ndarray           # (n,) int32
    status: np.ndarray               # (n,) int32, 0 ok / 1 no boundary

    def thresholds(self, i: int) -> list:
        return [int(t) for t in self.topk[i, : self.topk_count[i]]]


class Context:
    """A libkohler_cuda context on one CUDA device (its stream + workspace)."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        _raise_for(lib.kohler_cuda_create(int(device), C.byref(h)))
        self._h = h
        self._lib = lib
        self.device = device

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.kohler_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def last_launch_count(self) -> int:
        return int(self._lib.kohler_cuda_last_launch_count(self._h))

    def set_pipeline_depth(self, depth: int) -> None:
        """Throughput mode for back-to-back device calls (include/kohler_cuda.h):
        depth d in [1, 4] accumulation launches run side by side on 1/d of the
        SMs each.  Results are unchanged."""
        _raise_for(self._lib.kohler_cuda_set_pipeline_depth(self._h, int(depth)))

    # ---- host-memory API ------------------------------------------------
    def curve(self, px: np.ndarray) -> ContrastCurve:
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        c = ContrastCurve()
        _raise_for(self._lib.kohler_cuda_curve(self._h, _ptr(px), w, h, w, _ptr(c.contrast_sum),
                                               _ptr(c.cardinality)))
        return c

    def direct_curve(self, px: np.ndarray) -> ContrastCurve:
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        c = ContrastCurve()
        _raise_for(self._lib.kohler_cuda_direct_curve(self._h, _ptr(px), w, h, w,
                                                      _ptr(c.contrast_sum), _ptr(c.cardinality)))
        return c

    def analyze_batch(self, px: np.ndarray, k: int = 6, curves: bool = True,
                      mean: bool = True) -> BatchResult:
        """Per-image pipeline over a host batch px[n, h, w] (u8)."""
        px = np.ascontiguousarray(px, dtype=np.uint8)
        if px.ndim == 2:
            px = px[None]
        n, h, w = px.shape
        r = _alloc_result(n, k, curves, mean)
        _raise_for(self._lib.kohler_cuda_analyze_batch(
            self._h, _ptr(px), n, w, h, w, w * h, int(k),
            _optr(r.sums), _optr(r.cards), _optr(r.values), _optr(r.defined),
            _ptr(r.t0), _ptr(r.topk), _ptr(r.topk_count), _ptr(r.status)))
        return r

    def select_host(self, sum_: np.ndarray, card: np.ndarray) -> MeanContrastCurve:
        sum_ = np.ascontiguousarray(sum_, dtype=np.uint64)
        card = np.ascontiguousarray(card, dtype=np.uint64)
        n = sum_.shape[0]
        vals = np.zeros(n, dtype=np.float64)
        dfn = np.zeros(n, dtype=np.uint8)
        if n:
            _raise_for(self._lib.kohler_cuda_mean_contrast(self._h, _ptr(sum_), _ptr(card), n,
                                                           _ptr(vals), _ptr(dfn)))
        return MeanContrastCurve(vals, dfn.astype(bool))

    def optimal_threshold(self, mc: MeanContrastCurve) -> int:
        v = np.ascontiguousarray(mc.values, dtype=np.float64)
        d = np.ascontiguousarray(mc.defined, dtype=np.uint8)
        if v.shape[0] == 0:
            raise NoBoundaryError()
        t0 = C.c_int(-1)
        _raise_for(self._lib.kohler_cuda_optimal_threshold(self._h, _ptr(v), _ptr(d), v.shape[0],
                                                           C.addressof(t0)))
        return int(t0.value)

    def top_k_local_maxima(self, mc: MeanContrastCurve, k: int) -> ThresholdSet:
        if k < 1:
            raise ValueError("top_k_local_maxima: k must be at least 1")
        v = np.ascontiguousarray(mc.values, dtype=np.float64)
        d = np.ascontiguousarray(mc.defined, dtype=np.uint8)
        if v.shape[0] == 0:
            raise NoBoundaryError()
        out = np.zeros(k, dtype=np.int32)
        cnt = C.c_int(0)
        _raise_for(self._lib.kohler_cuda_top_k_local_maxima(self._h, _ptr(v), _ptr(d), v.shape[0],
                                                            int(k), _ptr(out), C.addressof(cnt)))
        return ThresholdSet([int(t) for t in out[: cnt.value]])

    # ---- device-memory API (torch tensors as plumbing) -------------------
    def analyze_batch_device(self, px, w: int, h: int, pitch: int, image_stride: int, n: int,
                             k: int, out: dict, stream=None) -> None:
        """Asynchronous pipeline on device memory.  ``px`` is a CUDA uint8
        tensor (or raw pointer); ``out`` maps any of sums/cards/values/defined/
        t0/topk/topk_count/status to CUDA tensors.  Runs on ``stream`` (a
        torch.cuda.Stream) or the current torch stream."""
        _raise_for(self._lib.kohler_cuda_analyze_batch_device(
            self._h, _dptr(px), int(n), int(w), int(h), int(pitch), int(image_stride), int(k),
            *_outs(out, ("sums", "cards", "values", "defined", "t0", "topk", "topk_count",
                         "status")), _stream(stream)))

    def band_curve_device(self, band, w: int, pitch: int, h_total: int, r0: int, r1: int,
                          sum_, card, stream=None) -> None:
        _raise_for(self._lib.kohler_cuda_band_curve_device(
            self._h, _dptr(band), int(w), int(pitch), int(h_total), int(r0), int(r1),
            _dptr(sum_, "sums"), _dptr(card, "cards"), _stream(stream)))

    def select_device(self, sums, cards, n_curves: int, levels: int, k: int, out: dict,
                      stream=None) -> None:
        _raise_for(self._lib.kohler_cuda_select_device(
            self._h, _dptr(sums, "sums"), _dptr(cards, "cards"), int(n_curves), int(levels), int(k),
            *_outs(out, ("values", "defined", "t0", "topk", "topk_count", "status")),
            _stream(stream)))


    # ---- streaming host API ---------------------------------------------------
    def submit(self, px, k: int = 6) -> int:
        """Enqueue the pipeline on host image(s) px[n, h, w] / [h, w] (u8; a
        pinned torch tensor uploads at full PCIe speed) and return a ticket;
        ``collect(ticket)`` returns the results.  Two tickets may be in flight,
        so image i + 1's upload overlaps image i's kernels."""
        if hasattr(px, "data_ptr"):  # torch CPU tensor (e.g. pinned)
            t = px.contiguous()
            n, h, w = (1, *t.shape) if t.dim() == 2 else tuple(t.shape)
            ptr, keep = t.data_ptr(), t
        else:
            a = np.ascontiguousarray(px, dtype=np.uint8)
            if a.ndim == 2:
                a = a[None]
            n, h, w = a.shape
            ptr, keep = _ptr(a), a
        tk = C.c_longlong(-1)
        _raise_for(self._lib.kohler_cuda_submit(self._h, ptr, n, w, h, w, w * h, int(k),
                                                C.byref(tk)))
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[tk.value] = (keep, n, int(k))
        return tk.value

    def collect(self, ticket: int) -> BatchResult:
        keep, n, k = self._inflight.pop(ticket)
        r = _alloc_result(n, k, True, True)
        _raise_for(self._lib.kohler_cuda_collect(
            self._h, int(ticket), _optr(r.sums), _optr(r.cards), _optr(r.values), _optr(r.defined),
            _ptr(r.t0), _ptr(r.topk), _ptr(r.topk_count), _ptr(r.status)))
        del keep
        return r

    # ---- colour ingest ------------------------------
    def rgb_to_gray(self, rgb: np.ndarray) -> np.ndarray:
        """Rec. 601 integer luma of an (h, w, 3) u8 image on the GPU, as the
        reference's read_pnm reduces P6/P3 input (pnm.cpp:63-68)."""
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        if rgb.ndim != 3 or rgb.shape[2] != 3:
            raise ValueError("expected an (h, w, 3) RGB image")
        h, w = rgb.shape[:2]
        out = np.empty((h, w), np.uint8)
        _raise_for(self._lib.kohler_cuda_rgb_to_gray(self._h, _ptr(rgb), w, h, 3 * w, _ptr(out), w))
        return out

    def rgb_to_gray_device(self, rgb, n: int, w: int, h: int, rgb_pitch: int, rgb_stride: int,
                           gray, gray_pitch: int, gray_stride: int, stream=None) -> None:
        _raise_for(self._lib.kohler_cuda_rgb_to_gray_device(
            self._h, _dptr(rgb), int(n), int(w), int(h), int(rgb_pitch), int(rgb_stride),
            _dptr(gray), int(gray_pitch), int(gray_stride), _stream(stream)))

    def analyze_rgb_batch(self, rgb: np.ndarray, k: int = 6, curves: bool = True,
                          mean: bool = True) -> BatchResult:
        """analyze_batch on RGB input rgb[n, h, w, 3] (or [h, w, 3]): the
        luma is computed on the GPU and never leaves device staging memory."""
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        if rgb.ndim == 3:
            rgb = rgb[None]
        if rgb.ndim != 4 or rgb.shape[3] != 3:
            raise ValueError("expected RGB images of shape (n, h, w, 3)")
        n, h, w = rgb.shape[:3]
        r = _alloc_result(n, k, curves, mean)
        _raise_for(self._lib.kohler_cuda_analyze_rgb_batch(
            self._h, _ptr(rgb), n, w, h, 3 * w, 3 * w * h, int(k),
            _optr(r.sums), _optr(r.cards), _optr(r.values), _optr(r.defined),
            _ptr(r.t0), _ptr(r.topk), _ptr(r.topk_count), _ptr(r.status)))
        return r

    def analyze_rgb_batch_device(self, rgb, w: int, h: int, rgb_pitch: int, rgb_stride: int,
                                 n: int, k: int, out: dict, stream=None) -> None:
        _raise_for(self._lib.kohler_cuda_analyze_rgb_batch_device(
            self._h, _dptr(rgb), int(n), int(w), int(h), int(rgb_pitch), int(rgb_stride), int(k),
            *_outs(out, ("sums", "cards", "values", "defined", "t0", "topk", "topk_count",
                         "status")), _stream(stream)))

    # ---- segmentation -------------------------------
    def classify(self, px: np.ndarray, thresholds) -> np.ndarray:
        """labels[y, x] = number of thresholds strictly below px[y, x]."""
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        ts = np.ascontiguousarray(np.asarray(thresholds, dtype=np.int32).reshape(-1))
        out = np.empty((h, w), np.uint8)
        _raise_for(self._lib.kohler_cuda_classify(self._h, _ptr(px), w, h, w, _ptr(ts),
                                                  ts.shape[0], _ptr(out)))
        return out

    def quantize(self, px: np.ndarray, thresholds) -> np.ndarray:
        """Each pixel replaced by its class mean, rounded half up."""
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        ts = np.ascontiguousarray(np.asarray(thresholds, dtype=np.int32).reshape(-1))
        out = np.empty((h, w), np.uint8)
        _raise_for(self._lib.kohler_cuda_quantize(self._h, _ptr(px), w, h, w, _ptr(ts),
                                                  ts.shape[0], _ptr(out)))
        return out

    def segment_batch(self, px: np.ndarray, k: int = 0):
        """Per-image segmentation of px[n, h, w]: k == 0 the video pipeline
        (bench.cpp:266-281: {optimal_threshold}, two classes), k >= 1 the
        top-k quantize of the segment command.  Frames without boundary pass
        through (status 1).  -> (out[n, h, w], thresholds[n, max(k,1)],
        counts[n], status[n])."""
        px = np.ascontiguousarray(px, dtype=np.uint8)
        if px.ndim == 2:
            px = px[None]
        n, h, w = px.shape
        out = np.empty_like(px)
        ts = np.zeros((n, max(k, 1)), np.int32)
        cnt = np.zeros(n, np.int32)
        st = np.zeros(n, np.int32)
        _raise_for(self._lib.kohler_cuda_segment_batch(self._h, _ptr(px), n, w, h, int(k),
                                                       _ptr(out), _ptr(ts), _ptr(cnt), _ptr(st)))
        return out, ts, cnt, st

    def segment_batch_device(self, px, w: int, h: int, pitch: int, image_stride: int, n: int,
                             k: int, out, out_pitch: int, out_stride: int, thresholds, counts,
                             status, stream=None) -> None:
        _raise_for(self._lib.kohler_cuda_segment_batch_device(
            self._h, _dptr(px), int(n), int(w), int(h), int(pitch), int(image_stride), int(k),
            _dptr(out), int(out_pitch), int(out_stride), _dptr(thresholds, "topk"),
            _dptr(counts, "topk_count"), _dptr(status, "status"), _stream(stream)))


def _alloc_result(n: int, k: int, curves: bool, mean: bool) -> BatchResult:
    return BatchResult(
        sums=np.zeros((n, LEVELS), np.uint64) if curves else None,
        cards=np.zeros((n, LEVELS), np.uint64) if curves else None,
        values=np.zeros((n, LEVELS), np.float64) if mean else None,
        defined=np.zeros((n, LEVELS), np.uint8) if mean else None,
        t0=np.full(n, -1, np.int32), topk=np.zeros((n, k), np.int32),
        topk_count=np.zeros(n, np.int32), status=np.zeros(n, np.int32))


def _optr(a):
    return None if a is None else a.ctypes.data


_OUT_DTYPES = {"sums": ("int64", "uint64"), "cards": ("int64", "uint64"), "values": ("float64",),
               "defined": ("uint8", "bool"), "t0": ("int32",), "topk": ("int32",),
               "topk_count": ("int32",), "status": ("int32",)}


def _dptr(t, kind: str = None):
    """Device pointer of a CUDA tensor (or a raw int pointer, passed through).
    ``kind``: None for an image buffer (uint8, any strides: the pitch is
    explicit), else an output name of _OUT_DTYPES (contiguous, that dtype).
    A CPU tensor or a wrong dtype would silently compute garbage or fault in
    the kernel, so it is refused here."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not getattr(t, "is_cuda", False):
        raise ValueError("device API: expected a CUDA tensor")
    dt = str(t.dtype).replace("torch.", "")
    if kind is None:
        if dt != "uint8":
            raise ValueError(f"device API: image buffers must be uint8, got {dt}")
    else:
        if dt not in _OUT_DTYPES[kind]:
            raise ValueError(f"device API: '{kind}' must be {' or '.join(_OUT_DTYPES[kind])}, got {dt}")
        if not t.is_contiguous():
            raise ValueError(f"device API: '{kind}' must be contiguous")
    return t.data_ptr()


def _outs(out: dict, names) -> list:
    return [_dptr(out.get(n), n) for n in names]


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ---- process-wide default context (like the C++ drop-in) -------------------
_default = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _default_lock:
        if _default is None:
            _default = Context(int(os.environ.get("KOHLER_CUDA_DEVICE", "0")))
        return _default


def _as_array(img) -> np.ndarray:
    if isinstance(img, GrayImage):
        return img.pixels()
    a = np.asarray(img, dtype=np.uint8)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("GrayImage: dimensions must be at least 1x1")
    return a


def pair_contribution(lo: int, hi: int, acc: ContrastCurve) -> None:
    """Host utility (reference curve.cpp:10-14): tent of one pair lo <= hi."""
    for t in range(int(lo), int(hi)):
        acc.contrast_sum[t] += np.uint64(min(int(hi) - t, t - int(lo)))
        acc.cardinality[t] += np.uint64(1)


def merge_accumulators(parts: Sequence[ContrastCurve]) -> ContrastCurve:
    """Entrywise u64 sum (reference curve.cpp:16-30)."""
    if len(parts) == 0:
        raise ValueError("merge_accumulators: no partial results")
    out = ContrastCurve(parts[0].levels())
    for p in parts:
        if p.levels() != out.levels():
            raise ValueError("merge_accumulators: mismatched curve lengths")
        out.contrast_sum += p.contrast_sum
        out.cardinality += p.cardinality
    return out


def fast_contrast_curve(img, workers: int = 1) -> ContrastCurve:
    """GPU curve of one image (reference fast_contrast_curve, fast.cpp:36-62).
    ``workers`` is validated (0 raises ValueError) and otherwise irrelevant."""
    if workers < 1:
        raise ValueError("fast_contrast_curve: workers must be at least 1")
    return default_context().curve(_as_array(img))


def direct_contrast_curve(img) -> ContrastCurve:
    """Definition-level GPU curve (reference direct.cpp:10-43)."""
    return default_context().direct_curve(_as_array(img))


class DeviceGroup:
    """Several GPUs of one box driven from this thread (include/kohler_cuda.h,
    device groups): one context and one NCCL communicator per device.
    ``curve``/``analyze`` split ONE image into row bands like the reference's
    fast_contrast_curve (proj/src/fast.cpp:42-61); the band kernels add their
    exact partials into one accumulator on the first device over peer memory
    (``uses_peer``), or, where the devices cannot map each other's memory, one
    NCCL all-reduce merges them; ``analyze_batch`` shards a batch by image (no
    collective)."""

    def __init__(self, devices=None, n: int = 0):
        lib = _lib.load()
        devs = list(devices) if devices is not None else list(range(n or 1))
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        _raise_for(lib.kohler_cuda_multi_create(arr, len(devs), C.byref(h)))
        self._h, self._lib, self.devices = h, lib, devs

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.kohler_cuda_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self) -> int:
        return int(self._lib.kohler_cuda_multi_size(self._h))

    def uses_nccl(self) -> bool:
        return bool(self._lib.kohler_cuda_multi_uses_nccl(self._h))

    def uses_peer(self) -> bool:
        """Peer mode: the members' band kernels add straight into one
        accumulator on the first device (no collective)."""
        return bool(self._lib.kohler_cuda_multi_uses_peer(self._h))

    def curve(self, px: np.ndarray) -> ContrastCurve:
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        c = ContrastCurve()
        _raise_for(self._lib.kohler_cuda_multi_curve(self._h, _ptr(px), w, h, w,
                                                     _ptr(c.contrast_sum), _ptr(c.cardinality)))
        return c

    def analyze(self, px: np.ndarray, k: int = 6) -> BatchResult:
        """One image over the group; a one-image BatchResult (status 1 = no boundary)."""
        px = np.ascontiguousarray(px, dtype=np.uint8)
        h, w = px.shape
        r = _alloc_result(1, k, True, True)
        rc = self._lib.kohler_cuda_multi_analyze(
            self._h, _ptr(px), w, h, w, int(k), _ptr(r.sums), _ptr(r.cards), _ptr(r.values),
            _ptr(r.defined), _ptr(r.t0), _ptr(r.topk), _ptr(r.topk_count))
        if rc not in (_lib.KOHLER_OK, _lib.KOHLER_NO_BOUNDARY):
            _raise_for(rc)
        r.status[0] = rc
        return r

    def analyze_batch(self, px: np.ndarray, k: int = 6) -> BatchResult:
        px = np.ascontiguousarray(px, dtype=np.uint8)
        if px.ndim == 2:
            px = px[None]
        n, h, w = px.shape
        r = _alloc_result(n, k, True, True)
        _raise_for(self._lib.kohler_cuda_multi_analyze_batch(
            self._h, _ptr(px), n, w, h, w, w * h, int(k), _ptr(r.sums), _ptr(r.cards),
            _ptr(r.values), _ptr(r.defined), _ptr(r.t0), _ptr(r.topk), _ptr(r.topk_count),
            _ptr(r.status)))
        return r


def mean_contrast(curve: ContrastCurve) -> MeanContrastCurve:
    return default_context().select_host(curve.contrast_sum, curve.cardinality)


def optimal_threshold(mc: MeanContrastCurve) -> int:
    return default_context().optimal_threshold(mc)


def top_k_local_maxima(mc: MeanContrastCurve, k: int) -> ThresholdSet:
    return default_context().top_k_local_maxima(mc, k)


def analyze_batch(px: np.ndarray, k: int = 6) -> BatchResult:
    return default_context().analyze_batch(px, k)


@dataclass
class LabelImage:
    """Class index per pixel (reference: kohler::LabelImage, threshold.hpp:40-48)."""
    width: int
    height: int
    labels: np.ndarray

    def __eq__(self, other) -> bool:
        return (isinstance(other, LabelImage) and self.width == other.width and
                self.height == other.height and np.array_equal(self.labels, other.labels))


def _ts_list(ts) -> list:
    return list(ts.thresholds) if isinstance(ts, ThresholdSet) else list(ts)


def classify(img, ts) -> LabelImage:
    """label(x) = number of thresholds strictly below the pixel value
    (threshold.cpp:84-101), on the GPU."""
    a = _as_array(img)
    return LabelImage(a.shape[1], a.shape[0], default_context().classify(a, _ts_list(ts)))


def quantize(img, ts) -> GrayImage:
    """Every pixel replaced by the mean grey value of its class, rounded half
    up (threshold.cpp:103-126), on the GPU."""
    a = _as_array(img)
    return GrayImage.from_array(default_context().quantize(a, _ts_list(ts)))

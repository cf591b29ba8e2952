"""Checkers for the Köhler path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as part of the product path.

* :class:`Oracle`    — ctypes over ``_build/libkohler_oracle.so``, the C
  restatement in kohler_oracle.c (each function cites the reference lines it
  follows).
* :class:`Reference` — ctypes over ``_ref/libkohler_ref.so``, the reference
  library itself compiled from /root/reference/proj/src by oracle/Makefile
  (namespace-renamed, plus the C shim ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libkohler_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkohler_ref.so")
REFERENCE_SRC = "/root/reference/proj"

NO_BOUNDARY = 1
INVALID_K = 2


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when /root/reference is present, the
    reference library and the reference's acceptance runner relinked against
    the drop-in (outputs only under oracle/_build and oracle/_ref)."""
    targets = [ORACLE_SO]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets += ["ref", "acceptance"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


class Oracle:
    """The C restatement of the reference algorithm (kohler_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        vp, i = C.c_void_p, C.c_int
        for name, args, res in [
            ("oracle_pair_contribution", [i, i, vp, vp], None),
            ("oracle_curve_rows", [vp, i, i, C.c_size_t, i, i, vp, vp], None),
            ("oracle_fast_curve", [vp, i, i, vp, vp], None),
            ("oracle_fast_curve_blocks", [vp, i, i, C.c_uint, vp, vp], None),
            ("oracle_direct_curve", [vp, i, i, vp, vp], None),
            ("oracle_mean_contrast", [vp, vp, i, vp, vp], None),
            ("oracle_optimal_threshold", [vp, vp, i], i),
            ("oracle_top_k_local_maxima", [vp, vp, i, i, vp, vp], i),
            ("oracle_identities", [vp, i, i, vp, vp], None),
            ("oracle_analyze", [vp, i, i, i, vp, vp, vp, vp, vp, vp, vp], i),
            ("oracle_rgb_to_gray", [vp, i, i, C.c_size_t, vp], None),
        ]:
            f = getattr(self.lib, name)
            f.argtypes = args
            f.restype = res

    @staticmethod
    def _img(px):
        px = np.ascontiguousarray(px, dtype=np.uint8)
        if px.ndim != 2:
            raise ValueError("expected a 2-D image")
        return px, px.shape[1], px.shape[0]

    def rgb_to_gray(self, rgb):
        """rgb: (h, w, 3) uint8 -> (h, w) luma (pnm.cpp:63-68 restated)."""
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        if rgb.ndim != 3 or rgb.shape[2] != 3:
            raise ValueError("expected an (h, w, 3) RGB image")
        h, w = rgb.shape[:2]
        out = np.empty((h, w), np.uint8)
        self.lib.oracle_rgb_to_gray(_p(rgb), w, h, 3 * w, _p(out))
        return out

    def pair_contribution(self, lo, hi):
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.oracle_pair_contribution(int(lo), int(hi), _p(s), _p(c))
        return s, c

    def fast_curve(self, px):
        px, w, h = self._img(px)
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.oracle_fast_curve(_p(px), w, h, _p(s), _p(c))
        return s, c

    def curve_rows(self, px, r0, r1):
        """Partial curve of the pairs rows [r0, r1) own (fast.cpp:18-32)."""
        px, w, h = self._img(px)
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.oracle_curve_rows(_p(px), w, h, w, int(r0), int(r1), _p(s), _p(c))
        return s, c

    def fast_curve_blocks(self, px, blocks):
        px, w, h = self._img(px)
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.oracle_fast_curve_blocks(_p(px), w, h, int(blocks), _p(s), _p(c))
        return s, c

    def direct_curve(self, px):
        px, w, h = self._img(px)
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.oracle_direct_curve(_p(px), w, h, _p(s), _p(c))
        return s, c

    def mean_contrast(self, s, c):
        s = np.ascontiguousarray(s, np.uint64)
        c = np.ascontiguousarray(c, np.uint64)
        n = s.shape[0]
        v = np.zeros(n, np.float64)
        d = np.zeros(n, np.uint8)
        self.lib.oracle_mean_contrast(_p(s), _p(c), n, _p(v), _p(d))
        return v, d

    def optimal_threshold(self, v, d):
        v = np.ascontiguousarray(v, np.float64)
        d = np.ascontiguousarray(d, np.uint8)
        return int(self.lib.oracle_optimal_threshold(_p(v), _p(d), v.shape[0]))

    def top_k(self, v, d, k):
        """-> (status, thresholds); status 0 ok, 1 no boundary, 2 invalid k."""
        v = np.ascontiguousarray(v, np.float64)
        d = np.ascontiguousarray(d, np.uint8)
        out = np.zeros(max(int(k), 1), np.int32)
        cnt = np.zeros(1, np.int32)
        st = self.lib.oracle_top_k_local_maxima(_p(v), _p(d), v.shape[0], int(k), _p(out), _p(cnt))
        return int(st), [int(t) for t in out[: cnt[0]]]

    def identities(self, px):
        px, w, h = self._img(px)
        tv = np.zeros(1, np.uint64)
        qs = np.zeros(1, np.uint64)
        self.lib.oracle_identities(_p(px), w, h, _p(tv), _p(qs))
        return int(tv[0]), int(qs[0])

    def analyze(self, px, k=6):
        """-> dict(sum, card, values, defined, t0, topk, status)."""
        px, w, h = self._img(px)
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        v = np.zeros(256, np.float64)
        d = np.zeros(256, np.uint8)
        t0 = np.zeros(1, np.int32)
        tk = np.zeros(k, np.int32)
        cnt = np.zeros(1, np.int32)
        st = self.lib.oracle_analyze(_p(px), w, h, int(k), _p(s), _p(c), _p(v), _p(d), _p(t0),
                                     _p(tk), _p(cnt))
        return dict(sum=s, card=c, values=v, defined=d, t0=int(t0[0]),
                    topk=[int(t) for t in tk[: cnt[0]]], status=int(st))


class Reference:
    """The reference library compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        self.lib = C.CDLL(path)
        vp, i, u = C.c_void_p, C.c_int, C.c_uint
        for name, args, res in [
            ("kref_active_kernel", [], C.c_char_p),
            ("kref_image_new", [vp, i, i], vp),
            ("kref_image_free", [vp], None),
            ("kref_fast_curve", [vp, u, vp, vp], i),
            ("kref_direct_curve", [vp, vp, vp], i),
            ("kref_pair_contribution", [i, i, vp, vp], None),
            ("kref_mean_contrast", [vp, vp, i, vp, vp], None),
            ("kref_optimal_threshold", [vp, vp, i, vp], i),
            ("kref_top_k", [vp, vp, i, i, vp, vp], i),
            ("kref_pipeline", [vp, u, i, vp, vp, vp, vp, vp, vp, vp], i),
            ("kref_pipeline_batch", [vp, i, u, i, i, vp, vp, vp, vp, vp], i),
            ("kref_time_pipeline", [vp, u, i, i, i], C.c_double),
            ("kref_classify", [vp, vp, i, vp], None),
            ("kref_quantize", [vp, vp, i, vp], None),
            ("kref_segment", [vp, u, i, vp, vp, vp], i),
            ("kref_read_pnm", [vp, C.c_size_t, vp, C.c_size_t, vp, vp], i),
        ]:
            f = getattr(self.lib, name)
            f.argtypes = args
            f.restype = res

    def read_pnm(self, data: bytes) -> np.ndarray:
        """The reference's read_pnm (proj/src/pnm.cpp:87-139) on a PNM byte
        stream -> (h, w) uint8; ValueError on a PnmError."""
        buf = np.frombuffer(bytes(data), np.uint8)
        cap = max(len(data), 1)
        out = np.empty(cap, np.uint8)
        w, h = C.c_int(0), C.c_int(0)
        rc = self.lib.kref_read_pnm(_p(buf), len(data), _p(out), cap, C.byref(w), C.byref(h))
        if rc:
            raise ValueError("reference read_pnm rejected the stream")
        return out[: w.value * h.value].reshape(h.value, w.value).copy()

    def active_kernel(self) -> str:
        return self.lib.kref_active_kernel().decode()

    def image(self, px) -> "RefImage":
        return RefImage(self, px)

    def fast_curve(self, px, workers=1):
        with self.image(px) as im:
            s = np.zeros(256, np.uint64)
            c = np.zeros(256, np.uint64)
            st = self.lib.kref_fast_curve(im.h, int(workers), _p(s), _p(c))
            if st:
                raise ValueError("fast_contrast_curve: workers must be at least 1")
            return s, c

    def direct_curve(self, px):
        with self.image(px) as im:
            s = np.zeros(256, np.uint64)
            c = np.zeros(256, np.uint64)
            self.lib.kref_direct_curve(im.h, _p(s), _p(c))
            return s, c

    def pair_contribution(self, lo, hi):
        s = np.zeros(256, np.uint64)
        c = np.zeros(256, np.uint64)
        self.lib.kref_pair_contribution(int(lo), int(hi), _p(s), _p(c))
        return s, c

    def mean_contrast(self, s, c):
        s = np.ascontiguousarray(s, np.uint64)
        c = np.ascontiguousarray(c, np.uint64)
        n = s.shape[0]
        v = np.zeros(n, np.float64)
        d = np.zeros(n, np.uint8)
        self.lib.kref_mean_contrast(_p(s), _p(c), n, _p(v), _p(d))
        return v, d

    def optimal_threshold(self, v, d):
        v = np.ascontiguousarray(v, np.float64)
        d = np.ascontiguousarray(d, np.uint8)
        t = np.zeros(1, np.int32)
        st = self.lib.kref_optimal_threshold(_p(v), _p(d), v.shape[0], _p(t))
        return -1 if st else int(t[0])

    def top_k(self, v, d, k):
        v = np.ascontiguousarray(v, np.float64)
        d = np.ascontiguousarray(d, np.uint8)
        out = np.zeros(max(int(k), 1) + v.shape[0], np.int32)
        cnt = np.zeros(1, np.int32)
        st = self.lib.kref_top_k(_p(v), _p(d), v.shape[0], int(k), _p(out), _p(cnt))
        return int(st), [int(t) for t in out[: cnt[0]]]

    def analyze(self, px, k=6, workers=1):
        with self.image(px) as im:
            s = np.zeros(256, np.uint64)
            c = np.zeros(256, np.uint64)
            v = np.zeros(256, np.float64)
            d = np.zeros(256, np.uint8)
            t0 = np.zeros(1, np.int32)
            tk = np.zeros(k, np.int32)
            cnt = np.zeros(1, np.int32)
            st = self.lib.kref_pipeline(im.h, int(workers), int(k), _p(s), _p(c), _p(v), _p(d),
                                        _p(t0), _p(tk), _p(cnt))
            return dict(sum=s, card=c, values=v, defined=d, t0=int(t0[0]),
                        topk=[int(t) for t in tk[: cnt[0]]], status=int(st))


    def analyze_batch(self, imgs, k=6, workers=1, threads=None):
        """Per-image pipeline over imgs[n, h, w], frame-parallel over `threads`
        host threads (kref_pipeline_batch).  -> dict of stacked outputs."""
        imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
        n = imgs.shape[0]
        threads = threads or os.cpu_count() or 1
        handles = [RefImage(self, imgs[i]) for i in range(n)]
        arr = (C.c_void_p * n)(*[hh.h for hh in handles])
        sums = np.zeros((n, 256), np.uint64)
        cards = np.zeros((n, 256), np.uint64)
        t0 = np.zeros(n, np.int32)
        tk = np.zeros((n, k), np.int32)
        cnt = np.zeros(n, np.int32)
        self.lib.kref_pipeline_batch(arr, n, int(workers), int(threads), int(k), _p(sums),
                                     _p(cards), _p(t0), _p(tk), _p(cnt))
        for hh in handles:
            hh.close()
        return dict(sums=sums, cards=cards, t0=t0, topk=tk, topk_count=cnt)


def _ref_thresholds(ts):
    return np.ascontiguousarray(np.asarray(ts, dtype=np.int32).reshape(-1))


def ref_classify(ref, img, ts):
    """Reference classify (threshold.cpp:84-101) -> u8 labels, same shape."""
    t = _ref_thresholds(ts)
    out = np.zeros(img.shape, np.uint8)
    with RefImage(ref, img) as im:
        ref.lib.kref_classify(im.h, _p(t), t.shape[0], _p(out))
    return out


def ref_quantize(ref, img, ts):
    """Reference quantize (threshold.cpp:103-126) -> u8 image."""
    t = _ref_thresholds(ts)
    out = np.zeros(img.shape, np.uint8)
    with RefImage(ref, img) as im:
        ref.lib.kref_quantize(im.h, _p(t), t.shape[0], _p(out))
    return out


def ref_segment(ref, img, k=0, workers=1):
    """One frame of the reference video pipeline (bench.cpp:266-281; k > 0:
    the segment command's top-k).  -> (out image, thresholds, status)."""
    out = np.zeros(img.shape, np.uint8)
    ts = np.zeros(max(k, 1), np.int32)
    cnt = np.zeros(1, np.int32)
    with RefImage(ref, img) as im:
        st = ref.lib.kref_segment(im.h, int(workers), int(k), _p(out), _p(ts), _p(cnt))
    return out, list(ts[:int(cnt[0])]), int(st)


class RefImage:
    """A kohler_ref::GrayImage built once (outside any timed region)."""

    def __init__(self, ref: Reference, px):
        px = np.ascontiguousarray(px, dtype=np.uint8)
        self.ref = ref
        self.h = ref.lib.kref_image_new(_p(px), px.shape[1], px.shape[0])
        if not self.h:
            raise ValueError("GrayImage: invalid dimensions")

    def close(self):
        if self.h:
            self.ref.lib.kref_image_free(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        self.close()

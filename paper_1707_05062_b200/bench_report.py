"""GPU rows in the reference's benchmark report.

Restates the reference's image and video benchmarks with their semantics and
CSV layout, as a separate harness whose rows name the GPU paths.  "gpu" is
deliberately not a value of the reference's ``Impl`` enum
(proj/tests/test_bench.cpp:55 pins that it is rejected), so the reference's
own harness stays untouched:

* ``bench_image`` (proj/src/bench.cpp:131-187): correctness before timing --
  every implementation must produce the same curve as the first one or
  ``CurveMismatchError`` is raised and nothing is timed; then ``warmup +
  runs`` executions of curve + mean_contrast (the normalisation is timed,
  :174-181), wall clock, the last ``runs`` kept, median as in ``median_of``
  (:19-24, even counts average the middle pair).
* ``write_report_csv`` (:189-210): ``name,width,height,runs,median_s,
  run<i>_s...,gain_vs_direct``; durations with 6 decimals, the gain with 2
  (empty without a direct row).  Here the direct row is ``gpu_direct``, the
  definition-level GPU kernel (proj/src/direct.cpp:10-43 restated).
* ``bench_video`` (:223-299): per frame, curve -> (boundary?) mean curve ->
  optimal threshold -> two-class quantize, timed together; constant frames
  pass through and are tallied; decode time is excluded (frames are arrays).

Implementations are names ("gpu", "gpu_direct") or ``(name, callable)``
pairs like the reference's ``CurveImpl`` (bench.hpp:58-63), so tests can
inject a corrupted one.
"""
from __future__ import annotations

import argparse
import time
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import api

DIRECT = "gpu_direct"


class CurveMismatchError(RuntimeError):
    """Implementations disagree on a curve; nothing was timed."""


def _gpu_fast(img):
    return api.fast_contrast_curve(img)


def _gpu_direct(img):
    return api.direct_contrast_curve(img)


_STANDARD = {"gpu": _gpu_fast, DIRECT: _gpu_direct}


def _resolve(impls) -> list:
    out = []
    for it in impls:
        if isinstance(it, str):
            if it not in _STANDARD:
                raise ValueError(f"unknown implementation {it!r} (known: {sorted(_STANDARD)})")
            out.append((it, _STANDARD[it]))
        else:
            name, fn = it
            out.append((str(name), fn))
    if not out:
        raise ValueError("bench_image: no implementations selected")
    return out


def median_of(v: Sequence[float]) -> float:
    s = sorted(v)
    n = len(s)
    return s[n // 2] if n % 2 == 1 else 0.5 * (s[n // 2 - 1] + s[n // 2])


@dataclass
class ImplTiming:
    name: str
    runs_s: list = field(default_factory=list)
    median_s: float = 0.0


@dataclass
class BenchReport:
    image_id: str = "image"
    width: int = 0
    height: int = 0
    runs: int = 0
    warmup: int = 0
    workers: int = 1
    results: list = field(default_factory=list)

    def find(self, name: str) -> Optional[ImplTiming]:
        for t in self.results:
            if t.name == name:
                return t
        return None

    def gain_vs_direct(self, name: str) -> Optional[float]:
        """median(direct) / median(name); None without a direct row."""
        d, s = self.find(DIRECT), self.find(name)
        if d is None or s is None:
            return None
        return d.median_s / s.median_s


def bench_image(img, impls: Iterable = ("gpu_direct", "gpu"), runs: int = 5, warmup: int = 1,
                workers: int = 1, image_id: str = "image") -> BenchReport:
    if runs < 1:
        raise ValueError("bench_image: runs must be at least 1")
    if warmup < 0:
        raise ValueError("bench_image: warmup must be non-negative")
    chosen = _resolve(impls)
    a = api._as_array(img)
    curves = [fn(a) for _, fn in chosen]
    for i in range(1, len(curves)):
        if curves[i] != curves[0]:
            c0, ci = curves[0], curves[i]
            t = next((t for t in range(c0.levels())
                      if c0.contrast_sum[t] != ci.contrast_sum[t]
                      or c0.cardinality[t] != ci.cardinality[t]), -1)
            raise CurveMismatchError(f"bench: {chosen[i][0]} and {chosen[0][0]} disagree at "
                                     f"t={t}; refusing to time broken code")
    rep = BenchReport(image_id, a.shape[1], a.shape[0], runs, warmup, workers)
    for name, fn in chosen:
        tm = ImplTiming(name)
        for r in range(warmup + runs):
            t0 = time.perf_counter()
            api.mean_contrast(fn(a))  # the normalisation is timed (bench.cpp:174-181)
            t1 = time.perf_counter()
            if r >= warmup:
                tm.runs_s.append(max(t1 - t0, 1e-9))
        tm.median_s = median_of(tm.runs_s)
        rep.results.append(tm)
    return rep


def write_report_csv(report: BenchReport) -> str:
    out = "name,width,height,runs,median_s"
    for r in range(1, report.runs + 1):
        out += f",run{r}_s"
    out += ",gain_vs_direct\n"
    for t in report.results:
        out += f"{t.name},{report.width},{report.height},{report.runs},{t.median_s:.6f}"
        for s in t.runs_s:
            out += f",{s:.6f}"
        out += ","
        g = report.gain_vs_direct(t.name)
        if g is not None:
            out += f"{g:.2f}"
        out += "\n"
    return out


@dataclass
class Throughput:
    name: str
    seconds: float = 0.0
    fps: float = 0.0


@dataclass
class VideoReport:
    frame_count: int = 0
    width: int = 0
    height: int = 0
    workers: int = 1
    results: list = field(default_factory=list)
    decode_seconds: float = 0.0
    constant_frames: int = 0

    def find(self, name: str) -> Optional[Throughput]:
        for t in self.results:
            if t.name == name:
                return t
        return None

    def gain_vs_direct(self, name: str) -> Optional[float]:
        d, s = self.find(DIRECT), self.find(name)
        if d is None or s is None:
            return None
        return s.fps / d.fps


def bench_video(frames: Sequence, impls: Iterable = ("gpu",), workers: int = 1,
                segmented_out: Optional[list] = None) -> VideoReport:
    """Two-class segmentation throughput over decoded frames (bench.cpp:
    223-299).  With ``segmented_out`` (a list), the first implementation's
    output frames are appended to it, outside the timed section."""
    if len(frames) == 0:
        raise ValueError("bench_video: empty frame sequence")
    chosen = _resolve(impls)
    fr = [api._as_array(f) for f in frames]
    rep = VideoReport(len(fr), fr[0].shape[1], fr[0].shape[0], workers)
    first = True
    for name, fn in chosen:
        seconds = 0.0
        constant = 0
        for a in fr:
            t0 = time.perf_counter()
            curve = fn(a)
            seg = None
            if bool(np.any(curve.cardinality)):
                mc = api.mean_contrast(curve)
                seg = api.quantize(a, [api.optimal_threshold(mc)])  # two classes
            t1 = time.perf_counter()
            seconds += t1 - t0
            if seg is None:
                seg = api.GrayImage.from_array(a)  # constant frame: passed through
                if first:
                    constant += 1
            if first and segmented_out is not None:
                segmented_out.append(seg)
        seconds = max(seconds, 1e-9)
        rep.results.append(Throughput(name, seconds, len(fr) / seconds))
        if first:
            rep.constant_frames = constant
        first = False
    return rep


def main(argv=None) -> None:
    from . import synth
    ap = argparse.ArgumentParser(description="GPU rows of the reference's bench CSV")
    ap.add_argument("--config", default="C2", help="synthetic BASELINE config (C1..C5)")
    ap.add_argument("--image", type=int, default=0, help="image of the config's batch")
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args(argv)
    img = synth.generate(a.config, device="cpu")[a.image].numpy()
    rep = bench_image(img, runs=a.runs, warmup=a.warmup, image_id=a.config)
    print(write_report_csv(rep), end="")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Benchmark of the Köhler contrast-curve hot path on B200.

Workload (BASELINE.json configs[1], "C2"): one 5184x3456 uint8 image
(gradient + 40 ellipses + N(0,5^2), seeded), full N4 curve (u64 sum/count),
IEEE f64 mean curve, optimal threshold and top-6 local maxima.  One step =
one pass of that pipeline over the image.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: per step one K1 launch (accumulate) and one finish launch (K3
reconstruct + K4 select), PDL-chained; pipeline depth 3 (three steps in
flight on a third of the SMs each) and the step loop replayed from CUDA
graphs of 500 steps captured through the public device API.  e2e: the host C
ABI with a pinned host image every step (streaming submit/collect, and the
synchronous call beside it).
N > 1 (torchrun, one process per GPU, NCCL): the image is split into row
bands with a one-row halo (proj/src/fast.cpp:42-57); per step each rank runs
K1 on its band, one all-reduce of the 512 u64 partials (overlapped with the
next step's band), then K4 — strong scaling (the image is fixed); also
graph-replayed.  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks; the last step's result is
re-checked against the oracle after the timed loop.  L2 (126 MB) is defeated
by rotating through input copies totalling > 2x L2.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libkohler_ref.so, compiled from the reference sources) on this
host's cores with the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "Gpixel/s (full 8-bit N4 Koehler curve + optimal threshold + top-6 maxima)"
UNIT = "Gpixel/s"
K_TOP = 6
CONFIG_NAME = "C2"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    --set full capture summary (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(CONFIG_NAME)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the workload runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=3.0):
        """Block until nvidia-smi has produced its first sample."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.mark = len(self.lines)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_input(device="cpu"):
    from paper_1707_05062_b200 import synth
    return synth.generate(CONFIG_NAME, device=device)[0]


def cpu_reference_time(img: np.ndarray, budget_s: float, max_runs: int):
    """Median steady_clock time of the reference pipeline (curve + mean +
    t0 + top-6) with workers = all host cores — bench.cpp:171-185 method."""
    import oracle
    ref = oracle.Reference()
    cores = os.cpu_count() or 1
    with ref.image(img) as im:
        one = ref.lib.kref_time_pipeline(im.h, cores, K_TOP, 1, 1)
        runs = int(max(3, min(max_runs, budget_s / max(one, 1e-6))))
        med = ref.lib.kref_time_pipeline(im.h, cores, K_TOP, 0, runs)
    return med, runs, cores, ref.active_kernel()


def workload_name(w: int, h: int) -> str:
    return f"{CONFIG_NAME} {w}x{h} gradient+40 ellipses+N(0,5^2), seed 0x51C2, k={K_TOP}"


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference's CPU implementation on this host."""
    if rank != 0:
        return
    import oracle
    img = make_input("cpu").numpy()
    h, w = img.shape
    ref = oracle.Reference()
    cores = os.cpu_count() or 1
    with ref.image(img) as im:
        for _ in range(args.warmup):
            ref.lib.kref_time_pipeline(im.h, cores, K_TOP, 0, 1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref.lib.kref_time_pipeline(im.h, cores, K_TOP, 0, 1)
        el = time.perf_counter() - t0
    val = w * h * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": workload_name(w, h),
                   "parallelism": f"{cores} host threads (reference fast_contrast_curve workers)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"full {CONFIG_NAME} image per step, kernel={ref.active_kernel()}"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-budget", type=float, default=12.0,
                    help="seconds of CPU-baseline sampling (rank 0, N=1)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: min(steps, 200)")
    ap.add_argument("--depth", type=int, default=3,
                    help="K1 launches in flight for the device-resident step loop "
                         "(kohler_cuda_set_pipeline_depth; 1 = each launch on all SMs)")
    ap.add_argument("--graph-steps", type=int, default=500,
                    help="N=1: replay the step loop from CUDA graphs of this many consecutive "
                         "steps (PDL edges between them inside the graph); 0 = eager launches")
    ap.add_argument("--band-depth", type=int, default=2,
                    help="N>1: pipeline depth of the band kernels (kohler_cuda_set_pipeline_depth)")
    ap.add_argument("--bucket", type=int, default=8,
                    help="N>1: steps per all-reduce (the partial curves of this many steps "
                         "reduced in one NCCL call, their selections in one launch); 1 = one "
                         "all-reduce per step, overlapped with the next step's band kernel")
    ap.add_argument("--eager-bands", action="store_true",
                    help="N>1 (or --force-bands): launch the band steps eagerly instead of "
                         "replaying them (NCCL all-reduces included) from CUDA graphs")
    ap.add_argument("--force-reduce", action="store_true",
                    help="with --force-bands at N=1: issue the all-reduce anyway (tests)")
    ap.add_argument("--force-bands", action="store_true",
                    help="run the multi-GPU row-band path (NCCL) even at N=1 (launch under "
                         "torchrun; exercises the N>1 code on one GPU, not a scaling number)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    bands = world > 1 or (args.force_bands and args.impl == "ours")
    if world > 1 or bands:
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")

    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    from paper_1707_05062_b200 import Context
    from paper_1707_05062_b200.bands import BandedAnalyzer

    dev = torch.device("cuda", torch.cuda.current_device())
    ctx = Context(dev.index)
    img = make_input("cpu")
    h, w = img.shape
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    stream = torch.cuda.current_stream()

    if not bands:
        pitch = (w + 127) // 128 * 128
        img_bytes = pitch * h
        copies = max(2, (2 * l2) // img_bytes + 1)
        buf = torch.zeros((copies, h, pitch), dtype=torch.uint8, device=dev)
        buf[:, :, :w] = img.to(dev)[None]
        out = {"sums": torch.zeros(256, dtype=torch.int64, device=dev),
               "cards": torch.zeros(256, dtype=torch.int64, device=dev),
               "values": torch.zeros(256, dtype=torch.float64, device=dev),
               "defined": torch.zeros(256, dtype=torch.uint8, device=dev),
               "t0": torch.zeros(1, dtype=torch.int32, device=dev),
               "topk": torch.zeros(K_TOP, dtype=torch.int32, device=dev),
               "topk_count": torch.zeros(1, dtype=torch.int32, device=dev),
               "status": torch.zeros(1, dtype=torch.int32, device=dev)}

        ctx.set_pipeline_depth(args.depth)

        def step(i, st=stream):
            ctx.analyze_batch_device(buf[i % copies], w, h, pitch, img_bytes, 1, K_TOP, out, st)
        launches_per_step = None  # counted after the first step (K1 walk + K3/K4 finish)
        bytes_per_step = w * h
        parallel = ("1 GPU, K1 walk + K3/K4 finish per step (PDL-chained)"
                    + (f"; {args.depth} steps in flight, K1 on 1/{args.depth} of the SMs each "
                       "(kohler_cuda_set_pipeline_depth)" if args.depth > 1 else ""))
    else:
        ba = BandedAnalyzer(ctx, w, h, world, rank, K_TOP)
        ba.always_reduce = args.force_reduce
        ctx.set_pipeline_depth(args.band_depth)
        pitch = (w + 127) // 128 * 128
        rows = ba.rows_held
        band_bytes = max(rows, 1) * pitch
        copies = max(2, (2 * l2) // band_bytes + 1)
        buf = torch.zeros((copies, max(rows, 1), pitch), dtype=torch.uint8, device=dev)
        if rows:
            buf[:, :rows, :w] = img[ba.lo:ba.hi].to(dev)[None]
        bucket = max(1, args.bucket)
        if bucket > 1:
            ba.enable_buckets(bucket)
            out = ba.bout

            def step(i):
                # band K1 of step i into slot i % m; every m steps one async
                # all-reduce of the m partials, then (behind the next bucket's
                # first band kernel) one selection launch for the previous m
                ba.step_bucketed(buf[i % copies], pitch)
            launches_per_step = 2 + 1.0 / bucket  # band K1 + finish per step, a select per bucket
            parallel = (f"row bands x{world} + 1-row halo; NCCL all-reduce of the 512 u64 partials "
                        f"of {bucket} steps at once (async, overlapped with the next bucket's band "
                        "kernels), one selection launch per bucket; strong scaling")
        else:
            out = ba.out

            def step(i):
                # all-reduce of step i overlapped with step i + 1's band K1; the
                # selection of step i runs behind it (drain() after the last step)
                ba.step_pipelined(i, buf[i % copies], pitch)
            launches_per_step = 3  # band K1 + finish, select
            parallel = (f"row bands x{world} + 1-row halo, NCCL all-reduce of 512 u64 overlapped "
                        "with the next step's band kernel, strong scaling")
        bytes_per_step = w * h  # whole job processes the full image per step

    def drain():
        if bands:
            if getattr(ba, "m", 0):
                ba.drain_buckets()
            else:
                ba.drain()

    def first_result():
        tk = out["topk"][0] if out["topk"].dim() == 2 else out["topk"]
        return int(out["t0"][0]), tk[: int(out["topk_count"][0])].tolist()

    # correctness gate before timing (bench.cpp:141-161 semantics)
    step(0)
    drain()
    torch.cuda.synchronize()
    if launches_per_step is None:
        launches_per_step = ctx.last_launch_count()
    if rank == 0:
        import oracle
        exp = oracle.Oracle().analyze(img.numpy(), K_TOP)
        got_t0, got_tk = first_result()
        ok = got_t0 == exp["t0"] and got_tk == exp["topk"]
        if not bands:
            ok = ok and np.array_equal(out["sums"].cpu().numpy().view(np.uint64), exp["sum"]) \
                and np.array_equal(out["cards"].cpu().numpy().view(np.uint64), exp["card"])
        if not ok:
            raise SystemExit("refusing to time: GPU result differs from the oracle")

    for i in range(args.warmup):
        step(i)
    drain()
    torch.cuda.synchronize()

    # A step is a few launches (~9-15 us of host API time per step through
    # ctypes, as long as the device step): replay the loop from CUDA graphs of
    # G consecutive steps, captured through the same public device API on the
    # capture stream (N=1: PDL edges between the steps inside; N>1: the band
    # kernels, the NCCL all-reduces and the selections with their overlap)
    graph = None
    # (longer graphs: fewer pipeline drains at graph boundaries -- C2 at
    # depth 3: 60 steps 11.80 us/step, 120: 11.52, 250: 11.39, 500: 11.34)
    G = min(args.graph_steps, args.steps) if (not bands or not args.eager_bands) else 0
    if G > 0:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cap = torch.cuda.current_stream()
                for j in range(G):
                    if bands:
                        step(j)
                    else:
                        step(j, cap)
                drain()
            graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # keep a (slower, eager) bench line rather than none
            print(f"bench: CUDA-graph capture failed ({type(exc).__name__}: {exc}); eager steps",
                  file=sys.stderr, flush=True)
            graph = None
            torch.cuda.synchronize()
            if bands:
                ba._pending = None
                ba._bpending, ba._bfill = None, 0

    sampler = ClockSampler(dev.index if world == 1 else local).start()
    sampler.wait_first()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    i = 0
    if graph is not None:
        with torch.cuda.stream(stream):
            while i + G <= args.steps:
                graph.replay()
                i += G
    for i in range(i, args.steps):
        step(i)
    drain()  # the last step's selection is inside the timed region
    e1.record(stream)
    e1.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if rank == 0:
        # the replayed / pipelined steps left the last image's full result
        ok = first_result() == (exp["t0"], exp["topk"])
        if not bands:
            ok = ok and np.array_equal(out["sums"].cpu().numpy().view(np.uint64), exp["sum"])
        if not ok:
            raise SystemExit("timed steps produced a result that differs from the oracle")
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = bytes_per_step * args.steps / (ms * 1e-3) / 1e9

    # kernel-level timing of K1 alone (its own events, same stream), for the roofline
    kern_ms = None
    if not bands:
        # one K1 launch per step: with d launches in flight the step time is
        # K1's effective (throughput) time per launch
        kern_ms = ms_step
    else:
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        nk = min(args.steps, 200)
        k0.record(stream)
        for i in range(nk):
            if ba.r1 > ba.r0:
                ctx.band_curve_device(buf[i % copies], w, pitch, h, ba.r0, ba.r1,
                                      ba.curve.data_ptr(), ba.curve.data_ptr() + 2048, stream)
        k1.record(stream)
        k1.synchronize()
        kern_ms = k0.elapsed_time(k1) / nk
    peak, peak_src = peaks()
    kbytes = w * h if not bands else (ba.r1 - ba.r0) * w
    achieved = kbytes / (kern_ms * 1e-3) / 1e9

    # N > 1: every rank uploads its band (own rows + halo) from pinned host
    # memory each step, runs K1 on it, all-reduces, selects and reads the
    # thresholds back; wall clock, max over ranks
    e2e_bands = None
    if bands:
        try:
            e2e_bands = measure_e2e_bands(ba, img, args, dev, pitch)
        except Exception as exc:  # keep the device-timed line
            e2e_bands = {"error": f"{type(exc).__name__}: {exc}"}

    line = None
    if rank == 0:
        e2e = None
        cpu = None
        if not bands:
            ctx.set_pipeline_depth(1)  # the host API call is measured one call at a time
            e2e = measure_e2e(ctx, img, args)
        else:
            e2e = e2e_bands
        if world == 1:  # the CPU baseline: rank 0 at N=1 only
            med, runs, cores, kern = cpu_reference_time(img.numpy(), args.cpu_budget, 2000)
            cpu = {"value": w * h / med / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"full {CONFIG_NAME} image, median of {runs} runs (1 warm-up), "
                             f"workers={cores}, kernel={kern}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": workload_name(w, h),
                       "parallelism": parallel,
                       "l2": f"rotating {copies} input copies ({copies * buf[0].numel() / 1e6:.0f} MB"
                             f" > 2x L2 {l2 / 1e6:.0f} MB)",
                       "launch": (f"CUDA-graph replay, {G} steps per graph (PDL edges inside), "
                                  "captured through kohler_cuda_analyze_batch_device"
                                  if graph is not None else "eager"),
                       "pipeline_depth": args.depth if not bands else 1},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(),
                         "kernel": "walk_kernel<true> (K1; finish_kernel K3/K4 PDL-overlapped)" if not bands
                         else "walk_kernel<true> band partial (K1)",
                         "algorithmic_bytes_per_launch": kbytes, "kernel_ms": kern_ms,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def measure_e2e_bands(ba, img, args, dev, pitch):
    """e2e at N > 1 through the band API: pinned host rows of this rank's
    band -> H2D -> K1 band partial -> NCCL all-reduce -> device selection ->
    D2H of t0 / top-k, every step; wall clock per rank, max over ranks."""
    h, w = img.shape
    rows = max(ba.rows_held, 1)
    host = torch.zeros((rows, pitch), dtype=torch.uint8).pin_memory()
    if ba.rows_held:
        host[:, :w] = img[ba.lo:ba.hi]
    dbuf = torch.empty((rows, pitch), dtype=torch.uint8, device=dev)
    res = torch.zeros(2 + K_TOP, dtype=torch.int32).pin_memory()
    n = args.e2e_steps or min(args.steps, 200)

    def call():
        dbuf.copy_(host, non_blocking=True)
        ba.step(dbuf, pitch)
        res[0:1].copy_(ba.out["t0"], non_blocking=True)
        res[1:2].copy_(ba.out["topk_count"], non_blocking=True)
        res[2:].copy_(ba.out["topk"], non_blocking=True)
        torch.cuda.current_stream().synchronize()
    for _ in range(3):
        call()
    dist.barrier()
    st = time.perf_counter()
    for _ in range(n):
        call()
    el = time.perf_counter() - st
    t = torch.tensor([el, float(rows * pitch), 4.0 * (2 + K_TOP)], dtype=torch.float64, device=dev)
    tb = t.clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(tb, op=dist.ReduceOp.SUM)
    el = float(t[0].item())
    return {"value": w * h * n / el / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int(tb[1].item()), "d2h_bytes_per_step": int(tb[2].item()),
            "steps": n, "path": "per rank: pinned band rows -> H2D -> band K1 -> NCCL all-reduce "
                                "-> select -> D2H, wall clock, max over ranks"}


def measure_e2e(ctx, img, args):
    """Same metric through the public host C ABI, every step: the image from
    pinned host memory -> H2D -> K1 + finish -> D2H of curve, mean curve and
    thresholds.  Headline: the streaming API (kohler_cuda_submit /
    kohler_cuda_collect, two steps in flight, so step i + 1's upload runs
    under step i's kernels); also reported: the synchronous
    kohler_cuda_analyze (one blocking call per step).  Wall clock, best of
    three blocks of n steps each (a shared box's host / PCIe jitter)."""
    import ctypes as C
    h, w = img.shape
    pinned = torch.empty((h, w), dtype=torch.uint8).pin_memory()
    pinned.copy_(img)
    n = args.e2e_steps or min(args.steps, 200)
    res = {k: np.zeros(256, np.uint64) for k in ("s", "c")}
    vals = np.zeros(256, np.float64)
    dfn = np.zeros(256, np.uint8)
    t0 = np.zeros(1, np.int32)
    tk = np.zeros(K_TOP, np.int32)
    cnt = np.zeros(1, np.int32)
    stt = np.zeros(1, np.int32)
    lib = ctx._lib
    hd = ctx.handle
    ptr = pinned.data_ptr()
    outs = (res["s"].ctypes.data, res["c"].ctypes.data, vals.ctypes.data, dfn.ctypes.data,
            t0.ctypes.data, tk.ctypes.data, cnt.ctypes.data, stt.ctypes.data)
    ticket = C.c_longlong(-1)

    def sync_call():
        return lib.kohler_cuda_analyze(hd, ptr, w, h, w, K_TOP, *outs[:7])

    def submit():
        if lib.kohler_cuda_submit(hd, ptr, 1, w, h, w, w * h, K_TOP, C.byref(ticket)):
            raise RuntimeError("e2e submit failed")
        return ticket.value

    def collect(t):
        if lib.kohler_cuda_collect(hd, t, *outs):
            raise RuntimeError("e2e collect failed")

    def stream_block():
        prev = submit()
        for _ in range(n - 1):
            nxt = submit()
            collect(prev)
            prev = nxt
        collect(prev)

    def sync_block():
        for _ in range(n):
            if sync_call() not in (0, 1):
                raise RuntimeError("e2e call failed")

    def best(block):
        block()  # warm-up block
        el = []
        for _ in range(3):
            st = time.perf_counter()
            block()
            el.append(time.perf_counter() - st)
        return min(el)
    el_sync = best(sync_block)
    el = best(stream_block)
    if int(t0[0]) < 0 or int(cnt[0]) < 1:
        raise RuntimeError("e2e produced no thresholds")
    d2h = 256 * 8 * 2 + 256 * 8 + 256 + 4 * 3 + 4 * K_TOP
    return {"value": w * h * n / el / 1e9, "unit": UNIT, "h2d_bytes_per_step": w * h,
            "d2h_bytes_per_step": d2h, "steps": n,
            "call_us": el / n * 1e6,
            "sync_value": w * h * n / el_sync / 1e9, "sync_call_us": el_sync / n * 1e6,
            "path": "kohler_cuda_submit / kohler_cuda_collect (host C ABI, two steps in flight), "
                    "pinned input, wall clock, best of 3 blocks; sync_* = kohler_cuda_analyze"}


if __name__ == "__main__":
    main()

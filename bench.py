#!/usr/bin/env python3
"""Benchmark of the Köhler contrast-curve hot path on B200.

Headline workload (BASELINE.json configs[1], "C2"): one 5184x3456 uint8 image
(gradient + 40 ellipses + N(0,5^2), seeded), full N4 curve (u64 sum/count),
IEEE f64 mean curve, optimal threshold and top-6 local maxima.  One step =
one pass of that pipeline over the image.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--no-per-config]

--gpus N > 1 without torchrun: the script relaunches itself under
``torch.distributed.run`` with N processes (one per GPU, NCCL, 127.0.0.1).

N = 1: per step one K1 launch: the walk accumulates, and the CTA whose flush
lands last runs K3 (reconstruct) + K4 (select); PDL-chained; pipeline depth
3 (three steps in flight on a third of the SMs each).
N > 1: the image is split into row bands with a one-row halo
(proj/src/fast.cpp:42-57); per step each rank runs K1 on its band, the 512
u64 partials of 8 steps are merged by one NCCL all-reduce (asynchronous,
overlapped with the next steps' bands), then one selection launch — strong
scaling (the image is fixed).

Timing (the same for every line): the W warm-up steps and the K timed steps
are captured into ONE CUDA graph through the public device API; the start
event is an event-record node on a side branch behind step W (the step
chain itself is not cut, so the timed steps run in the same steady-state
pipeline as in a long run) and the stop event follows step W+K's selection.
The graph is replayed a few times untimed first (clock ramp), then once more
with no host sync in between; barrier + synchronize on both sides, CUDA
events, max over ranks.  Inputs rotate through copies totalling > 2x L2
(126 MB) or are larger than L2 themselves.  The result of the last timed step
is re-checked against the oracle after timing; a mismatch before or after
refuses the line.

per_config (default on): C1 (N=1), C3 shards, C4 bands, C5 shards at the
same N, each with Gpx/s and %roofline, the all-reduce time of the band path,
and at N=1 the reference CPU implementation as shipped (sequential calls,
all cores as workers: proj/src/bench.cpp:263-277) and frame-parallel
(workers = 1 per image over all cores) on a bounded sample.  The per-config
CPU runs double as the correctness gate of those configs.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libkohler_ref.so, compiled from the reference sources) on this
host's cores with the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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


def ncu_traffic(name=CONFIG_NAME):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    --set full capture summary (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(name)
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
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

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


# ---------------------------------------------------------------------------
# timing: W warm-up + K timed steps in one graph, event nodes inside
# ---------------------------------------------------------------------------
class GraphSteps:
    """W warm-up steps and K timed steps captured into ONE CUDA graph.

    e0 is an external event-record node on a side stream forked right after
    step W's work, so the chain of steps (PDL edges between the kernels) is
    not cut at the start of the timed region; e1 is recorded after the last
    step (and ``drain``, which completes a pipelined / bucketed last step).
    Elapsed(e0, e1) is therefore the time of exactly K steps of the steady
    pipeline, with the pipeline drain of the last steps inside it."""

    def __init__(self, step, W, K, drain=None):
        self.W, self.K = W, K
        self.e0 = torch.cuda.Event(enable_timing=True, external=True)
        self.e1 = torch.cuda.Event(enable_timing=True, external=True)
        side = torch.cuda.Stream()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            cap = torch.cuda.current_stream()
            for i in range(W):
                step(i)
            fork = torch.cuda.Event()
            fork.record(cap)
            side.wait_event(fork)
            self.e0.record(side)
            join = torch.cuda.Event()
            join.record(side)
            for i in range(W, W + K):
                step(i)
            if drain is not None:
                drain()
            cap.wait_event(join)
            self.e1.record(cap)

    def run(self, world: int, prewarm_s: float = 0.03) -> float:
        """Replay untimed for ~prewarm_s (clock ramp; at least once), then the
        timed replay with no host sync in between.  -> ms of the K steps,
        max over ranks."""
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.graph.replay()
        self.e1.synchronize()
        one = max(time.perf_counter() - t0, 1e-6)
        for _ in range(max(1, min(200, int(prewarm_s / one)))):
            self.graph.replay()
        self.graph.replay()  # the timed one: e0 / e1 of this replay
        self.e1.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = self.e0.elapsed_time(self.e1)
        return max_over_ranks(ms, world)


def max_over_ranks(x: float, world: int) -> float:
    if world <= 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world <= 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_ranks_ok(ok: bool, world: int) -> bool:
    if world <= 1:
        return bool(ok)
    t = torch.tensor([0 if ok else 1], dtype=torch.int32, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(t.item()) == 0


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


def spawn(args) -> int:
    """--gpus N > 1 without torchrun: relaunch under torch.distributed.run."""
    if torch.cuda.device_count() < args.gpus:
        log(f"bench: --gpus {args.gpus} but only {torch.cuda.device_count()} GPU(s) visible")
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def gpu_local_cpus(dev: int):
    """CPUs of the NUMA node the GPU hangs off (sysfs), or None."""
    try:
        bus = torch.cuda.get_device_properties(dev).pci_bus_id.lower()
    except Exception:
        return None
    for cand in (bus, bus[4:] if len(bus) > 12 else "0000:" + bus):
        p = f"/sys/bus/pci/devices/{cand}/local_cpulist"
        if os.path.exists(p):
            out = []
            for part in open(p).read().strip().split(","):
                if "-" in part:
                    a, b = part.split("-")
                    out += range(int(a), int(b) + 1)
                elif part:
                    out.append(int(part))
            return out or None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-budget", type=float, default=8.0,
                    help="seconds of CPU-baseline sampling for the headline (rank 0, N=1)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: max(min(steps, 200), 20)")
    ap.add_argument("--depth", type=int, default=3,
                    help="K1 launches in flight for the device-resident step loop "
                         "(kohler_cuda_set_pipeline_depth; 1 = each launch on all SMs)")
    ap.add_argument("--band-depth", type=int, default=2,
                    help="N>1: pipeline depth of the band kernels (kohler_cuda_set_pipeline_depth)")
    ap.add_argument("--bucket", type=int, default=8,
                    help="N>1: steps per all-reduce (the partial curves of this many steps "
                         "reduced in one NCCL call, their selections in one launch); 1 = one "
                         "all-reduce per step, overlapped with the next step's band kernel")
    ap.add_argument("--force-reduce", action="store_true",
                    help="with --force-bands at N=1: issue the all-reduce anyway (tests)")
    ap.add_argument("--force-bands", action="store_true",
                    help="run the multi-GPU row-band path (NCCL) even at N=1 (launch under "
                         "torchrun; exercises the N>1 code on one GPU, not a scaling number)")
    ap.add_argument("--no-per-config", action="store_true", help="headline (C2) line only")
    ap.add_argument("--per-config", default="C1,C3,C4,C5",
                    help="configs of the per_config block")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn(args))

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
    sampler = ClockSampler(dev.index).start()
    sampler.wait_first()

    if not bands:
        pitch = (w + 127) // 128 * 128
        img_bytes = pitch * h
        copy_bytes = img_bytes
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

        def step(i):
            ctx.analyze_batch_device(buf[i % copies], w, h, pitch, img_bytes, 1, K_TOP, out)
        drain = None
        launches_per_step = None  # counted after the first step (one K1: walk + in-CTA K3/K4)
        parallel = ("1 GPU, one K1 per step (walk; K3/K4 by its last-flushing CTA; PDL-chained)"
                    + (f"; {args.depth} steps in flight, K1 on 1/{args.depth} of the SMs each "
                       "(kohler_cuda_set_pipeline_depth)" if args.depth > 1 else ""))
    else:
        ba = BandedAnalyzer(ctx, w, h, world, rank, K_TOP)
        ba.always_reduce = args.force_reduce
        ctx.set_pipeline_depth(args.band_depth)
        pitch = (w + 127) // 128 * 128
        rows = ba.rows_held
        band_bytes = max(rows, 1) * pitch
        copy_bytes = band_bytes
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
            drain = ba.drain_buckets
            launches_per_step = 1 + 1.0 / bucket  # band K1 (self-finishing) per step, a select per bucket
            parallel = (f"row bands x{world} + 1-row halo; NCCL all-reduce of the 512 u64 partials "
                        f"of {bucket} steps at once (async, overlapped with the next bucket's band "
                        "kernels), one selection launch per bucket; strong scaling")
        else:
            out = ba.out

            def step(i):
                ba.step_pipelined(i, buf[i % copies], pitch)
            drain = ba.drain
            launches_per_step = 2  # band K1 (self-finishing), select
            parallel = (f"row bands x{world} + 1-row halo, NCCL all-reduce of 512 u64 overlapped "
                        "with the next step's band kernel, strong scaling")

    def first_result():
        tk = out["topk"][0] if out["topk"].dim() == 2 else out["topk"]
        t0v = out["t0"][0] if out["t0"].dim() == 1 else out["t0"]
        cnt = out["topk_count"][0] if out["topk_count"].dim() == 1 else out["topk_count"]
        return int(t0v), tk[: int(cnt)].tolist()

    def last_result():
        if bands and getattr(ba, "m", 0):
            j = (args.warmup + args.steps - 1) % ba.m
            return int(out["t0"][j]), out["topk"][j][: int(out["topk_count"][j])].tolist()
        return first_result()

    # correctness gate before timing (bench.cpp:141-161 semantics)
    step(0)
    if drain is not None:
        drain()
    torch.cuda.synchronize()
    if launches_per_step is None:
        launches_per_step = ctx.last_launch_count()
    exp = None
    if rank == 0:
        import oracle
        exp = oracle.Oracle().analyze(img.numpy(), K_TOP)
        got = first_result() if not (bands and getattr(ba, "m", 0)) else \
            (int(out["t0"][0]), out["topk"][0][: int(out["topk_count"][0])].tolist())
        ok = got == (exp["t0"], exp["topk"])
        if not bands:
            ok = ok and np.array_equal(out["sums"].cpu().numpy().view(np.uint64), exp["sum"]) \
                and np.array_equal(out["cards"].cpu().numpy().view(np.uint64), exp["card"])
        if not ok:
            raise SystemExit("refusing to time: GPU result differs from the oracle")
    if bands and getattr(ba, "m", 0):
        ba._bblock, ba._bfill, ba._bpending = 0, 0, None

    timer = None
    try:
        timer = GraphSteps(step, args.warmup, args.steps, drain)
    except Exception as exc:
        log(f"bench: CUDA-graph capture failed ({type(exc).__name__}: {exc}); eager steps")
        torch.cuda.synchronize()
        if bands:
            ba._pending = None
            ba._bblock, ba._bfill, ba._bpending = 0, 0, None
    if timer is not None:
        ms = timer.run(world)
        launch = (f"one CUDA graph of {args.warmup} warm-up + {args.steps} timed steps captured "
                  "through kohler_cuda_analyze_batch_device" if not bands else
                  f"one CUDA graph of {args.warmup} warm-up + {args.steps} timed band steps "
                  "(NCCL all-reduces inside)")
        launch += ("; e0 = event-record node behind step W on a side branch, e1 after the last "
                   "step: K steps of the steady pipeline")
    else:
        for i in range(args.warmup):
            step(i)
        if drain is not None:
            drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.warmup, args.warmup + args.steps):
            step(i)
        if drain is not None:
            drain()
        e1.record()
        e1.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1), world)
        launch = "eager"
    clocks = sampler.stop()
    if rank == 0:
        ok = last_result() == (exp["t0"], exp["topk"])
        if not bands:
            ok = ok and np.array_equal(out["sums"].cpu().numpy().view(np.uint64), exp["sum"])
        if not ok:
            raise SystemExit("timed steps produced a result that differs from the oracle")
    ms_step = ms / args.steps
    value = w * h * args.steps / (ms * 1e-3) / 1e9

    # kernel-level time of K1 for the roofline
    if not bands:
        # one K1 launch per step: with d launches in flight the step time is
        # K1's effective (throughput) time per launch
        kern_ms = ms_step
        kbytes = w * h
    else:
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        nk = min(args.steps, 200)
        st = torch.cuda.current_stream()
        k0.record(st)
        for i in range(nk):
            if ba.r1 > ba.r0:
                ctx.band_curve_device(buf[i % copies], w, pitch, h, ba.r0, ba.r1,
                                      ba.curve.data_ptr(), ba.curve.data_ptr() + 2048, st)
        k1.record(st)
        k1.synchronize()
        kern_ms = k0.elapsed_time(k1) / nk
        kbytes = (ba.r1 - ba.r0) * w
    peak, peak_src = peaks()
    achieved = kbytes / (kern_ms * 1e-3) / 1e9

    e2e_bands = None
    if bands:
        try:
            e2e_bands = measure_e2e_bands(ba, img, args, dev, pitch)
        except Exception as exc:  # keep the device-timed line
            e2e_bands = {"error": f"{type(exc).__name__}: {exc}"}

    del buf
    torch.cuda.empty_cache()
    per_config = None
    if not args.no_per_config:
        names = [x.strip() for x in args.per_config.split(",") if x.strip()]
        per_config = {}
        for name in names:
            try:
                per_config[name] = measure_config(ctx, name, world, rank, dev, args)
            except Exception as exc:
                per_config[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.empty_cache()
            if world > 1:
                dist.barrier()
        per_config = {k: v for k, v in per_config.items() if v is not None}

    line = None
    if rank == 0:
        cpu = None
        if not bands:
            ctx.set_pipeline_depth(1)  # the host API call is measured one call at a time
            e2e = measure_e2e(ctx, img, args, dev.index)
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
                       "l2": f"rotating {copies} input copies ({copies * copy_bytes / 1e6:.0f} MB"
                             f" > 2x L2 {l2 / 1e6:.0f} MB)",
                       "launch": launch,
                       "pipeline_depth": args.depth if not bands else args.band_depth},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(),
                         "kernel": "walk_kernel<true> (K1; K3/K4 in its last-flushing CTA)" if not bands
                         else "walk_kernel<true> band partial (K1)",
                         "algorithmic_bytes_per_launch": kbytes, "kernel_ms": kern_ms,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": clocks,
        }
        if per_config is not None:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# per-config block
# ---------------------------------------------------------------------------
PER_CONFIG_STEPS = {"C1": 300, "C3": 10, "C4": 20, "C5": 10}
CPU_SAMPLE = {"C1": None, "C3": 64, "C4": None, "C5": 4096}


def cpu_config_baselines(x_host: np.ndarray, name: str, ksel: int):
    """Reference CPU implementation on a bounded sample: as shipped
    (sequential calls, workers = all cores: bench.cpp:263-277) and, for
    batches, frame-parallel (workers = 1 per image, one host thread per
    core).  -> (baselines dict, reference outputs of the sample)."""
    import oracle
    ref = oracle.Reference()
    cores = os.cpu_count() or 1
    n = x_host.shape[0]
    res = {}
    outs = None
    single = n == 1
    runs = 2 if name == "C4" else (30 if name == "C1" else 1)
    t = []
    for r in range(runs + 1):
        s = time.perf_counter()
        o = ref.analyze_batch(x_host, k=ksel, workers=cores, threads=1)
        if r:
            t.append(time.perf_counter() - s)
        outs = o
    el = statistics.median(t)
    px = x_host.size
    res["as_shipped"] = {"value": px / el / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{n} image(s) of {name}, sequential calls, workers={cores}, "
                                   f"median of {runs} (1 warm-up)"}
    if not single:
        s = time.perf_counter()
        o2 = ref.analyze_batch(x_host, k=ksel, workers=1, threads=cores)
        el2 = time.perf_counter() - s
        res["frame_parallel"] = {"value": px / el2 / 1e9, "unit": UNIT, "cores": cores,
                                 "kind": "reference",
                                 "sample": f"{n} images of {name}, workers=1, {cores} threads"}
        for key in ("sums", "cards", "t0", "topk_count"):
            if not np.array_equal(o2[key], outs[key]):
                raise RuntimeError("reference as-shipped and frame-parallel disagree")
    return res, outs


def measure_config(ctx, name: str, world: int, rank: int, dev, args):
    """One per_config entry: the config's device-resident throughput at this
    N (C3/C5: image shards, C4: row bands + NCCL, C1: N=1 only), gated by the
    reference on a sample (rank 0) and re-checked after timing."""
    from paper_1707_05062_b200 import synth
    from paper_1707_05062_b200.bands import BandedAnalyzer
    from paper_1707_05062_b200.shard import shard_bounds
    if name == "C1" and world > 1:
        return None
    cfg = synth.CONFIGS[name]
    x = synth.generate(name, device=dev)  # (n, h, w) u8 on the device
    n, h, w = x.shape
    K = PER_CONFIG_STEPS[name]
    W = 3
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    entry = {"workload": f"{name}: {cfg.desc}, seed {cfg.seed:#x}", "images": n, "w": w, "h": h,
             "steps": K, "warmup": W}
    peak, _ = peaks()
    ksel = K_TOP

    # ---- correctness gate + CPU baselines (rank 0) -------------------------
    sample = CPU_SAMPLE[name]
    idx = np.arange(n) if sample is None else np.unique(np.linspace(0, n - 1, sample).astype(int))
    want = None
    if rank == 0:
        xh = x[torch.as_tensor(idx, device=dev)].cpu().numpy()
        if world == 1:
            cpu, want = cpu_config_baselines(xh, name, ksel)
            entry["cpu_baseline"] = cpu
        else:
            import oracle
            want = oracle.Reference().analyze_batch(xh, k=ksel, workers=1)

    def check(res_sums, res_t0, res_cnt, res_topk, imgs):
        """imgs: global indices the result rows belong to (rank 0)."""
        pos = {int(g): j for j, g in enumerate(idx)}
        for row, g in enumerate(imgs):
            j = pos.get(int(g))
            if j is None:
                continue
            if res_sums is not None and not np.array_equal(res_sums[row], want["sums"][j]):
                return False
            if int(res_t0[row]) != int(want["t0"][j]) or int(res_cnt[row]) != int(want["topk_count"][j]):
                return False
            c = int(res_cnt[row])
            if list(res_topk[row][:c]) != list(want["topk"][j][:c]):
                return False
        return True

    if name == "C4" and world > 1:
        # row bands + one NCCL all-reduce per bucket of steps
        ba = BandedAnalyzer(ctx, w, h, world, rank, ksel)
        ctx.set_pipeline_depth(1)
        band = x[0, ba.lo:ba.hi].contiguous() if ba.rows_held else torch.zeros((1, w), dtype=torch.uint8, device=dev)
        ba.enable_buckets(4)

        def step(i):
            ba.step_bucketed(band, w)
        ba.step_bucketed(band, w)
        ba.drain_buckets()
        torch.cuda.synchronize()
        ok = True
        if rank == 0:
            ok = check(None, ba.bout["t0"].cpu().numpy(), ba.bout["topk_count"].cpu().numpy(),
                       ba.bout["topk"].cpu().numpy(), [0])
        if not all_ranks_ok(ok, world):
            return {"error": "refusing to time: band result differs from the reference"}
        ba._bblock, ba._bfill, ba._bpending = 0, 0, None
        timer = GraphSteps(step, W, K, ba.drain_buckets)
        ms = timer.run(world)
        # the NCCL all-reduce alone (4 KB partials of one step), for the record
        ar = torch.zeros(512, dtype=torch.int64, device=dev)
        for _ in range(5):
            dist.all_reduce(ar)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(50):
            dist.all_reduce(ar)
        a1.record()
        a1.synchronize()
        entry["allreduce_us"] = max_over_ranks(a0.elapsed_time(a1) / 50 * 1e3, world)
        entry["parallelism"] = f"row bands x{world} + 1-row halo, NCCL all-reduce per 4 steps"
        entry["scaling"] = "strong"
        px_step = w * h
        launches = 2 + 0.25
    else:
        i0, i1 = shard_bounds(n, world, rank)
        loc = i1 - i0
        xs = x[i0:i1]
        copies = 1
        if loc and xs.numel() < 2 * l2:
            copies = int(2 * l2 // xs.numel()) + 1
        bufs = xs[None].expand(copies, *xs.shape).contiguous() if copies > 1 else xs[None]
        ctx.set_pipeline_depth(3 if name == "C1" else 1)
        o = {"sums": torch.zeros((max(loc, 1), 256), dtype=torch.int64, device=dev),
             "cards": torch.zeros((max(loc, 1), 256), dtype=torch.int64, device=dev),
             "t0": torch.zeros(max(loc, 1), dtype=torch.int32, device=dev),
             "topk": torch.zeros((max(loc, 1), ksel), dtype=torch.int32, device=dev),
             "topk_count": torch.zeros(max(loc, 1), dtype=torch.int32, device=dev),
             "status": torch.zeros(max(loc, 1), dtype=torch.int32, device=dev)}

        def step(i):
            if loc:
                ctx.analyze_batch_device(bufs[i % copies], w, h, w, w * h, loc, ksel, o)
        step(0)
        torch.cuda.synchronize()
        launches = ctx.last_launch_count() if loc else 0

        def verify():
            # rank 0 checks the sampled images of its own shard; every rank
            # checks its shard's first images against the C oracle restatement
            good = True
            if loc and w * h <= (1 << 22):
                import oracle
                orc = oracle.Oracle()
                for j in range(min(2, loc)):
                    e = orc.analyze(xs[j].cpu().numpy(), ksel)
                    good = good and np.array_equal(o["sums"][j].cpu().numpy().view(np.uint64), e["sum"]) \
                        and int(o["t0"][j]) == e["t0"]
            if rank == 0 and loc:
                mine = [g for g in idx if i0 <= g < i1]
                sel = torch.as_tensor([g - i0 for g in mine], device=dev, dtype=torch.int64)
                good = good and check(o["sums"][sel].cpu().numpy().view(np.uint64),
                                      o["t0"][sel].cpu().numpy(), o["topk_count"][sel].cpu().numpy(),
                                      o["topk"][sel].cpu().numpy(), mine)
            return all_ranks_ok(good, world)
        if not verify():
            return {"error": "refusing to time: GPU result differs from the reference"}
        timer = GraphSteps(step, W, K)
        ms = timer.run(world)
        if not verify():
            return {"error": "timed steps produced a result that differs from the reference"}
        entry["parallelism"] = (f"image shards x{world} (contiguous, no collective)" if world > 1
                                else "1 GPU, whole batch per step")
        if name == "C1":
            entry["parallelism"] += "; pipeline depth 3"
        entry["scaling"] = "strong"
        entry["l2"] = (f"{copies} rotating copies" if copies > 1 else "input > 2x L2")
        px_step = n * w * h
    entry["ms_per_step"] = ms / K
    entry["value"] = px_step * K / (ms * 1e-3) / 1e9
    entry["unit"] = UNIT
    entry["images_per_s"] = n * K / (ms * 1e-3)
    entry["roofline"] = {"bound": "hbm", "achieved": entry["value"], "peak": peak, "unit": "GB/s",
                         "frac": entry["value"] / peak, "traffic": ncu_traffic(name)}
    entry["gpu_launches"] = int(round(sum_over_ranks(launches, world) * K))
    return entry


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
    n = args.e2e_steps or max(min(args.steps, 200), 20)

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


def measure_e2e(ctx, img, args, dev_index):
    """Same metric through the public host C ABI, every step: the image from
    pinned host memory -> H2D -> K1 (+ K3/K4) -> D2H of curve, mean curve and
    thresholds.  Headline: the streaming API (kohler_cuda_submit /
    kohler_cuda_collect, two steps in flight, so step i + 1's upload runs
    under step i's kernels); also reported: the synchronous
    kohler_cuda_analyze (one blocking call per step).  The host thread is
    placed on the GPU's NUMA node while the pinned buffer is allocated and
    the calls run (pinned pages first-touched there), and the box's raw
    pinned H2D copy rate is recorded beside it (the floor of this path).
    Wall clock, best of five blocks of n steps each (a box's pinned H2D rate
    has slow stretches of tens of milliseconds, profiles/r02e)."""
    import ctypes as C
    h, w = img.shape
    old_aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    local = gpu_local_cpus(dev_index)
    placed = None
    if local and old_aff is not None:
        try:
            os.sched_setaffinity(0, local)
            placed = f"{len(local)} CPUs of the GPU's NUMA node"
        except OSError:
            placed = None
    try:
        pinned = torch.empty((h, w), dtype=torch.uint8).pin_memory()
        pinned.copy_(img)
        n = args.e2e_steps or max(min(args.steps, 200), 20)
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
            for _ in range(5):
                st = time.perf_counter()
                block()
                el.append(time.perf_counter() - st)
            return min(el)
        el_sync = best(sync_block)
        el = best(stream_block)
        if int(t0[0]) < 0 or int(cnt[0]) < 1:
            raise RuntimeError("e2e produced no thresholds")
        # the box's pinned H2D copy rate (the floor of this path)
        dst = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            dst.copy_(pinned, non_blocking=True)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(10):
            dst.copy_(pinned, non_blocking=True)
        c1.record()
        c1.synchronize()
        h2d_gbs = w * h * 10 / (c0.elapsed_time(c1) * 1e-3) / 1e9
    finally:
        if placed and old_aff is not None:
            os.sched_setaffinity(0, old_aff)
    d2h = 256 * 8 * 2 + 256 * 8 + 256 + 4 * 3 + 4 * K_TOP
    return {"value": w * h * n / el / 1e9, "unit": UNIT, "h2d_bytes_per_step": w * h,
            "d2h_bytes_per_step": d2h, "steps": n,
            "call_us": el / n * 1e6,
            "sync_value": w * h * n / el_sync / 1e9, "sync_call_us": el_sync / n * 1e6,
            "box_pinned_h2d_gbs": h2d_gbs,
            "host_placement": placed or "unpinned (NUMA node of the GPU unknown)",
            "path": "kohler_cuda_submit / kohler_cuda_collect (host C ABI, two steps in flight), "
                    "pinned input, wall clock, best of 5 blocks; sync_* = kohler_cuda_analyze"}


if __name__ == "__main__":
    main()

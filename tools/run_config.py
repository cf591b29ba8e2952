"""Run / time one config through the device API (for ncu, sanitizer and the
per-config throughput table in DESIGN.md)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_05062_b200 import Context, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--time", action="store_true")
ap.add_argument("--depth", type=int, default=1, help="kohler_cuda_set_pipeline_depth")
ap.add_argument("--graph", type=int, default=0,
                help="replay the timed loop from CUDA graphs of this many calls (launch-bound "
                     "configs: removes the per-call Python/ctypes issue cost)")
ap.add_argument("--rgb", action="store_true",
                help="colour ingest: time the pipeline on an RGB version of the config "
                     "(channels: the grey map shifted by 3 px, itself, its negative)")
ap.add_argument("--segment", type=int, default=-1,
                help=">= 0: time the segmentation pipeline instead (0: curve -> {t0} -> "
                     "two-class quantize per image, bench.cpp:266-281; k: top-k quantize)")
a = ap.parse_args()
x = synth.generate(a.config, device="cuda")
n, h, w = x.shape
copies = 1
l2 = torch.cuda.get_device_properties(0).L2_cache_size
if x.numel() < 2 * l2:  # rotate copies so every step reads HBM
    copies = int(2 * l2 // x.numel()) + 1
    x = torch.stack([x] * copies)
else:
    x = x[None]
ctx = Context(0)
ctx.set_pipeline_depth(a.depth)
k = 6
out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
       "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
       "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
       "topk": torch.zeros((n, k), dtype=torch.int32, device="cuda"),
       "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
       "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
if a.rgb:
    xr = torch.stack([torch.roll(x, 3, dims=-1), x, 255 - x], dim=-1).contiguous()

    def call(i):
        ctx.analyze_rgb_batch_device(xr[i % copies], w, h, 3 * w, 3 * w * h, n, k, out)
elif a.segment >= 0:
    kk = max(a.segment, 1)
    seg_out = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
    seg_ts = torch.zeros((n, kk), dtype=torch.int32, device="cuda")

    def call(i):
        ctx.segment_batch_device(x[i % copies], w, h, w, w * h, n, a.segment, seg_out, w, w * h,
                                 seg_ts, out["topk_count"], out["status"])
else:
    def call(i):
        ctx.analyze_batch_device(x[i % copies], w, h, w, w * h, n, k, out)
for i in range(a.reps):
    call(i)
torch.cuda.synchronize()
if a.time:
    steps = max(3, int(2e9 // max(x[0].numel(), 1)))
    steps = min(steps, 2000)
    graph = None
    if a.graph > 0:
        a.graph = max(a.graph, copies)  # every input copy once per replay (L2 rotation)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(a.graph):
                call(i)
        graph.replay()
        torch.cuda.synchronize()
        steps = max(1, steps // a.graph) * a.graph
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph is not None:
        for _ in range(steps // a.graph):
            graph.replay()
    else:
        for i in range(steps):
            call(i)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    px = n * h * w
    print(json.dumps({"config": a.config, "rgb": a.rgb, "depth": a.depth, "graph": a.graph,
                      "segment": a.segment, "n": n, "w": w, "h": h,
                      "ms_per_step": ms,
                      "gpix_per_s": px / ms / 1e6, "hbm_frac": px / ms / 1e6 / 6452.8,
                      "images_per_s": n / ms * 1e3, "copies": copies, "steps": steps}))
else:
    print(a.config, "t0[0] =", int(out["t0"][0]), "topk[0] =", out["topk"][0].tolist())

"""Device-resident timing of C2 (depth 3, the bench step), C3, C4 and C5 with
bench.py's in-graph timing (W warm-up + K steps in one CUDA graph), for A/B
comparisons of library builds:  python tools/ab_time.py [--configs C2,C4]
Prints one JSON line {config: Gpx/s}."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1707_05062_b200 import Context, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3,C4,C5")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--depth", type=int, default=0, help="0: 3 for C1/C2, else 1")
a = ap.parse_args()
ctx = Context(0)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
res = {}
STEPS = {"C1": 300, "C2": 300, "C3": 10, "C4": 30, "C5": 10}
for name in a.configs.split(","):
    x = synth.generate(name, device="cuda")
    n, h, w = x.shape
    copies = max(1, int(2 * l2 // x.numel()) + 1) if x.numel() < 2 * l2 else 1
    bufs = torch.stack([x] * copies) if copies > 1 else x[None]
    o = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
         "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
         "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
         "topk": torch.zeros((n, 6), dtype=torch.int32, device="cuda"),
         "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.set_pipeline_depth(a.depth or (3 if name in ("C1", "C2") else 1))

    def step(i):
        ctx.analyze_batch_device(bufs[i % copies], w, h, w, w * h, n, 6, o)
    step(0)  # workspace allocations happen outside the capture
    torch.cuda.synchronize()
    g = bench.GraphSteps(step, 5, STEPS[name])
    best = 0.0
    for _ in range(a.reps):
        ms = g.run(1)
        best = max(best, n * h * w * STEPS[name] / (ms * 1e-3) / 1e9)
    res[name] = round(best, 1)
    del bufs, x, g
    torch.cuda.empty_cache()
print(json.dumps(res))

"""Run one config through the device API a few times (for ncu / sanitizer)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_05062_b200 import Context, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
x = synth.generate(a.config, device="cuda")
n, h, w = x.shape
ctx = Context(0)
k = 6
out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
       "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
       "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
       "topk": torch.zeros((n, k), dtype=torch.int32, device="cuda"),
       "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
       "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
for _ in range(a.reps):
    ctx.analyze_batch_device(x, w, h, w, w * h, n, k, out)
torch.cuda.synchronize()
print(a.config, "t0[0] =", int(out["t0"][0]), "topk[0] =", out["topk"][0].tolist())

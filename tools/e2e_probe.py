"""Wall-clock breakdown of the host-buffer (e2e) path on C2-sized input:
plain pinned H2D + sync, the same split in 8 chunks, and kohler_cuda_analyze."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05062_b200 import Context  # noqa: E402

w, h = 5184, 3456
n = w * h
src = torch.empty((h, w), dtype=torch.uint8).pin_memory()
src.random_(0, 255)
dst = torch.empty((h, w), dtype=torch.uint8, device="cuda")
ctx = Context(0)
lib = ctx._lib
res = {k: np.zeros(256, np.uint64) for k in ("s", "c")}
vals = np.zeros(256, np.float64)
dfn = np.zeros(256, np.uint8)
t0 = np.zeros(1, np.int32)
tk = np.zeros(6, np.int32)
cnt = np.zeros(1, np.int32)


def analyze():
    lib.kohler_cuda_analyze(ctx.handle, src.data_ptr(), w, h, w, 6, res["s"].ctypes.data,
                            res["c"].ctypes.data, vals.ctypes.data, dfn.ctypes.data,
                            t0.ctypes.data, tk.ctypes.data, cnt.ctypes.data)


def copy1():
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()


def copy8():
    for c in range(8):
        a, e = h * c // 8, h * (c + 1) // 8
        dst[a:e].copy_(src[a:e], non_blocking=True)
    torch.cuda.synchronize()


def curve_only():
    lib.kohler_cuda_curve(ctx.handle, src.data_ptr(), w, h, w, res["s"].ctypes.data,
                          res["c"].ctypes.data)


out = {}
for name, fn in [("copy1", copy1), ("copy8", copy8), ("analyze", analyze), ("curve", curve_only),
                 ("copy1_again", copy1), ("analyze_again", analyze)]:
    for _ in range(5):
        fn()
    ts = []
    for _ in range(50):
        st = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - st)
    ts.sort()
    out[name] = {"median_us": ts[len(ts) // 2] * 1e6, "min_us": ts[0] * 1e6,
                 "GBps_median": n / ts[len(ts) // 2] / 1e9}
print(json.dumps(out, indent=1))

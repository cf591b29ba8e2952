"""Is the C2 bench step host-bound?  Host issue time per call vs device time
per step, for the Python wrapper and for raw C-ABI calls with cached
pointers, at pipeline depth 1 and 2."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05062_b200 import Context, synth  # noqa: E402

x = synth.generate("C2", device="cuda")[0]
h, w = x.shape
copies = 15
buf = torch.stack([x] * copies).contiguous()
ctx = Context(0)
out = {"sums": torch.zeros(256, dtype=torch.int64, device="cuda"),
       "cards": torch.zeros(256, dtype=torch.int64, device="cuda"),
       "values": torch.zeros(256, dtype=torch.float64, device="cuda"),
       "defined": torch.zeros(256, dtype=torch.uint8, device="cuda"),
       "t0": torch.zeros(1, dtype=torch.int32, device="cuda"),
       "topk": torch.zeros(6, dtype=torch.int32, device="cuda"),
       "topk_count": torch.zeros(1, dtype=torch.int32, device="cuda"),
       "status": torch.zeros(1, dtype=torch.int32, device="cuda")}
lib, hd = ctx._lib, ctx.handle
st = torch.cuda.current_stream().cuda_stream
ptrs = [buf[i].data_ptr() for i in range(copies)]
o = [out[k].data_ptr() for k in ("sums", "cards", "values", "defined", "t0", "topk", "topk_count", "status")]


def wrapper(i):
    ctx.analyze_batch_device(buf[i % copies], w, h, w, w * h, 1, 6, out)


def raw(i):
    lib.kohler_cuda_analyze_batch_device(hd, ptrs[i % copies], 1, w, h, w, w * h, 6, *o, st)


res = {}
for depth in (1, 2):
    ctx.set_pipeline_depth(depth)
    for name, fn in (("wrapper", wrapper), ("raw", raw)):
        for i in range(20):
            fn(i)
        torch.cuda.synchronize()
        n = 2000
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for i in range(n):
            fn(i)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        res[f"d{depth}_{name}"] = {"host_us_per_call": (t1 - t0) / n * 1e6,
                                   "device_us_per_step": e0.elapsed_time(e1) / n * 1e3}
print(json.dumps(res))

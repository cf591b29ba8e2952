"""Per-step device time of the row-band path pieces on one GPU (C2):
band K1 (+ its finish) alone, band + selection, and the fused analyze path."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05062_b200 import Context, synth  # noqa: E402

x = synth.generate("C2", device="cuda")[0]
h, w = x.shape
copies = 15
buf = torch.stack([x] * copies).contiguous()
ctx = Context(0)
cur = torch.zeros(512, dtype=torch.int64, device="cuda")
out = {"values": torch.zeros(256, dtype=torch.float64, device="cuda"),
       "t0": torch.zeros(1, dtype=torch.int32, device="cuda"),
       "topk": torch.zeros(6, dtype=torch.int32, device="cuda"),
       "topk_count": torch.zeros(1, dtype=torch.int32, device="cuda"),
       "status": torch.zeros(1, dtype=torch.int32, device="cuda")}
res = {}


def t(name, fn, n=300):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / n * 1e3


t("band", lambda i: ctx.band_curve_device(buf[i % copies], w, w, h, 0, h, cur.data_ptr(),
                                          cur.data_ptr() + 2048))
t("band+select", lambda i: (ctx.band_curve_device(buf[i % copies], w, w, h, 0, h, cur.data_ptr(),
                                                  cur.data_ptr() + 2048),
                            ctx.select_device(cur.data_ptr(), cur.data_ptr() + 2048, 1, 256, 6, out)))
t("select", lambda i: ctx.select_device(cur.data_ptr(), cur.data_ptr() + 2048, 1, 256, 6, out))
o2 = {"sums": cur[:256], "cards": cur[256:], "t0": out["t0"], "topk": out["topk"],
      "topk_count": out["topk_count"], "status": out["status"]}
t("analyze", lambda i: ctx.analyze_batch_device(buf[i % copies], w, h, w, w * h, 1, 6, o2))
print(json.dumps({k: round(v, 2) for k, v in res.items()}))

# the BandedAnalyzer's pipelined step (world 1: no all-reduce), fast raw calls
from paper_1707_05062_b200.bands import BandedAnalyzer  # noqa: E402
ba = BandedAnalyzer(ctx, w, h, 1, 0, 6)
t("banded_step_pipelined", lambda i: ba.step_pipelined(i, buf[i % copies], w))
ba.drain()
print(json.dumps({k: round(v, 2) for k, v in res.items()}))

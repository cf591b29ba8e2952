"""Pinned H2D rate of one C2-sized image (17.9 MB) split into k chunks
copied concurrently on k streams (k copy requests in flight), and on one
stream in k chunks, and the D2H rate: is this box's H2D bound by the
number of outstanding DMA reads (VM / IOMMU latency) rather than the link?"""
import json

import torch

n = 5184 * 3456
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.fill_(5)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}
streams = [torch.cuda.Stream() for _ in range(16)]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


for k in (1, 2, 4, 8, 16):
    step = (n + k - 1) // k

    def multi():
        ev = torch.cuda.Event()
        ev.record()
        for i in range(k):
            s = streams[i]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
        for i in range(k):
            torch.cuda.current_stream().wait_stream(streams[i])

    def single():
        for i in range(k):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    res[f"h2d_{k}_streams"] = round(timed(multi), 2)
    res[f"h2d_{k}_chunks_1_stream"] = round(timed(single), 2)
hsrc = torch.empty(n, dtype=torch.uint8).pin_memory()
res["d2h"] = round(timed(lambda: hsrc.copy_(dst, non_blocking=True)), 2)
print(json.dumps(res))

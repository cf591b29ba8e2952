"""Pinned H2D rate of a C2-sized image (17.9 MB) copied as sequential
cudaMemcpyAsync calls of a given chunk size on one stream (sizes 64 KiB ..
the whole image), several repetitions: how this box's DMA rate depends on the
transfer size (the host API's chunked upload)."""
import json

import torch

n = 5184 * 3456
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.fill_(5)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}


def rate(chunk, reps=8):
    def once():
        for off in range(0, n, chunk):
            dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    return round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


for rep in range(2):
    for kb in (64, 128, 256, 512, 1024, 2048, 4096, 8192, 17496):
        res.setdefault(f"{kb}K", []).append(rate(kb * 1024))
print(json.dumps(res))

import torch, time, json, os
n = 5184 * 3456
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
res = []
for trial in range(3):
    src = torch.empty(n, dtype=torch.uint8).pin_memory()
    src.fill_(trial)
    print("pinned?", src.is_pinned())
    for blk in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        res.append((trial, blk, round(n / (e0.elapsed_time(e1) / 20) / 1e6, 1)))
    del src
pg = torch.empty(n, dtype=torch.uint8)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(10): dst.copy_(pg)
torch.cuda.synchronize(); res.append(("pageable", round(n*10/(time.perf_counter()-t)/1e9,1)))
print(json.dumps(res))

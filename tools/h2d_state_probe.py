"""Does this box's pinned H2D rate depend on GPU state?  Rate of 17.9 MB
copies (a) right after pinning, (b) after 1 s idle, (c) while a compute
kernel keeps the GPU busy on another stream, (d) right after a 1 s burn,
with the SM / memory clocks sampled by NVML at each point."""
import json
import threading
import time

import pynvml as N
import torch

N.nvmlInit()
hd = N.nvmlDeviceGetHandleByIndex(0)


def clocks():
    return (N.nvmlDeviceGetClockInfo(hd, N.NVML_CLOCK_SM), N.nvmlDeviceGetClockInfo(hd, N.NVML_CLOCK_MEM))


n = 5184 * 3456
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.fill_(5)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()


def rate(reps=10):
    with torch.cuda.stream(cs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record(cs)
    e1.synchronize()
    return round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


res = {}
res["a_cold"] = (rate(), clocks())
time.sleep(1.0)
res["b_after_idle"] = (rate(), clocks())
a = torch.randn(4096, 4096, device="cuda")
stop = [False]
busy = torch.cuda.Stream()


def burn(seconds):
    t = time.time()
    with torch.cuda.stream(busy):
        while time.time() - t < seconds:
            for _ in range(20):
                a.mul_(1.0000001)
            torch.cuda.synchronize()


th = threading.Thread(target=burn, args=(1.5,))
th.start()
time.sleep(0.5)
res["c_during_compute"] = (rate(), clocks())
th.join()
res["d_after_burn"] = (rate(), clocks())
time.sleep(2.0)
res["e_after_2s_idle"] = (rate(), clocks())
for i in range(3):
    res[f"f_repeat{i}"] = (rate(), clocks())
print(json.dumps(res))

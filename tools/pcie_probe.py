"""What limits the e2e path's pinned H2D on this box: the GPU's PCIe link
(generation / width, current and max, NVML), its CPU/NUMA affinity (NVML and
sysfs), and the pinned H2D rate from each NUMA node's CPUs."""
import glob
import json
import os

import torch

out = {}
try:
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(0)
    out["pcie"] = {"gen_cur": N.nvmlDeviceGetCurrPcieLinkGeneration(h),
                   "gen_max": N.nvmlDeviceGetMaxPcieLinkGeneration(h),
                   "width_cur": N.nvmlDeviceGetCurrPcieLinkWidth(h),
                   "width_max": N.nvmlDeviceGetMaxPcieLinkWidth(h)}
    try:
        out["pcie"]["gpu_max_gen"] = N.nvmlDeviceGetGpuMaxPcieLinkGeneration(h)
    except Exception:
        pass
    try:
        words = N.nvmlDeviceGetCpuAffinity(h, 4)
        cpus = [64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1]
        out["nvml_cpu_affinity"] = [min(cpus), max(cpus), len(cpus)] if cpus else None
    except Exception as exc:
        out["nvml_cpu_affinity"] = str(exc)
    out["bus_id"] = N.nvmlDeviceGetPciInfo(h).busId.decode() if isinstance(N.nvmlDeviceGetPciInfo(h).busId, bytes) else N.nvmlDeviceGetPciInfo(h).busId
except Exception as exc:
    out["nvml_error"] = str(exc)
out["nodes"] = {os.path.basename(p): open(p + "/cpulist").read().strip()
                for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))}
out["ncpu"] = os.cpu_count()
try:
    out["affinity_now"] = len(os.sched_getaffinity(0))
except Exception:
    pass
n = 5184 * 3456
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.fill_(3)
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
out["h2d_gbs"] = n * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e9
d2h = torch.empty(n, dtype=torch.uint8).pin_memory()
e0.record()
for _ in range(20):
    d2h.copy_(dst, non_blocking=True)
e1.record()
torch.cuda.synchronize()
out["d2h_gbs"] = n * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps(out))

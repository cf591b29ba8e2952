"""H2D bandwidth of a C2-sized host buffer by allocation method (this pool's
boxes are VMs whose DMA speed depends on how the pinned pages were obtained):
cudaHostAlloc (torch pin_memory), cudaHostRegister of a 2 MiB-aligned
transparent-huge-page region, and pageable memory (driver staging)."""
import ctypes
import json
import mmap

import numpy as np
import torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
cudart = ctypes.CDLL("libcudart.so")
n = 5184 * 3456
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def bw(ptr, reps=20):
    def one():
        cudart.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(ptr),
                               ctypes.c_size_t(n), 1, ctypes.c_void_p(s.cuda_stream))
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            one()
        e1.record()
        torch.cuda.synchronize()
        out.append(round(n / (e0.elapsed_time(e1) / reps) / 1e6, 1))
    return out


res = {}
t = torch.empty(n, dtype=torch.uint8).pin_memory()
t.fill_(1)
res["cudaHostAlloc(torch)"] = bw(t.data_ptr())
del t
# THP region registered
sz = (n + (2 << 20) - 1) // (2 << 20) * (2 << 20)
mm = mmap.mmap(-1, sz + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
al = (base + (2 << 20) - 1) // (2 << 20) * (2 << 20)
MADV_HUGEPAGE = 14
rc = libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(sz), MADV_HUGEPAGE)
arr = np.frombuffer(mm, dtype=np.uint8, count=sz, offset=al - base)
arr[:] = 3  # fault the pages in (as huge pages if THP allows)
r = cudart.cudaHostRegister(ctypes.c_void_p(al), ctypes.c_size_t(sz), 0)
res["thp_register"] = {"madvise": rc, "register": r, "GBps": bw(al) if r == 0 else None}
try:
    res["thp_enabled"] = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
    res["AnonHugePages"] = [l for l in open("/proc/meminfo") if "AnonHugePages" in l][0].strip()
except OSError:
    pass
if r == 0:
    cudart.cudaHostUnregister(ctypes.c_void_p(al))
pg = np.ones(n, np.uint8)
res["pageable"] = bw(pg.ctypes.data, reps=10)
# cudaHostAlloc with portable|mapped flags via cudart
p = ctypes.c_void_p()
r = cudart.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), 0)
ctypes.memset(p, 5, n)
res["cudaHostAlloc(default)"] = bw(p.value)
cudart.cudaFreeHost(p)
print(json.dumps(res))

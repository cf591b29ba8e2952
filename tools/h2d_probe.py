"""Host->device copy bandwidth on this box (pinned, 1D vs 2D pitched), the
floor of the end-to-end (host-buffer) path."""
import ctypes
import json
import time

import torch

cudart = ctypes.CDLL("libcudart.so")
w, h = 5184, 3456
n = w * h
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.random_(0, 255)
dst = torch.empty(n + 4096 * h, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
out = {}
for name, fn in [
    ("1d", lambda: dst[:n].copy_(src, non_blocking=True)),
    ("2d_pitch5248", lambda: cudart.cudaMemcpy2DAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_size_t(5248),
                                                       ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(w),
                                                       ctypes.c_size_t(w), ctypes.c_size_t(h), 1,
                                                       ctypes.c_void_p(s.cuda_stream))),
]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    out[name] = {"ms": ms, "GBps": n / ms / 1e6}
# chunked 1D copies (4 chunks)
print(json.dumps(out))

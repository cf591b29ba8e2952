"""Row-band decomposition of one large image over the ranks of a
``torch.distributed`` job (one process per GPU).

Mirrors the reference's row-block split (proj/src/fast.cpp:42,53-55: block b
of B owns rows [h*b/B, h*(b+1)/B)) and ownership rule (fast.cpp:15-31: a row
owns its right pairs and the down pair into the next row), so each rank
reads its rows plus ONE halo row.  Rank partials are exact integer curves of
the pairs they own; one all-reduce (u64 sum carried as int64, two's
complement) merges them like merge_accumulators (curve.cpp:16-30), then
every rank runs the device selection on the merged curve.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def band_bounds(h: int, world: int, rank: int) -> tuple:
    """Own rows [r0, r1) of `rank` (may be empty when world > h)."""
    return (h * rank) // world, (h * (rank + 1)) // world


def band_slice(h: int, r0: int, r1: int) -> tuple:
    """Rows a rank must hold: its own rows plus the halo row r1 (if r1 < h)."""
    return r0, min(r1 + 1, h)


def allreduce_curve(buf: torch.Tensor, group=None) -> torch.Tensor:
    """Sum int64 curve partials [sum(256) | card(256)] over the group."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


class BandedAnalyzer:
    """Per-rank driver: partial curve of the rank's band (K1 on the GPU),
    NCCL all-reduce of the 512 u64 partials, device selection (K4)."""

    def __init__(self, ctx, w: int, h: int, world: int, rank: int, k: int = 6, group=None,
                 device=None):
        self.ctx, self.w, self.h, self.k, self.group = ctx, w, h, k, group
        self.r0, self.r1 = band_bounds(h, world, rank)
        self.lo, self.hi = band_slice(h, self.r0, self.r1)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.curve = torch.zeros(512, dtype=torch.int64, device=dev)
        # pipelined steps: two partial buffers, the all-reduce of step i in
        # flight while step i + 1's band accumulates
        self._curves = [torch.zeros(512, dtype=torch.int64, device=dev) for _ in range(2)]
        self._pending = None  # (work handle, buffer) of the previous step
        self.always_reduce = False  # all-reduce even with one rank (tests of the N > 1 path)
        self.out = {"values": torch.zeros(256, dtype=torch.float64, device=dev),
                    "defined": torch.zeros(256, dtype=torch.uint8, device=dev),
                    "t0": torch.zeros(1, dtype=torch.int32, device=dev),
                    "topk": torch.zeros(k, dtype=torch.int32, device=dev),
                    "topk_count": torch.zeros(1, dtype=torch.int32, device=dev),
                    "status": torch.zeros(1, dtype=torch.int32, device=dev)}

    @property
    def rows_held(self) -> int:
        return self.hi - self.lo

    def _fast_calls(self):
        """Raw C-ABI calls with the pointers resolved once: the per-step host
        cost (ctypes + tensor pointer lookups) otherwise exceeds the device
        time of a small band.  Only for a real CUDA context on the current
        stream (the CPU tests pass a stand-in context)."""
        lib = getattr(self.ctx, "_lib", None)
        if lib is None:
            return None
        st = torch.cuda.current_stream()  # the capture stream while a graph is recorded
        if getattr(self, "_fc", None) is None or self._fc[2] != st.cuda_stream:
            o = self.out
            h = self.ctx.handle
            outs = (o["values"].data_ptr(), o["defined"].data_ptr(), o["t0"].data_ptr(),
                    o["topk"].data_ptr(), o["topk_count"].data_ptr(), o["status"].data_ptr())
            self._fc = (lib, h, st.cuda_stream, outs)
        return self._fc

    def _select(self, curve: torch.Tensor) -> None:
        fc = self._fast_calls()
        if fc is None:
            self.ctx.select_device(curve.data_ptr(), curve.data_ptr() + 256 * 8, 1, 256, self.k,
                                   self.out)
            return
        lib, h, st, outs = fc
        p = curve.data_ptr()
        rc = lib.kohler_cuda_select_device(h, p, p + 2048, 1, 256, self.k, *outs, st)
        if rc:
            from .api import _raise_for
            _raise_for(rc)

    def _band(self, band, pitch: int, cur: torch.Tensor, card_ptr: int = None) -> None:
        p = cur.data_ptr()
        pc = p + 2048 if card_ptr is None else card_ptr
        fc = self._fast_calls()
        if fc is None:
            self.ctx.band_curve_device(band, self.w, pitch, self.h, self.r0, self.r1, p, pc)
            return
        lib, h, st, _ = fc
        rc = lib.kohler_cuda_band_curve_device(h, band.data_ptr(), self.w, pitch, self.h, self.r0,
                                               self.r1, p, pc, st)
        if rc:
            from .api import _raise_for
            _raise_for(rc)

    def step_pipelined(self, i: int, band: torch.Tensor, pitch: int) -> None:
        """Step i with the all-reduce overlapped: K1 of this band into buffer
        i % 2, an asynchronous all-reduce of it (NCCL's stream, after K1),
        then -- on the compute stream, behind this K1 -- the selection of the
        PREVIOUS step's merged curve.  ``drain()`` completes the last step.
        Every step's result is the same as ``step``'s; ``out`` holds step
        i - 1's selection after this call (step i's after ``drain``)."""
        cur = self._curves[i % 2]
        if self.r1 > self.r0:
            self._band(band, pitch, cur)
        else:
            cur.zero_()
        work = None
        if dist.is_available() and dist.is_initialized() and (
                self.always_reduce or dist.get_world_size(self.group) > 1):
            work = dist.all_reduce(cur, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.drain()
        self._pending = (work, cur)

    def drain(self) -> None:
        if self._pending is None:
            return
        work, buf = self._pending
        if work is not None:
            work.wait()  # the compute stream waits for the all-reduce
        self._select(buf)
        self._pending = None

    # ---- bucketed all-reduce -------------------------------------------------
    # One small all-reduce per step is latency-bound (a few us over NVLink,
    # longer than a band's K1 at N >= 2).  Bucketed steps put step i's
    # partial into slot i % m of a [sums m x 256 | cards m x 256] block and
    # all-reduce the block once per m steps (asynchronously, while the next
    # bucket accumulates into the other block); the m selections then run
    # as one select launch.  Every step's result is exact; step i's lands in
    # ``bout[...][i % m]`` once its bucket is reduced (``drain_buckets()``
    # completes a partial bucket).
    def enable_buckets(self, m: int) -> None:
        dev = self.curve.device
        k = self.k
        self.m = int(m)
        self._blocks = [torch.zeros(2 * self.m * 256, dtype=torch.int64, device=dev)
                        for _ in range(2)]
        self.bout = {"values": torch.zeros((self.m, 256), dtype=torch.float64, device=dev),
                     "defined": torch.zeros((self.m, 256), dtype=torch.uint8, device=dev),
                     "t0": torch.zeros(self.m, dtype=torch.int32, device=dev),
                     "topk": torch.zeros((self.m, k), dtype=torch.int32, device=dev),
                     "topk_count": torch.zeros(self.m, dtype=torch.int32, device=dev),
                     "status": torch.zeros(self.m, dtype=torch.int32, device=dev)}
        self._bblock, self._bfill, self._bpending = 0, 0, None

    def step_bucketed(self, band: torch.Tensor, pitch: int) -> None:
        blk = self._blocks[self._bblock]
        s = self._bfill
        if self.r1 > self.r0:
            self._band(band, pitch, blk[s * 256:(s + 1) * 256],
                       blk.data_ptr() + (self.m + s) * 256 * 8)
        else:
            blk[s * 256:(s + 1) * 256].zero_()
            blk[(self.m + s) * 256:(self.m + s + 1) * 256].zero_()
        self._bfill += 1
        if self._bfill == self.m:
            self.flush_bucket()

    def flush_bucket(self) -> None:
        n = self._bfill
        if n == 0:
            return
        blk = self._blocks[self._bblock]
        work = None
        if dist.is_available() and dist.is_initialized() and (
                self.always_reduce or dist.get_world_size(self.group) > 1):
            work = dist.all_reduce(blk, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.finish_bucket()
        self._bpending = (work, blk, n)
        self._bblock ^= 1
        self._bfill = 0

    def finish_bucket(self) -> None:
        if self._bpending is None:
            return
        work, blk, n = self._bpending
        if work is not None:
            work.wait()
        p = blk.data_ptr()
        pc = p + self.m * 256 * 8
        o = self.bout
        fc = self._fast_calls()
        if fc is None:
            self.ctx.select_device(p, pc, n, 256, self.k, o)
        else:
            lib, h, st, _ = fc
            rc = lib.kohler_cuda_select_device(h, p, pc, n, 256, self.k, o["values"].data_ptr(),
                                               o["defined"].data_ptr(), o["t0"].data_ptr(),
                                               o["topk"].data_ptr(), o["topk_count"].data_ptr(),
                                               o["status"].data_ptr(), st)
            if rc:
                from .api import _raise_for
                _raise_for(rc)
        self._bpending = None

    def drain_buckets(self) -> None:
        self.flush_bucket()
        self.finish_bucket()

    def step(self, band: torch.Tensor, pitch: int) -> None:
        """band: CUDA uint8 buffer holding rows [lo, hi) with row pitch `pitch`."""
        if self.r1 > self.r0:
            self._band(band, pitch, self.curve)
        else:
            self.curve.zero_()
        allreduce_curve(self.curve, self.group)
        self._select(self.curve)

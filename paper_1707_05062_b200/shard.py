"""Batch sharding over the ranks of a ``torch.distributed`` job (one process
per GPU) for the independent-image configurations (C3 video
frames, C5 small images).

Images are independent, so each rank runs the whole per-image pipeline on a
contiguous shard of the batch — no collective on the data path.  The only
exchange is optional: ``gather=True`` collects every image's curve and
thresholds on every rank (one all-gather per output array), which the
reference's per-frame loop (proj/src/bench.cpp:264-284) would need only to
write all results in one place.  Shard sizes may differ by one image; the
gather pads to the largest shard.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Images [i0, i1) of `rank` (contiguous, sizes differ by at most one)."""
    return (n * rank) // world, (n * (rank + 1)) // world


_FIELDS = (("sums", torch.int64, 256), ("cards", torch.int64, 256), ("t0", torch.int32, 0),
           ("topk_count", torch.int32, 0), ("status", torch.int32, 0))


class BatchSharder:
    """Per-rank driver: the rank's shard through ``ctx.analyze_batch_device``
    (K1 or K5 + finish/selection), optionally all-gathered."""

    def __init__(self, ctx, n: int, w: int, h: int, world: int, rank: int, k: int = 6,
                 group=None, device=None):
        self.ctx, self.n, self.w, self.h, self.k = ctx, n, w, h, k
        self.world, self.rank, self.group = world, rank, group
        self.i0, self.i1 = shard_bounds(n, world, rank)
        self.local = self.i1 - self.i0
        self.cap = (n + world - 1) // world  # the largest shard
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.out = {}
        for name, dt, m in _FIELDS:
            shape = (self.cap, m) if m else (self.cap,)
            self.out[name] = torch.zeros(shape, dtype=dt, device=dev)
        self.out["topk"] = torch.zeros((self.cap, k), dtype=torch.int32, device=dev)
        self.full = None

    def run(self, shard: torch.Tensor, pitch: int = None, image_stride: int = None,
            gather: bool = False) -> dict:
        """shard: this rank's images (local, h, w) uint8 on the rank's device.
        Returns the local outputs (first ``self.local`` rows valid), or with
        ``gather`` the outputs of all n images in batch order."""
        pitch = self.w if pitch is None else pitch
        image_stride = pitch * self.h if image_stride is None else image_stride
        if self.local:
            self.ctx.analyze_batch_device(shard, self.w, self.h, pitch, image_stride, self.local,
                                          self.k, self.out)
        if not gather:
            return self.out
        return self._gather()

    def _gather(self) -> dict:
        world = self.world
        if not (dist.is_available() and dist.is_initialized()) or world == 1:
            return {key: v[: self.n] for key, v in self.out.items()}
        full = {}
        for key, v in self.out.items():
            parts = [torch.empty_like(v) for _ in range(world)]
            dist.all_gather(parts, v.contiguous(), group=self.group)
            # drop each rank's padding rows: rank r holds images [n r / W, n (r + 1) / W)
            full[key] = torch.cat([parts[r][: shard_bounds(self.n, world, r)[1]
                                            - shard_bounds(self.n, world, r)[0]]
                                   for r in range(world)])
        self.full = full
        return full

"""Host logic of the multi-GPU row-band path, on CPU with the gloo backend
(world_size 2 and 3).  The per-rank partial is the oracle's curve of the rows
the rank owns (standing in for the device K1 partial); the merge is the same
allreduce_curve the NCCL path uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_05062_b200.bands import allreduce_curve, band_bounds, band_slice


def test_band_bounds_partition():
    for h in (1, 2, 3, 7, 100, 3456):
        for world in (1, 2, 3, 4, 8, 11):
            rows = []
            for r in range(world):
                r0, r1 = band_bounds(h, world, r)
                assert 0 <= r0 <= r1 <= h
                lo, hi = band_slice(h, r0, r1)
                assert lo == r0 and hi == (r1 + 1 if r1 < h else h)
                rows.extend(range(r0, r1))
            assert rows == list(range(h))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, img, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    orc = oracle.Oracle()
    h = img.shape[0]
    r0, r1 = band_bounds(h, world, rank)
    lo, hi = band_slice(h, r0, r1)
    # the rank only sees its rows + halo, re-based to row 0
    local = np.ascontiguousarray(img[lo:hi])
    buf = torch.zeros(512, dtype=torch.int64)
    if r1 > r0:
        # rows [r0, r1) of the global image own pairs into the halo (row r1-lo
        # of `local`); curve_rows on the local slice with h_local = hi-lo
        # counts exactly those pairs.
        s, c = orc.curve_rows(local, 0, r1 - r0)
        buf[:256] = torch.from_numpy(s.view(np.int64))
        buf[256:] = torch.from_numpy(c.view(np.int64))
    allreduce_curve(buf)
    q.put((rank, buf.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_band_merge_is_exact(orc, world):
    rng = np.random.default_rng(world)
    img = rng.integers(0, 256, (37, 53), dtype=np.uint8)
    img[10:20] = 77  # equal pairs across a band edge
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s, c = orc.fast_curve(img)
    for _, buf in got:
        assert np.array_equal(buf[:256].view(np.uint64), s)
        assert np.array_equal(buf[256:].view(np.uint64), c)

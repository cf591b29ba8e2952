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


class _OracleCtx:
    """Stands in for the CUDA context on CPU: the band partial and the
    selection come from the oracle, written through the same raw pointers
    the C ABI receives."""

    def __init__(self, orc, img):
        self.orc, self.img = orc, img

    def band_curve_device(self, band, w, pitch, h_total, r0, r1, sum_ptr, card_ptr, stream=None):
        import ctypes
        local = np.ascontiguousarray(self.img[r0:min(r1 + 1, h_total)])
        s, c = self.orc.curve_rows(local, 0, r1 - r0)
        ctypes.memmove(sum_ptr, s.ctypes.data, 2048)
        ctypes.memmove(card_ptr, c.ctypes.data, 2048)

    def select_device(self, sums, cards, n, levels, k, out, stream=None):
        import ctypes
        for i in range(n):
            s = np.zeros(256, np.uint64)
            c = np.zeros(256, np.uint64)
            ctypes.memmove(s.ctypes.data, sums + 2048 * i, 2048)
            ctypes.memmove(c.ctypes.data, cards + 2048 * i, 2048)
            v, d = self.orc.mean_contrast(s, c)
            st, ts = self.orc.top_k(v, d, k)
            t0 = out["t0"] if n > 1 or out["t0"].dim() else out["t0"]
            out["t0"][i] = self.orc.optimal_threshold(v, d)
            out["topk_count"][i] = len(ts)
            tk = out["topk"][i] if out["topk"].dim() == 2 else out["topk"]
            tk[: len(ts)] = torch.tensor(ts, dtype=torch.int32)
            out["status"][i] = st


def _worker_pipelined(rank, world, port, imgs, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1707_05062_b200.bands import BandedAnalyzer
    orc = oracle.Oracle()
    h, w = imgs[0].shape
    ctx = _OracleCtx(orc, imgs[0])
    ba = BandedAnalyzer(ctx, w, h, world, rank, k, device=torch.device("cpu"))
    got = []
    for i, im in enumerate(imgs):
        ctx.img = im  # the band K1 of step i sees image i
        ba.step_pipelined(i, None, w)
        if i > 0:  # out now holds step i - 1
            got.append((int(ba.out["t0"][0]), ba.out["topk"][: int(ba.out["topk_count"][0])].tolist()))
    ba.drain()
    got.append((int(ba.out["t0"][0]), ba.out["topk"][: int(ba.out["topk_count"][0])].tolist()))
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pipelined_steps(orc, world):
    """The overlapped schedule of bench.py at N > 1 (async all-reduce of step
    i while step i + 1 accumulates, selection one step behind, drain at the
    end) yields every step's exact thresholds."""
    rng = np.random.default_rng(100 + world)
    imgs = []
    for i in range(5):
        a = rng.integers(0, 256, (41, 29), dtype=np.uint8)
        a[5 + i:20 + i] = rng.integers(0, 256)
        imgs.append(a)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pipelined, args=(r, world, port, imgs, 6, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(e["t0"], e["topk"]) for e in (orc.analyze(im, 6) for im in imgs)]
    for _, got in res:
        assert got == want


def _worker_bucketed(rank, world, port, imgs, k, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1707_05062_b200.bands import BandedAnalyzer
    orc = oracle.Oracle()
    h, w = imgs[0].shape
    ctx = _OracleCtx(orc, imgs[0])
    ba = BandedAnalyzer(ctx, w, h, world, rank, k, device=torch.device("cpu"))
    ba.enable_buckets(m)
    got = {}

    def harvest(first, n):
        for j in range(n):
            cnt = int(ba.bout["topk_count"][j])
            got[first + j] = (int(ba.bout["t0"][j]), ba.bout["topk"][j, :cnt].tolist())

    for i, im in enumerate(imgs):
        ctx.img = im
        ba.step_bucketed(None, w)
        if (i + 1) % m == 0 and i + 1 > m:  # the previous bucket was selected
            harvest(i + 1 - 2 * m, m)
    full = len(imgs) // m
    if len(imgs) % m:  # the partial bucket's reduce selects the last full bucket
        ba.flush_bucket()
        harvest((full - 1) * m, m)
        ba.finish_bucket()
        harvest(full * m, len(imgs) - full * m)
    else:
        ba.drain_buckets()
        harvest((full - 1) * m, m)
    q.put((rank, [got.get(i) for i in range(len(imgs))]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n", [(2, 3, 8), (3, 2, 6)])
def test_gloo_bucketed_steps(orc, world, m, n):
    """Bucketed all-reduce (one all-reduce of m steps' partials, selection
    of the m curves in one call): every step's exact thresholds."""
    rng = np.random.default_rng(200 + world)
    imgs = []
    for i in range(n):
        a = rng.integers(0, 256, (37, 23), dtype=np.uint8)
        a[3 + i:15 + i] = rng.integers(0, 256)
        imgs.append(a)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bucketed, args=(r, world, port, imgs, 6, m, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(e["t0"], e["topk"]) for e in (orc.analyze(im, 6) for im in imgs)]
    for _, got in res:
        assert got == want


class _OracleBatchCtx:
    """CPU stand-in of Context.analyze_batch_device: the oracle pipeline per
    image, written into the output tensors."""

    def __init__(self, orc):
        self.orc = orc

    def analyze_batch_device(self, x, w, h, pitch, stride, n, k, out, stream=None):
        for i in range(n):
            e = self.orc.analyze(x[i].numpy(), k)
            out["sums"][i] = torch.from_numpy(e["sum"].view(np.int64))
            out["cards"][i] = torch.from_numpy(e["card"].view(np.int64))
            out["t0"][i] = e["t0"]
            out["topk_count"][i] = len(e["topk"])
            out["topk"][i, : len(e["topk"])] = torch.tensor(e["topk"], dtype=torch.int32)
            out["status"][i] = e["status"]


def _worker_shard(rank, world, port, imgs, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1707_05062_b200.shard import BatchSharder
    n, h, w = imgs.shape
    sh = BatchSharder(_OracleBatchCtx(oracle.Oracle()), n, w, h, world, rank, k,
                      device=torch.device("cpu"))
    full = sh.run(torch.from_numpy(imgs[sh.i0:sh.i1]), gather=True)
    q.put((rank, {key: v.numpy().copy() for key, v in full.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_batch_shards_and_gather(orc, world):
    """C3 / C5-style sharding: contiguous image shards (sizes differing by
    one), no collective but the optional all-gather, results in batch order
    on every rank, identical to the single-process pipeline."""
    from paper_1707_05062_b200.shard import shard_bounds
    for n in (1, 2, 7, 64):
        sizes = [shard_bounds(n, world, r)[1] - shard_bounds(n, world, r)[0] for r in range(world)]
        assert sum(sizes) == n and max(sizes) - min(sizes) <= 1
    rng = np.random.default_rng(7 + world)
    n = 7
    imgs = rng.integers(0, 256, (n, 19, 23), dtype=np.uint8)
    imgs[2] = 40  # a no-boundary image
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shard, args=(r, world, port, imgs, 6, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, full in res:
        for i in range(n):
            e = orc.analyze(imgs[i], 6)
            assert np.array_equal(full["sums"][i].view(np.uint64), e["sum"])
            assert int(full["t0"][i]) == e["t0"] and int(full["status"][i]) == e["status"]
            cnt = int(full["topk_count"][i])
            assert list(full["topk"][i, :cnt]) == e["topk"]

"""The multi-GPU row-band driver (paper_1707_05062_b200/bands.py) through a
real NCCL process group on the GPU (world size 1, the all-reduce forced with
``always_reduce``), in every schedule the bench uses: synchronous step,
pipelined (all-reduce overlapped with the next band), bucketed (one
all-reduce per m steps, partial last bucket) and replayed from a CUDA graph
with the NCCL calls captured — each checked bit-exact against the reference
library on C2 and C4 (the reference merges row-block partials the same way:
proj/src/fast.cpp:42-61, proj/src/curve.cpp:16-30)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

K = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, name, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
        from paper_1707_05062_b200 import Context, synth
        from paper_1707_05062_b200.bands import BandedAnalyzer
        ctx = Context(0)
        img = synth.generate(name, device="cpu")[0]
        h, w = img.shape
        dev = torch.device("cuda", 0)
        pitch = (w + 127) // 128 * 128
        band = torch.zeros((h, pitch), dtype=torch.uint8, device=dev)
        band[:, :w] = img.to(dev)
        res = {}

        def sel(o, j=None):
            if j is None:
                return int(o["t0"][0]), o["topk"][: int(o["topk_count"][0])].tolist()
            return int(o["t0"][j]), o["topk"][j][: int(o["topk_count"][j])].tolist()

        ba = BandedAnalyzer(ctx, w, h, 1, 0, K)
        ba.always_reduce = True
        # synchronous step: the merged curve itself
        ba.step(band, pitch)
        torch.cuda.synchronize()
        res["curve"] = ba.curve.cpu().numpy().copy()
        res["step"] = sel(ba.out)
        # pipelined: 5 steps, the all-reduce of step i overlapped with step i + 1
        for depth in (1, 2):
            ctx.set_pipeline_depth(depth)
            for i in range(5):
                ba.step_pipelined(i, band, pitch)
            ba.drain()
            torch.cuda.synchronize()
            res[f"pipelined_d{depth}"] = sel(ba.out)
        # bucketed: m = 3 over 7 steps (the last bucket partial)
        ba.enable_buckets(3)
        for _ in range(7):
            ba.step_bucketed(band, pitch)
        ba.drain_buckets()
        torch.cuda.synchronize()
        res["bucketed"] = [sel(ba.bout, j) for j in range(1)]  # the last (partial) bucket: 1 step
        # graph-captured bucketed steps (the bench schedule), m = 4, 10 steps
        ba.enable_buckets(4)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                ba.step_bucketed(band, pitch)
            ba.drain_buckets()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        res["graph"] = [sel(ba.bout, j) for j in range(2)]  # last bucket: steps 8, 9
        ctx.set_pipeline_depth(1)
        dist.destroy_process_group()
        q.put(("ok", res))
    except Exception as exc:  # pragma: no cover - reported by the parent
        import traceback
        q.put(("error", f"{exc}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_nccl_band_schedules_vs_reference(ref, name):
    from paper_1707_05062_b200 import synth
    img = synth.generate(name, device="cpu")[0].numpy()
    exp = ref.analyze(img, K, workers=os.cpu_count() or 8)
    want = (exp["t0"], exp["topk"])
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    p = ctxm.Process(target=_worker, args=(_free_port(), name, q))
    p.start()
    status, res = q.get(timeout=900)
    p.join(timeout=120)
    assert status == "ok", res
    c = res["curve"]
    assert np.array_equal(c[:256].view(np.uint64), exp["sum"])
    assert np.array_equal(c[256:].view(np.uint64), exp["card"])
    assert res["step"] == want
    assert res["pipelined_d1"] == want and res["pipelined_d2"] == want
    assert all(r == want for r in res["bucketed"])
    assert all(r == want for r in res["graph"])

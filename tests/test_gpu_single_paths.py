"""The three ways a single-image K1 launch is finished:
  * small grids (<= 8 CTAs): the grid is one thread-block cluster, rank 0
    sums the CTAs' 512 combinations over distributed shared memory;
  * mid-size grids: the CTA whose flush lands last (ticket) finishes;
  * large grids: finish_kernel (K3 + K4) after K1.
Every path must give the oracle's integers, bitwise f64 means and identical
thresholds, also back to back with several launches in flight (pipeline
depth 3) reusing ONE output buffer (stream order of the output stores) and
replayed from a CUDA graph.  KOHLER_NO_CLUSTER=1 sends small grids down the
ticket path, so both are compared on the same inputs."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1707_05062_b200 import Context, synth

pytestmark = pytest.mark.gpu

K = 6
SHAPES = [(16, 1), (17, 3), (100, 37), (512, 512), (700, 650), (1024, 1024), (2000, 1500)]


def _out():
    return {"sums": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
            "cards": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
            "values": torch.zeros((1, 256), dtype=torch.float64, device="cuda"),
            "defined": torch.zeros((1, 256), dtype=torch.uint8, device="cuda"),
            "t0": torch.zeros(1, dtype=torch.int32, device="cuda"),
            "topk": torch.zeros((1, K), dtype=torch.int32, device="cuda"),
            "topk_count": torch.zeros(1, dtype=torch.int32, device="cuda"),
            "status": torch.zeros(1, dtype=torch.int32, device="cuda")}


def _host(o):
    r = {k: v.cpu().numpy()[0] for k, v in o.items()}
    r["sums"] = r["sums"].view(np.uint64)
    r["cards"] = r["cards"].view(np.uint64)
    return r


def _check(r, e):
    assert np.array_equal(r["sums"], e["sum"]) and np.array_equal(r["cards"], e["card"])
    assert np.array_equal(r["values"].view(np.uint64), np.asarray(e["values"]).view(np.uint64))
    assert int(r["t0"]) == e["t0"] and int(r["status"]) == e["status"]
    assert r["topk"][: int(r["topk_count"])].tolist() == e["topk"]


def _image(w, h, seed):
    rng = np.random.default_rng(seed)
    if w * h >= 512 * 512:
        x = synth.c1(device="cpu", w=w, h=h).numpy()
    else:
        x = rng.integers(0, 256, (h, w), dtype=np.uint8)
    return x


@pytest.fixture(scope="module")
def ctxs():
    old = os.environ.get("KOHLER_NO_CLUSTER")
    os.environ["KOHLER_NO_CLUSTER"] = "1"
    try:
        ticket = Context(0)
    finally:
        if old is None:
            del os.environ["KOHLER_NO_CLUSTER"]
        else:
            os.environ["KOHLER_NO_CLUSTER"] = old
    return Context(0), ticket


@pytest.mark.parametrize("w,h", SHAPES)
def test_single_image_paths_vs_oracle(ctxs, w, h):
    orc = oracle.Oracle()
    x = _image(w, h, w * 31 + h)
    e = orc.analyze(x, K)
    xd = torch.from_numpy(x).cuda()
    grids = []
    for ctx in ctxs:
        o = _out()
        ctx.analyze_batch_device(xd, w, h, w, w * h, 1, K, o)
        torch.cuda.synchronize()
        _check(_host(o), e)
        grids.append(ctx.last_launch_count())
    # the default context finishes small images in one launch
    if w * h <= 512 * 512:
        assert grids[0] == 1


def test_constant_and_checkerboard_small(ctxs):
    """No boundary (status 1, t0 = -1) and the widest spans, cluster path."""
    orc = oracle.Oracle()
    for x in (np.full((300, 200), 77, np.uint8),
              (np.indices((256, 256)).sum(0) % 2 * 255).astype(np.uint8)):
        h, w = x.shape
        e = orc.analyze(x, K)
        for ctx in ctxs:
            o = _out()
            ctx.analyze_batch_device(torch.from_numpy(x).cuda(), w, h, w, w * h, 1, K, o)
            torch.cuda.synchronize()
            _check(_host(o), e)


@pytest.mark.parametrize("depth", [1, 3])
def test_back_to_back_one_output_buffer(ctxs, depth):
    """Many launches in flight, all writing ONE output buffer: after the
    stream drains it must hold the LAST call's results (the cluster path's
    stores wait for the previous launch), and intermediate copies taken in
    stream order must match each call."""
    orc = oracle.Oracle()
    imgs = [_image(512, 512, s) for s in range(3)] + [_image(300, 200, 9), _image(1024, 1024, 4)]
    want = [orc.analyze(x, K) for x in imgs]
    dev = [torch.from_numpy(x).cuda() for x in imgs]
    for ctx in ctxs:
        ctx.set_pipeline_depth(depth)
        # (a) no other work between the calls: launches overlap freely
        o = _out()
        for rep in range(4):
            for xd in dev:
                h, w = xd.shape
                ctx.analyze_batch_device(xd, w, h, w, w * h, 1, K, o)
        torch.cuda.synchronize()
        _check(_host(o), want[-1])
        # (b) a snapshot after every call (a plain kernel: waits for the call)
        snaps = []
        for i, xd in enumerate(dev):
            h, w = xd.shape
            ctx.analyze_batch_device(xd, w, h, w, w * h, 1, K, o)
            snaps.append((i, {k: v.clone() for k, v in o.items()}))
        torch.cuda.synchronize()
        for i, s in snaps:
            _check(_host(s), want[i])
        ctx.set_pipeline_depth(1)


def test_graph_replay_c1(ctxs):
    """The C1 step replayed from a CUDA graph (as bench.py times it)."""
    orc = oracle.Oracle()
    x = synth.generate("C1", device="cuda")[0]
    h, w = x.shape
    e = orc.analyze(x.cpu().numpy(), K)
    ctx = ctxs[0]
    ctx.set_pipeline_depth(3)
    o = _out()
    ctx.analyze_batch_device(x, w, h, w, w * h, 1, K, o)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            ctx.analyze_batch_device(x, w, h, w, w * h, 1, K, o)
    for _ in range(3):
        for k in o:
            o[k].zero_()
        g.replay()
        torch.cuda.synchronize()
        _check(_host(o), e)
    ctx.set_pipeline_depth(1)

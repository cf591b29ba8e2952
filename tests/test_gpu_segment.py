"""Segmentation against the reference library:
classify / quantize (proj/src/threshold.cpp:84-126) with given threshold
sets, and the per-frame video pipeline (proj/src/bench.cpp:266-281: curve ->
{optimal_threshold} -> two-class quantize, pass-through without boundary)
plus the segment command's top-k quantize (tools/kohler_main.cpp:91-103).
Bit-exact images and identical thresholds are required."""
import numpy as np
import pytest
import torch

import oracle
import paper_1707_05062_b200 as kb
from paper_1707_05062_b200 import synth

pytestmark = pytest.mark.gpu

TS_SETS = [[], [0], [255], [127], [3, 60, 200], [10, 11, 12, 250], list(range(0, 256, 37))]


def test_classify_quantize_golden_corpus(ctx, ref, corpus):
    imgs = corpus[0]
    for i, im in enumerate(imgs[:60]):
        for ts in TS_SETS:
            assert np.array_equal(ctx.classify(im, ts), oracle.ref_classify(ref, im, ts)), (i, ts)
            assert np.array_equal(ctx.quantize(im, ts), oracle.ref_quantize(ref, im, ts)), (i, ts)


@pytest.mark.parametrize("hw", [(1, 1), (1, 97), (61, 1), (33, 47), (480, 502), (1080, 1920)])
def test_classify_quantize_shapes(ctx, ref, hw):
    rng = np.random.default_rng(hw[0] * 1000 + hw[1])
    im = rng.integers(0, 256, size=hw, dtype=np.uint8)
    for ts in ([64], [17, 99, 180], [255]):
        assert np.array_equal(ctx.classify(im, ts), oracle.ref_classify(ref, im, ts))
        assert np.array_equal(ctx.quantize(im, ts), oracle.ref_quantize(ref, im, ts))


def test_dropin_classify_quantize_types(ctx, ref):
    im = synth.c1(device="cpu", w=96, h=80).numpy()
    ts = kb.ThresholdSet([40, 150])
    lab = kb.classify(im, ts)
    assert lab.width == 96 and lab.height == 80
    assert np.array_equal(lab.labels, oracle.ref_classify(ref, im, [40, 150]))
    q = kb.quantize(kb.GrayImage.from_array(im), ts)
    assert np.array_equal(q.pixels(), oracle.ref_quantize(ref, im, [40, 150]))


@pytest.mark.parametrize("k", [0, 1, 3, 6])
def test_segment_batch_video_frames(ctx, ref, k):
    """C3-style frames (K1 path) and one constant frame (pass-through)."""
    x = synth.generate("C3", device="cuda")[:3].cpu().numpy().copy()
    x = np.concatenate([x, np.full((1,) + x.shape[1:], 77, np.uint8)])
    out, ts, cnt, st = ctx.segment_batch(x, k)
    for i in range(x.shape[0]):
        exp, ets, est = oracle.ref_segment(ref, x[i], k, workers=8)
        assert int(st[i]) == est, i
        assert list(ts[i, :int(cnt[i])]) == list(ets), i
        assert np.array_equal(out[i], exp), i


def test_segment_batch_small_images(ctx, ref):
    """C5-style tiles (K5 path): all four families, incl. constant images."""
    x = synth.generate("C5", device="cuda")[:64].cpu().numpy()
    out, ts, cnt, st = ctx.segment_batch(x, 0)
    for i in range(x.shape[0]):
        exp, ets, est = oracle.ref_segment(ref, x[i], 0)
        assert int(st[i]) == est, i
        assert list(ts[i, :int(cnt[i])]) == list(ets), i
        assert np.array_equal(out[i], exp), i


def test_segment_batch_device_matches_host(ctx):
    x = synth.generate("C3", device="cuda")[:4]
    n, h, w = x.shape
    out = torch.empty_like(x)
    ts = torch.zeros((n, 1), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    st = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.segment_batch_device(x, w, h, w, w * h, n, 0, out, w, w * h, ts, cnt, st)
    torch.cuda.synchronize()
    hout, hts, hcnt, hst = ctx.segment_batch(x.cpu().numpy(), 0)
    assert np.array_equal(out.cpu().numpy(), hout)
    assert np.array_equal(ts.cpu().numpy(), hts)
    assert np.array_equal(st.cpu().numpy(), hst)

"""Colour ingest on the GPU: Rec. 601 integer luma,
bit-identical to the reference's read_pnm colour reduction (luma601,
proj/src/pnm.cpp:63-68, pinned by tests/golden/luma.npz and
tests/test_oracle.py), and the full pipeline on RGB input."""
import os

import numpy as np
import pytest
import torch

from paper_1707_05062_b200 import synth

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "luma.npz"))


def closed_form(rgb):
    a = rgb.astype(np.int64)
    t = 299 * a[..., 0] + 587 * a[..., 1] + 114 * a[..., 2] + 500
    return np.minimum(t // 1000, 255).astype(np.uint8)


def test_luma_all_2_24_triples(ctx):
    """Every RGB triple once: a 4096 x 4096 image whose pixel i is (i >> 16,
    i >> 8 & 255, i & 255), on the vector path and on an unaligned pitch."""
    i = torch.arange(1 << 24, dtype=torch.int64, device="cuda")
    rgb = torch.stack([(i >> 16) & 255, (i >> 8) & 255, i & 255], dim=1).to(torch.uint8)
    rgb = rgb.reshape(4096, 4096, 3).contiguous()
    gray = torch.empty((4096, 4096), dtype=torch.uint8, device="cuda")
    ctx.rgb_to_gray_device(rgb, 1, 4096, 4096, 3 * 4096, 3 * 4096 * 4096, gray, 4096, 4096 * 4096)
    torch.cuda.synchronize()
    want = closed_form(rgb.cpu().numpy())
    assert np.array_equal(gray.cpu().numpy(), want)
    # odd pitch: the per-pixel path
    rows = 64
    buf = torch.zeros((rows, 3 * 4096 + 7), dtype=torch.uint8, device="cuda")
    buf[:, 1:1 + 3 * 4096] = rgb[:rows].reshape(rows, -1)
    g2 = torch.empty((rows, 4099), dtype=torch.uint8, device="cuda")
    ctx.rgb_to_gray_device(buf.data_ptr() + 1, 1, 4096, rows, 3 * 4096 + 7, 0, g2, 4099, 0)
    torch.cuda.synchronize()
    assert np.array_equal(g2[:, :4096].cpu().numpy(), want[:rows])


def test_luma_golden_reference(ctx):
    assert np.array_equal(ctx.rgb_to_gray(GOLD["samples"][None])[0], GOLD["sample_gray"])
    assert np.array_equal(ctx.rgb_to_gray(GOLD["rgb"]), GOLD["gray"])
    assert np.array_equal(ctx.rgb_to_gray(GOLD["rgb"][:5, :7]), GOLD["gray_p3"])


def test_analyze_rgb_golden(ctx):
    r = ctx.analyze_rgb_batch(GOLD["rgb"], k=6)
    assert np.array_equal(r.sums[0], GOLD["sums"]) and np.array_equal(r.cards[0], GOLD["cards"])
    assert int(r.t0[0]) == int(GOLD["t0"]) and r.thresholds(0) == list(GOLD["topk"])


@pytest.mark.parametrize("w,h,n", [(1, 1, 1), (15, 9, 1), (17, 33, 3), (1000, 7, 2), (129, 130, 4)])
def test_analyze_rgb_host_and_device_vs_oracle(ctx, orc, w, h, n):
    rng = np.random.default_rng(w * 1000 + h + n)
    rgb = rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)
    rgb[:, h // 3:, : w // 2] = (10, 200, 30)
    r = ctx.analyze_rgb_batch(rgb, k=6)
    d = torch.from_numpy(rgb).cuda()
    out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
           "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "topk": torch.zeros((n, 6), dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.analyze_rgb_batch_device(d, w, h, 3 * w, 3 * w * h, n, 6, out)
    torch.cuda.synchronize()
    for i in range(n):
        e = orc.analyze(orc.rgb_to_gray(rgb[i]), 6)
        assert np.array_equal(r.sums[i], e["sum"]) and np.array_equal(r.cards[i], e["card"])
        assert np.array_equal(r.values[i], e["values"])
        assert int(r.t0[i]) == e["t0"] and r.thresholds(i) == e["topk"]
        assert np.array_equal(out["sums"][i].cpu().numpy().view(np.uint64), e["sum"])
        assert np.array_equal(out["cards"][i].cpu().numpy().view(np.uint64), e["card"])
        assert int(out["t0"][i]) == e["t0"] and int(out["status"][i]) == e["status"]
        cnt = int(out["topk_count"][i])
        assert out["topk"][i, :cnt].tolist() == e["topk"]


def test_analyze_rgb_c2_size_vs_reference(ctx, ref):
    """An 18 Mpx colour image (the C2 grey map in the green channel, shifted
    copies in red and blue): the GPU pipeline on RGB input against the
    reference's read_pnm + fast_contrast_curve + selection."""
    g = synth.generate("C2", device="cpu")[0].numpy()
    rgb = np.stack([np.roll(g, 3, axis=1), g, 255 - g], axis=2)
    h, w = g.shape
    r = ctx.analyze_rgb_batch(rgb, k=6)
    gray = ref.read_pnm(b"P6\n%d %d\n255\n" % (w, h) + rgb.tobytes())
    e = ref.analyze(gray, k=6, workers=8)
    assert np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"])
    assert int(r.t0[0]) == e["t0"] and r.thresholds(0) == e["topk"]


def test_rgb_argument_errors(ctx):
    with pytest.raises(ValueError):
        ctx.rgb_to_gray(np.zeros((4, 4), np.uint8))
    d = torch.zeros((4, 12), dtype=torch.uint8, device="cuda")
    g = torch.zeros((4, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):  # rgb pitch < 3 w
        ctx.rgb_to_gray_device(d, 1, 4, 4, 11, 0, g, 4, 0)

"""K1 over interleaved RGB (colour ingest fused into the accumulation walk,
SURVEY.md §8f rank 3): for rows of whole 16-pixel segments with 16-byte
aligned rows, kohler_cuda_analyze_rgb_batch_device runs the walk straight on
the RGB buffer (each lane converts its 48 bytes with the reference's
luma601, proj/src/pnm.cpp:63-68) -- no grey image is written.  Checked
against the oracle (luma601 + the reference's curve and selection,
proj/src/direct.cpp:10-43, threshold.cpp) and against the two-pass path
(luma_kernel + K1, forced by KOHLER_RGB_UNFUSED=1)."""
import os

import numpy as np
import pytest
import torch

from paper_1707_05062_b200 import Context

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def unfused():
    old = os.environ.get("KOHLER_RGB_UNFUSED")
    os.environ["KOHLER_RGB_UNFUSED"] = "1"
    try:
        c = Context(0)
    finally:
        if old is None:
            del os.environ["KOHLER_RGB_UNFUSED"]
        else:
            os.environ["KOHLER_RGB_UNFUSED"] = old
    yield c
    c.close()


def _out(n, k=6):
    z = lambda *s, dt=torch.int64: torch.zeros(s, dtype=dt, device="cuda")
    return {"sums": z(n, 256), "cards": z(n, 256), "values": z(n, 256, dt=torch.float64),
            "defined": z(n, 256, dt=torch.uint8), "t0": z(n, dt=torch.int32),
            "topk": z(n, k, dt=torch.int32), "topk_count": z(n, dt=torch.int32),
            "status": z(n, dt=torch.int32)}


def _image(rng, h, w, kind):
    if kind == "noise":
        return rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    if kind == "flat":
        return np.full((h, w, 3), 77, np.uint8)
    # regions + noise: smooth luma with boundaries, all three channels differ
    yy, xx = np.mgrid[0:h, 0:w]
    base = ((xx * 7 // max(w, 1) + yy * 5 // max(h, 1)) % 4) * 60 + 20
    rgb = np.stack([base, 255 - base, (base * 3) % 256], axis=2).astype(np.int64)
    rgb += rng.integers(-6, 7, rgb.shape)
    return np.clip(rgb, 0, 255).astype(np.uint8)


def _run(ctx, rgb, pad_pitch=0, pad_stride=0):
    """rgb[n, h, w, 3] through the device API in a (possibly padded) buffer."""
    n, h, w = rgb.shape[:3]
    pitch = 3 * w + pad_pitch
    stride = pitch * h + pad_stride
    buf = torch.zeros(n * stride + 64, dtype=torch.uint8, device="cuda")
    for i in range(n):
        v = buf[i * stride:i * stride + pitch * h].view(h, pitch)
        v[:, :3 * w] = torch.from_numpy(rgb[i].reshape(h, 3 * w)).cuda()
    out = _out(n)
    ctx.analyze_rgb_batch_device(buf, w, h, pitch, stride, n, 6, out)
    torch.cuda.synchronize()
    return out, ctx.last_launch_count()


def _check(out, orc, rgb):
    for i in range(rgb.shape[0]):
        e = orc.analyze(orc.rgb_to_gray(rgb[i]), 6)
        assert np.array_equal(out["sums"][i].cpu().numpy().view(np.uint64), e["sum"]), i
        assert np.array_equal(out["cards"][i].cpu().numpy().view(np.uint64), e["card"]), i
        assert np.array_equal(out["values"][i].cpu().numpy(), e["values"]), i
        assert int(out["t0"][i]) == e["t0"] and int(out["status"][i]) == e["status"], i
        cnt = int(out["topk_count"][i])
        assert out["topk"][i, :cnt].tolist() == e["topk"], i


@pytest.mark.parametrize("w,h,n,kind,pp,ps", [
    (16, 1, 1, "noise", 0, 0),          # one segment, one row (fake down pairs only)
    (16, 2, 1, "noise", 0, 0),
    (32, 37, 1, "regions", 16, 0),      # padded pitch
    (48, 300, 1, "noise", 0, 0),        # several walks per column
    (512, 129, 1, "regions", 0, 0),
    (528, 131, 1, "noise", 32, 0),      # 33 segments: one lane group wraps a row
    (1024, 1024, 1, "regions", 0, 0),   # many CTAs share the border rows
    (256, 300, 2, "noise", 0, 0),       # batch (images larger than the small-image path)
    (272, 257, 3, "regions", 48, 96),   # batch with padded pitch and stride
    (4096, 40, 2, "flat", 0, 0),        # no boundary: status / t0 = -1
])
def test_fused_rgb_vs_oracle(ctx, unfused, orc, w, h, n, kind, pp, ps):
    rng = np.random.default_rng(w * 7919 + h * 31 + n)
    rgb = np.stack([_image(rng, h, w, kind) for _ in range(n)])
    out, launches = _run(ctx, rgb, pp, ps)
    # K1 over RGB (+ finish_kernel unless the single-image K1 finishes itself):
    # no luma_kernel, no grey image
    assert launches in ((1, 2) if n == 1 else (2,))
    _check(out, orc, rgb)
    out2, launches2 = _run(unfused, rgb, pp, ps)
    assert launches2 == launches + 1  # + luma_kernel
    for key in ("sums", "cards", "values", "t0", "topk", "topk_count", "status"):
        assert torch.equal(out[key], out2[key]), key


def test_fused_rgb_layouts_that_take_the_two_pass_path(ctx, orc):
    """Widths off the 16-pixel grid, unaligned bases / pitches and small
    batches keep the luma_kernel path; results are the same either way."""
    rng = np.random.default_rng(5)
    rgb = rng.integers(0, 256, (1, 40, 100, 3), dtype=np.uint8)  # w % 16 != 0
    out, launches = _run(ctx, rgb)
    assert launches in (2, 3)  # luma_kernel + K1 (+ finish_kernel)
    _check(out, orc, rgb)
    rgb = rng.integers(0, 256, (1, 40, 96, 3), dtype=np.uint8)
    out, launches = _run(ctx, rgb, pad_pitch=8)  # pitch % 16 != 0
    assert launches in (2, 3)
    _check(out, orc, rgb)


def test_fused_rgb_pipelined_and_c3_frame(ctx, orc):
    """A 1080p colour frame at pipeline depth 3 (3 launches in flight share
    the SMs), repeated: identical results each time."""
    from paper_1707_05062_b200 import synth
    g = synth.generate("C3", device="cpu", n=1)[0].numpy()
    rgb = np.stack([g, np.roll(g, 5, axis=0), 255 - g], axis=2)[None]
    ctx.set_pipeline_depth(3)
    try:
        outs = [_run(ctx, rgb)[0] for _ in range(3)]
    finally:
        ctx.set_pipeline_depth(1)
    _check(outs[0], orc, rgb)
    for o in outs[1:]:
        for key in ("sums", "cards", "t0", "topk"):
            assert torch.equal(o[key], outs[0][key])


@pytest.mark.parametrize("w,h,n", [(2048, 2100, 1), (1024, 1500, 3), (64, 48, 1)])
def test_fused_rgb_host_path(ctx, unfused, orc, w, h, n):
    """kohler_cuda_analyze_rgb_batch from host memory: uploads in two chunks
    above 4 Mpx (a row band + its halo row for one image, whole images for a
    batch), K1 over the uploaded RGB rows."""
    rng = np.random.default_rng(w + h + n)
    rgb = np.stack([_image(rng, h, w, "regions") for _ in range(n)])
    r = ctx.analyze_rgb_batch(rgb, k=6)
    # one image: [K1 of band 1] + K1 of band 2, the last K1 finishing the image
    # itself; a batch: (K1 + finish_kernel) per chunk of several images
    lc = ctx.last_launch_count()
    assert lc in ((2, 3) if w * h >= 4 << 20 else (1, 2)) if n == 1 else lc == 4
    r2 = unfused.analyze_rgb_batch(rgb, k=6)
    for i in range(n):
        e = orc.analyze(orc.rgb_to_gray(rgb[i]), 6)
        assert np.array_equal(r.sums[i], e["sum"]) and np.array_equal(r.cards[i], e["card"])
        assert np.array_equal(r.values[i], e["values"])
        assert int(r.t0[i]) == e["t0"] and r.thresholds(i) == e["topk"]
        assert np.array_equal(r2.sums[i], r.sums[i]) and r2.thresholds(i) == r.thresholds(i)

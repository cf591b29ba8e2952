"""Argument guards and size limits of the device / host API:

* misaligned device output pointers are refused (KOHLER_INVALID_ARGUMENT ->
  ValueError) instead of raising a sticky misaligned-address fault;
* a very large k returns every local maximum (the reference truncates a
  shorter list, proj/src/threshold.cpp:69-81) without allocating k slots;
* rows wider than 2^32 / 160 bytes (the old 32-bit walk-offset limit) run
  through K1 with 64-bit row offsets, bit-exact against the oracle.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_misaligned_outputs_refused(ctx):
    x = torch.zeros((1, 64, 64), dtype=torch.uint8, device="cuda")
    x[0, 10:20, 10:20] = 9
    buf = torch.zeros(4096, dtype=torch.int64, device="cuda")
    for off in (8, 4):
        with pytest.raises(ValueError):
            ctx.analyze_batch_device(x, 64, 64, 64, 64 * 64, 1, 6, {"sums": buf.data_ptr() + off})
    with pytest.raises(ValueError):
        ctx.select_device(buf.data_ptr() + 8, buf.data_ptr() + 4096, 1, 256, 6,
                          {"t0": buf.data_ptr() + 2})
    # the context is still healthy afterwards (nothing faulted)
    s = torch.zeros((1, 256), dtype=torch.int64, device="cuda")
    ctx.analyze_batch_device(x, 64, 64, 64, 64 * 64, 1, 6, {"sums": s})
    torch.cuda.synchronize()
    assert int(s.sum()) > 0


def test_wrong_tensor_kinds_refused(ctx):
    x = torch.zeros((1, 16, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        ctx.analyze_batch_device(x.cpu(), 16, 16, 16, 256, 1, 6, {})
    with pytest.raises(ValueError):
        ctx.analyze_batch_device(x.int(), 16, 16, 16, 256, 1, 6, {})
    with pytest.raises(ValueError):
        ctx.analyze_batch_device(x, 16, 16, 16, 256, 1, 6,
                                 {"sums": torch.zeros((1, 256), dtype=torch.float32, device="cuda")})
    with pytest.raises(ValueError):
        ctx.analyze_batch_device(x, 16, 16, 16, 256, 1, 6,
                                 {"t0": torch.zeros((2, 2), dtype=torch.int32, device="cuda").t()})


def test_huge_k_returns_all_maxima(ctx, orc):
    from paper_1707_05062_b200 import mean_contrast, top_k_local_maxima
    from paper_1707_05062_b200 import synth
    img = synth.c1(device="cpu").numpy()
    c = ctx.curve(img)
    mc = mean_contrast(c)
    ts = top_k_local_maxima(mc, 2 ** 30)
    st, exp = orc.top_k(mc.values, mc.defined.astype(np.uint8), 256)
    assert st == 0 and ts.thresholds == exp and len(exp) > 6


def test_rows_wider_than_old_pitch_limit(ctx, orc):
    w, h = 28_000_000, 3  # pitch 28 MB > 2^32 / 160
    g = torch.Generator(device="cpu")
    g.manual_seed(3)
    steps = torch.randint(-3, 4, (h, w), generator=g, dtype=torch.int16)
    img = (torch.cumsum(steps, dim=1) % 256).to(torch.uint8)
    img[1] = img[0].roll(5)
    img[2] = 255 - img[0]
    e = orc.analyze(img.numpy(), 6)
    out = {"sums": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
           "cards": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
           "t0": torch.zeros(1, dtype=torch.int32, device="cuda")}
    x = img.cuda()[None]
    ctx.analyze_batch_device(x, w, h, w, w * h, 1, 6, out)
    torch.cuda.synchronize()
    assert np.array_equal(out["sums"][0].cpu().numpy().view(np.uint64), e["sum"])
    assert np.array_equal(out["cards"][0].cpu().numpy().view(np.uint64), e["card"])
    assert int(out["t0"][0]) == e["t0"]


@pytest.mark.parametrize("shape", [(1, 300, 260), (40, 128, 128)])  # K1 and K5 paths
def test_partial_output_sets(ctx, orc, shape):
    """Any output pointer may be NULL (include/kohler_cuda.h): sums without
    cards, cards without sums, thresholds only."""
    g = torch.Generator(device="cpu")
    g.manual_seed(11)
    x = torch.randint(0, 256, shape, generator=g, dtype=torch.uint8)
    n, h, w = shape
    exp = [orc.analyze(x[i].numpy(), 6) for i in range(n)]
    xd = x.cuda()
    for keys in (("sums",), ("cards",), ("t0", "topk_count"), ("sums", "t0")):
        out = {}
        for k in keys:
            if k in ("sums", "cards"):
                out[k] = torch.zeros((n, 256), dtype=torch.int64, device="cuda")
            else:
                out[k] = torch.zeros(n, dtype=torch.int32, device="cuda")
        if "topk_count" in out:
            out["topk"] = torch.zeros((n, 6), dtype=torch.int32, device="cuda")
        ctx.analyze_batch_device(xd, w, h, w, w * h, n, 6, out)
        torch.cuda.synchronize()
        for i in range(n):
            if "sums" in out:
                assert np.array_equal(out["sums"][i].cpu().numpy().view(np.uint64), exp[i]["sum"])
            if "cards" in out:
                assert np.array_equal(out["cards"][i].cpu().numpy().view(np.uint64), exp[i]["card"])
            if "t0" in out:
                assert int(out["t0"][i]) == exp[i]["t0"]

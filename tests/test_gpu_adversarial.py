"""Full-size adversarial inputs for K1 with closed-form expected curves.

The packed W lane words of K1 hold 16-bit fields whose epoch bound is proved
in kohler_launch.cuh (<= 8191 pixel events per lane word between spills, so
the sign-sum field, <= 8 per event, cannot overflow).  These inputs put every
pixel event of a lane onto ONE or TWO keys with the extreme B values:

* a constant 16384^2 image: every pixel on one key, B = 4 (all pairs equal):
  empty boundary, count = sum = 0 everywhere, NoBoundary (the reference's
  zero curve and NoBoundaryError, proj/tests/test_contrast.cpp:87-91,120-123);
* 0/255 checkerboards with cell 1 (B = 8 on the 0 pixels, B = 0 on the 255
  ones: every event on two keys) and cell 8: every boundary pair is (0, 255),
  whose tent is min(t, 255 - t) on [0, 255) (proj/src/kernels/pair_tent.hpp:12-18),
  so with N boundary pairs card[t] = N and sum[t] = N min(t, 255 - t) for
  t <= 254 (the 2x2 checker case of proj/tests/test_contrast.cpp:105-118 at
  full size), the mean curve is min(t, 255 - t), t0 = 127 (tie with 128 goes
  to the smaller t) and the only local maximum is 127;
* a 0/255 image of horizontal stripes (only down pairs cross) and of
  vertical stripes (only right pairs), same closed form.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K = 6
S = 16384


def run(ctx, x, k=K):
    n, h, w = x.shape
    out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
           "defined": torch.zeros((n, 256), dtype=torch.uint8, device="cuda"),
           "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "topk": torch.zeros((n, k), dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.analyze_batch_device(x, w, h, w, w * h, n, k, out)
    torch.cuda.synchronize()
    r = {key: v.cpu().numpy() for key, v in out.items()}
    r["sums"] = r["sums"].view(np.uint64)
    r["cards"] = r["cards"].view(np.uint64)
    return r


def expect_0_255(nb):
    t = np.arange(256, dtype=np.uint64)
    card = np.where(t <= 254, np.uint64(nb), np.uint64(0)).astype(np.uint64)
    s = np.minimum(t, np.uint64(255) - np.minimum(t, np.uint64(255))) * np.uint64(nb)
    s[255] = 0
    return s, card


def check_0_255(r, nb):
    s, c = expect_0_255(nb)
    assert np.array_equal(r["cards"][0], c)
    assert np.array_equal(r["sums"][0], s)
    t = np.arange(256)
    vals = np.where(t <= 254, np.minimum(t, 255 - t).astype(np.float64), 0.0)
    assert np.array_equal(r["values"][0], vals)
    assert int(r["t0"][0]) == 127 and int(r["status"][0]) == 0
    assert int(r["topk_count"][0]) == 1 and int(r["topk"][0][0]) == 127


@pytest.mark.parametrize("value", [0, 77, 255])
def test_constant_16384(ctx, value):
    x = torch.full((1, S, S), value, dtype=torch.uint8, device="cuda")
    r = run(ctx, x)
    assert not r["sums"].any() and not r["cards"].any()
    assert int(r["status"][0]) == 1 and int(r["t0"][0]) == -1 and int(r["topk_count"][0]) == 0
    assert not r["defined"].any()


@pytest.mark.parametrize("cell", [1, 8])
def test_checkerboard_16384(ctx, cell):
    ys = torch.arange(S, device="cuda")
    x = ((((ys[:, None] // cell) + (ys[None, :] // cell)) % 2) * 255).to(torch.uint8)[None]
    r = run(ctx, x.contiguous())
    per_line = (S - 1) // cell  # boundary crossings along one row / column
    check_0_255(r, 2 * S * per_line)


@pytest.mark.parametrize("axis", [0, 1])
def test_stripes_16384(ctx, axis):
    ys = torch.arange(S, device="cuda")
    v = ((ys % 2) * 255).to(torch.uint8)
    x = (v[:, None].expand(S, S) if axis == 0 else v[None, :].expand(S, S)).contiguous()[None]
    r = run(ctx, x)
    check_0_255(r, S * (S - 1))


def test_checkerboard_batch_of_small(ctx):
    """The small-image path (K5) on cell 1..8 checkerboards of 128^2 (the C5
    family (c)) and on constant 128^2 images, against the closed form."""
    n, m = 64, 128
    ys = torch.arange(m, device="cuda")
    cells = [1 + (i % 8) for i in range(n)]
    x = torch.stack([((((ys[:, None] // c) + (ys[None, :] // c)) % 2) * 255).to(torch.uint8)
                     if i % 2 == 0 else torch.full((m, m), i, dtype=torch.uint8, device="cuda")
                     for i, c in enumerate(cells)])
    r = run(ctx, x)
    for i, c in enumerate(cells):
        if i % 2:
            assert not r["cards"][i].any() and int(r["status"][i]) == 1
            continue
        nb = 2 * m * ((m - 1) // c)
        s, cc = expect_0_255(nb)
        assert np.array_equal(r["cards"][i], cc), i
        assert np.array_equal(r["sums"][i], s), i
        assert int(r["t0"][i]) == 127 and list(r["topk"][i][: r["topk_count"][i]]) == [127]

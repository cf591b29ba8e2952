"""Seeded randomized cross-check of every GPU entry path against the oracle:
random batch sizes, shapes (1 .. 700 on a side), value distributions, and
paths (host batch, device batch with unaligned base / odd pitch, RGB input,
streaming submit/collect, band partials over a random row split).  Catches
shape-dependent corner cases the hand-picked tests might miss."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K = 6


def random_images(rng, n, h, w):
    kind = int(rng.integers(0, 5))
    if kind == 0:
        x = rng.integers(0, 256, (n, h, w))
    elif kind == 1:
        x = np.where(rng.random((n, h, w)) < 0.5, rng.integers(0, 256), rng.integers(0, 256))
    elif kind == 2:
        x = np.clip(rng.normal(rng.integers(0, 256), rng.integers(1, 30), (n, h, w)), 0, 255)
    elif kind == 3:
        ys, xs = np.mgrid[0:h, 0:w]
        x = np.broadcast_to((xs * int(rng.integers(1, 9)) + ys * int(rng.integers(1, 9))) % 256,
                            (n, h, w))
    else:
        x = np.full((n, h, w), rng.integers(0, 256))
    return np.ascontiguousarray(x, dtype=np.uint8)


def check(r, i, e):
    assert np.array_equal(r.sums[i], e["sum"]) and np.array_equal(r.cards[i], e["card"])
    assert int(r.t0[i]) == e["t0"] and r.thresholds(i) == e["topk"]
    assert int(r.status[i]) == e["status"]


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_paths_vs_oracle(ctx, orc, seed):
    rng = np.random.default_rng(1000 + seed)
    for case in range(40):
        n = int(rng.choice([1, 1, 2, 3, 7, 16, 33]))
        h = int(rng.integers(1, 200 if n > 1 else 700))
        w = int(rng.integers(1, 200 if n > 1 else 700))
        x = random_images(rng, n, h, w)
        exp = [orc.analyze(x[i], K) for i in range(n)]
        path = case % 5
        if path == 0:  # host batch
            r = ctx.analyze_batch(x, K)
            for i in range(n):
                check(r, i, exp[i])
        elif path == 1:  # device batch, unaligned base and odd pitch
            pitch = w + int(rng.integers(1, 19))
            off = int(rng.integers(1, 16))
            buf = torch.zeros(off + n * h * pitch + 16, dtype=torch.uint8, device="cuda")
            v = buf[off: off + n * h * pitch].view(n, h, pitch)
            v[:, :, :w] = torch.from_numpy(x).cuda()
            out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
                   "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
                   "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
                   "topk": torch.zeros((n, K), dtype=torch.int32, device="cuda"),
                   "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
                   "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
            ctx.analyze_batch_device(buf.data_ptr() + off, w, h, pitch, h * pitch, n, K, out)
            torch.cuda.synchronize()
            for i in range(n):
                e = exp[i]
                assert np.array_equal(out["sums"][i].cpu().numpy().view(np.uint64), e["sum"])
                assert np.array_equal(out["cards"][i].cpu().numpy().view(np.uint64), e["card"])
                assert int(out["t0"][i]) == e["t0"] and int(out["status"][i]) == e["status"]
                cnt = int(out["topk_count"][i])
                assert out["topk"][i, :cnt].tolist() == e["topk"]
        elif path == 2:  # RGB: grey on every channel -> the same luma
            rgb = np.repeat(x[..., None], 3, axis=3)
            r = ctx.analyze_rgb_batch(rgb, K)
            for i in range(n):
                check(r, i, exp[i])
        elif path == 3:  # streaming, two in flight
            t1 = ctx.submit(x, K)
            t2 = ctx.submit(x[:, ::-1, :].copy(), K)
            r1, r2 = ctx.collect(t1), ctx.collect(t2)
            for i in range(n):
                check(r1, i, exp[i])
                e2 = orc.analyze(np.ascontiguousarray(x[i, ::-1, :]), K)
                check(r2, i, e2)
        else:  # band partials over a random split of one image
            img = x[0]
            cuts = sorted(set([0, h] + [int(c) for c in rng.integers(1, max(h, 2), 3) if 0 < c < h]))
            d = torch.from_numpy(img).cuda()
            tot_s = np.zeros(256, np.uint64)
            tot_c = np.zeros(256, np.uint64)
            for a, b in zip(cuts[:-1], cuts[1:]):
                band = d[a: min(b + 1, h)].contiguous()
                cs = torch.zeros(512, dtype=torch.int64, device="cuda")
                ctx.band_curve_device(band, w, w, h, a, b, cs.data_ptr(), cs.data_ptr() + 2048)
                torch.cuda.synchronize()
                c = cs.cpu().numpy().view(np.uint64)
                tot_s += c[:256]
                tot_c += c[256:]
            assert np.array_equal(tot_s, exp[0]["sum"]) and np.array_equal(tot_c, exp[0]["card"])

"""Parity of the CUDA path (through the C ABI) with the oracle, the
reference's golden vectors and the reference library itself.  Bit-exact for
the integer curves, the double curve (compared with ==) and the thresholds."""
import threading

import numpy as np
import pytest
import torch

import paper_1707_05062_b200 as kb
from paper_1707_05062_b200 import synth

pytestmark = pytest.mark.gpu

CHECKER = np.array([[0, 255], [255, 0]], np.uint8)
COLUMN_2_5 = np.array([[2], [5]], np.uint8)


def assert_result_matches(r, i, exp):
    assert np.array_equal(r.sums[i], exp["sum"]), "contrast_sum"
    assert np.array_equal(r.cards[i], exp["card"]), "cardinality"
    assert np.array_equal(r.values[i], exp["values"]), "mean curve (bitwise)"
    assert np.array_equal(r.defined[i], exp["defined"]), "defined"
    assert int(r.t0[i]) == exp["t0"]
    assert r.thresholds(i) == exp["topk"]
    assert int(r.status[i]) == exp["status"]


def test_hand_examples(ctx):
    c = kb.fast_contrast_curve(COLUMN_2_5)
    assert [int(x) for x in c.cardinality[:6]] == [0, 0, 1, 1, 1, 0]
    assert [int(x) for x in c.contrast_sum[2:5]] == [0, 1, 1]
    c = kb.fast_contrast_curve(CHECKER, 2)
    assert int(c.contrast_sum[127]) == 508
    assert all(int(c.cardinality[t]) == (4 if t <= 254 else 0) for t in range(256))
    assert kb.fast_contrast_curve(np.array([[42]], np.uint8)) == kb.ContrastCurve()
    assert kb.fast_contrast_curve(np.full((2, 2), 100, np.uint8)) == kb.ContrastCurve()
    mc = kb.mean_contrast(kb.fast_contrast_curve(CHECKER))
    assert kb.optimal_threshold(mc) == 127
    assert kb.top_k_local_maxima(mc, 1).thresholds == [127]
    assert kb.optimal_threshold(kb.mean_contrast(kb.fast_contrast_curve(COLUMN_2_5))) == 3
    with pytest.raises(kb.NoBoundaryError):
        kb.optimal_threshold(kb.mean_contrast(kb.fast_contrast_curve(np.full((3, 3), 42, np.uint8))))
    with pytest.raises(ValueError):
        kb.fast_contrast_curve(CHECKER, 0)


def test_golden_corpus_one_call_per_image(ctx, corpus):
    imgs, z = corpus
    for i, im in enumerate(imgs):
        r = ctx.analyze_batch(im[None], 6)
        exp = dict(sum=z["sums"][i], card=z["cards"][i], values=z["values"][i],
                   defined=z["defined"][i], t0=int(z["t0"][i]),
                   topk=[int(t) for t in z["topk"][i] if t >= 0], status=int(z["status"][i]))
        assert_result_matches(r, 0, exp)


def test_golden_corpus_dropin_functions(ctx, corpus):
    imgs, z = corpus
    for i, im in enumerate(imgs[:60]):
        c = kb.fast_contrast_curve(im, 1 + i % 4)
        assert np.array_equal(c.contrast_sum, z["sums"][i])
        assert np.array_equal(c.cardinality, z["cards"][i])
        d = kb.direct_contrast_curve(im)
        assert d == c
        mc = kb.mean_contrast(c)
        assert np.array_equal(mc.values, z["values"][i])
        if z["status"][i] == 0:
            assert kb.optimal_threshold(mc) == z["t0"][i]
            assert kb.top_k_local_maxima(mc, 6).thresholds == [int(t) for t in z["topk"][i] if t >= 0]
        else:
            with pytest.raises(kb.NoBoundaryError):
                kb.optimal_threshold(mc)
            with pytest.raises(kb.NoBoundaryError):
                kb.top_k_local_maxima(mc, 6)


def _mixed_batch(rng, n, h, w):
    out = np.empty((n, h, w), np.uint8)
    for i in range(n):
        kind = i % 5
        if kind == 0:
            out[i] = rng.integers(0, 256, (h, w))
        elif kind == 1:
            out[i] = np.where(rng.random((h, w)) < 0.5, rng.integers(0, 256), rng.integers(0, 256))
        elif kind == 2:
            out[i] = rng.integers(0, 256)
        elif kind == 3:
            out[i] = np.clip(rng.normal(rng.integers(0, 256), 4, (h, w)), 0, 255)
        else:
            ys, xs = np.mgrid[0:h, 0:w]
            out[i] = ((xs * 3 + ys * 7) % 256)
    return out


@pytest.mark.parametrize("shape", [(300, 23, 37), (40, 1, 200), (40, 200, 1), (16, 16, 16),
                                   (9, 31, 129), (5, 130, 512), (3, 3, 2000)])
def test_batch_against_oracle(ctx, orc, shape):
    rng = np.random.default_rng(sum(shape))
    imgs = _mixed_batch(rng, *shape)
    r = ctx.analyze_batch(imgs, 6)
    for i in range(shape[0]):
        assert_result_matches(r, i, orc.analyze(imgs[i], 6))


@pytest.mark.parametrize("k", [1, 2, 3, 6, 9, 40])
def test_batch_k_values(ctx, orc, k):
    rng = np.random.default_rng(k)
    imgs = _mixed_batch(rng, 25, 41, 57)
    r = ctx.analyze_batch(imgs, k)
    for i in range(25):
        exp = orc.analyze(imgs[i], k)
        assert int(r.t0[i]) == exp["t0"] and r.thresholds(i) == exp["topk"]


def test_device_api_unaligned_and_pitched(ctx, orc):
    rng = np.random.default_rng(3)
    n, h, w = 7, 45, 101
    imgs = _mixed_batch(rng, n, h, w)
    for pitch, stride, offset in [(w, w * h, 0), (w, w * h, 3), (112, 112 * h, 0),
                                  (128, 128 * h + 16, 16)]:
        buf = np.zeros(offset + stride * n + 64, np.uint8)
        for i in range(n):
            base = offset + i * stride
            for y in range(h):
                buf[base + y * pitch: base + y * pitch + w] = imgs[i, y]
        d = torch.from_numpy(buf).cuda()
        out = {k: torch.zeros((n, 256), dtype=torch.int64, device="cuda") for k in ("sums", "cards")}
        out["t0"] = torch.zeros(n, dtype=torch.int32, device="cuda")
        out["topk"] = torch.zeros((n, 6), dtype=torch.int32, device="cuda")
        out["topk_count"] = torch.zeros(n, dtype=torch.int32, device="cuda")
        ctx.analyze_batch_device(d.data_ptr() + offset, w, h, pitch, stride, n, 6, out)
        torch.cuda.synchronize()
        sums = out["sums"].cpu().numpy().view(np.uint64)
        cards = out["cards"].cpu().numpy().view(np.uint64)
        for i in range(n):
            exp = orc.analyze(imgs[i], 6)
            assert np.array_equal(sums[i], exp["sum"]) and np.array_equal(cards[i], exp["card"])
            cnt = int(out["topk_count"][i])
            assert int(out["t0"][i]) == exp["t0"]
            assert out["topk"][i, :cnt].tolist() == exp["topk"]


@pytest.mark.parametrize("hw", [(61, 97), (50, 1), (1, 50), (16, 16), (300, 700), (7, 33)])
def test_band_partials(ctx, orc, hw):
    h, w = hw
    rng = np.random.default_rng(h * 1000 + w)
    im = rng.integers(0, 256, (h, w), dtype=np.uint8)
    full = orc.fast_curve(im)
    splits = [[0, h]]
    if h > 1:
        splits.append([0, 1, h])
        splits.append(sorted(set([0, h] + list(rng.integers(1, h, size=min(5, h - 1))))))
        splits.append(list(range(0, h + 1)))  # 1-row bands
    d = torch.from_numpy(im).cuda()
    for cuts in splits:
        tot_s = torch.zeros(256, dtype=torch.int64, device="cuda")
        tot_c = torch.zeros(256, dtype=torch.int64, device="cuda")
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            s = torch.zeros(256, dtype=torch.int64, device="cuda")
            c = torch.zeros(256, dtype=torch.int64, device="cuda")
            band = d[r0:min(r1 + 1, h)].contiguous()
            ctx.band_curve_device(band, w, w, h, r0, r1, s, c)
            torch.cuda.synchronize()
            es, ec = orc.curve_rows(im, r0, r1)
            assert np.array_equal(s.cpu().numpy().view(np.uint64), es), (cuts, r0, r1)
            assert np.array_equal(c.cpu().numpy().view(np.uint64), ec), (cuts, r0, r1)
            tot_s += s
            tot_c += c
        assert np.array_equal(tot_s.cpu().numpy().view(np.uint64), full[0])
        assert np.array_equal(tot_c.cpu().numpy().view(np.uint64), full[1])


def test_selection_golden(ctx, selection):
    z = selection
    for i in range(z["values"].shape[0]):
        mc = kb.MeanContrastCurve(z["values"][i], z["defined"][i].astype(bool))
        if z["t0"][i] < 0:
            with pytest.raises(kb.NoBoundaryError):
                ctx.optimal_threshold(mc)
        else:
            assert ctx.optimal_threshold(mc) == z["t0"][i]
        for k in range(1, 9):
            if z["status"][i, k - 1] == 1:
                with pytest.raises(kb.NoBoundaryError):
                    ctx.top_k_local_maxima(mc, k)
            else:
                exp = [int(t) for t in z["topk"][i, k - 1] if t >= 0]
                assert ctx.top_k_local_maxima(mc, k).thresholds == exp, (i, k)


def test_selection_device_many_curves(ctx, orc, selection):
    """select_kernel on device curves (mean + t0 + top-k) vs the oracle."""
    rng = np.random.default_rng(11)
    n = 500
    card = rng.integers(0, 4, (n, 256)).astype(np.uint64) * np.uint64(3)
    sums = (card * rng.integers(0, 5, (n, 256)).astype(np.uint64))
    sums[card == 0] = 0
    card[::50] = 0
    sums[::50] = 0
    ds = torch.from_numpy(sums.view(np.int64)).cuda()
    dc = torch.from_numpy(card.view(np.int64)).cuda()
    out = {"values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
           "defined": torch.zeros((n, 256), dtype=torch.uint8, device="cuda"),
           "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "topk": torch.zeros((n, 5), dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.select_device(ds, dc, n, 256, 5, out)
    torch.cuda.synchronize()
    for i in range(n):
        v, d = orc.mean_contrast(sums[i], card[i])
        assert np.array_equal(out["values"][i].cpu().numpy(), v)
        assert np.array_equal(out["defined"][i].cpu().numpy(), d)
        assert int(out["t0"][i]) == orc.optimal_threshold(v, d)
        st, tk = orc.top_k(v, d, 5)
        assert int(out["status"][i]) == st
        assert out["topk"][i, : int(out["topk_count"][i])].tolist() == tk


def _select_patterns(rng, n):
    """(sums, cards) curves that stress the run / maxima rules: long plateaus
    across lane boundaries (8 thresholds per lane), alternating values (more
    than 32 maxima: the ranked top-k over 4 candidates per lane), sparse
    defined masks, equal maxima (ties to the smaller t), single defined
    entries, monotone ramps."""
    sums = np.zeros((n, 256), np.uint64)
    card = np.ones((n, 256), np.uint64)
    for i in range(n):
        kind = i % 8
        if kind == 0:    # plateaus of random length, few distinct values
            v = np.repeat(rng.integers(0, 4, 256), rng.integers(1, 40, 256))[:256]
        elif kind == 1:  # alternating: ~128 maxima, many equal
            v = (np.arange(256) % 2) * rng.integers(1, 3, 256)
        elif kind == 2:  # sparse defined mask over a noisy curve
            v = rng.integers(0, 50, 256)
            card[i] = (rng.random(256) < 0.15).astype(np.uint64)
        elif kind == 3:  # equal peaks on a flat floor
            v = np.zeros(256, np.int64)
            v[rng.choice(256, rng.integers(1, 20), replace=False)] = 7
        elif kind == 4:  # one defined entry / one defined run at a lane edge
            v = rng.integers(1, 9, 256)
            card[i] = 0
            a = int(rng.integers(0, 256))
            card[i, a:a + int(rng.integers(1, 10))] = 1
        elif kind == 5:  # monotone up, then down (one maximum), plateau top
            a = int(rng.integers(1, 255))
            v = np.minimum(np.arange(256), a) - np.maximum(np.arange(256) - a - int(rng.integers(0, 9)), 0)
            v = v - v.min()
        elif kind == 6:  # noisy with fractional means (card > 1)
            v = rng.integers(0, 1000, 256)
            card[i] = rng.integers(1, 7, 256).astype(np.uint64)
        else:            # two-valued blocks aligned to the 8-threshold lanes
            v = np.repeat(rng.integers(0, 3, 32), 8)
        sums[i] = np.asarray(v, np.int64).astype(np.uint64)
        sums[i][card[i] == 0] = 0
    return sums, card


@pytest.mark.parametrize("k", [1, 2, 6, 40, 200])
def test_selection_rule_patterns(ctx, orc, k):
    """select256_kernel (votes / indexed shuffles / ranked top-k) against the
    oracle's restatement of threshold.cpp:25-82 on adversarial curve shapes."""
    rng = np.random.default_rng(1000 + k)
    n = 640
    sums, card = _select_patterns(rng, n)
    ds = torch.from_numpy(sums.view(np.int64)).cuda()
    dc = torch.from_numpy(card.view(np.int64)).cuda()
    out = {"values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
           "defined": torch.zeros((n, 256), dtype=torch.uint8, device="cuda"),
           "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "topk": torch.full((n, k), -7, dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.select_device(ds, dc, n, 256, k, out)
    torch.cuda.synchronize()
    t0 = out["t0"].cpu().numpy()
    cnt = out["topk_count"].cpu().numpy()
    tk = out["topk"].cpu().numpy()
    st = out["status"].cpu().numpy()
    for i in range(n):
        v, d = orc.mean_contrast(sums[i], card[i])
        est, etk = orc.top_k(v, d, k)
        assert int(st[i]) == est, i
        assert int(t0[i]) == orc.optimal_threshold(v, d), i
        assert tk[i, : int(cnt[i])].tolist() == etk, (i, i % 8)


def test_selection_signed_values(ctx, orc):
    """Host curves with negative values and -0.0 (the selection orders values
    through an integer key; -0.0 must tie with +0.0 like the IEEE compare)."""
    rng = np.random.default_rng(5)
    for i in range(60):
        v = rng.integers(-3, 4, 256).astype(np.float64) * 0.5
        if i % 3 == 0:
            v[v == 0.0] = -0.0 if i % 2 else 0.0
            v[rng.integers(0, 256, 40)] = -0.0
        d = rng.random(256) < (0.9 if i % 2 else 0.3)
        if not d.any():
            d[17] = True
        mc = kb.MeanContrastCurve(v, d)
        dd = d.astype(np.uint8)
        assert ctx.optimal_threshold(mc) == orc.optimal_threshold(v, dd)
        for k in (1, 3, 9):
            est, etk = orc.top_k(v, dd, k)
            assert est == 0
            assert ctx.top_k_local_maxima(mc, k).thresholds == etk, (i, k)


def test_selection_errors(ctx):
    mc = kb.MeanContrastCurve(np.array([1.0]), np.array([True]))
    with pytest.raises(ValueError):
        ctx.top_k_local_maxima(mc, 0)
    empty = kb.MeanContrastCurve(np.zeros(256), np.zeros(256, bool))
    with pytest.raises(kb.NoBoundaryError):
        ctx.top_k_local_maxima(empty, 1)
    with pytest.raises(kb.NoBoundaryError):
        ctx.optimal_threshold(kb.MeanContrastCurve(np.zeros(0), np.zeros(0, bool)))


def test_concurrent_callers_identical(ctx, orc):
    rng = np.random.default_rng(3131)
    im = rng.integers(0, 256, (40, 48), dtype=np.uint8)
    exp = orc.direct_curve(im)
    res = [None] * 8

    def run(i):
        res[i] = kb.fast_contrast_curve(im, 1 + i % 3)

    th = [threading.Thread(target=run, args=(i,)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in res:
        assert np.array_equal(c.contrast_sum, exp[0]) and np.array_equal(c.cardinality, exp[1])


def test_repeat_determinism_and_merge(ctx):
    im = synth.c1(device="cpu").numpy()
    first = kb.fast_contrast_curve(im)
    for _ in range(5):
        assert kb.fast_contrast_curve(im) == first
    parts = [kb.ContrastCurve(), first]
    assert kb.merge_accumulators(parts) == first
    with pytest.raises(ValueError):
        kb.merge_accumulators([])

"""Pins the CPU oracle (oracle/kohler_oracle.c) — runs without a GPU.

1. Hand-derived constants of the reference's own tests
   (proj/tests/test_contrast.cpp:32-123, test_threshold.cpp:50-183,
   acceptance.cpp:158-202).
2. Golden vectors produced by the reference library itself
   (tests/golden/*.npz, written by tests/golden/make_golden.py).
3. Algebraic identities and invariances (test_support.hpp:70-144).
"""
import numpy as np
import pytest

CHECKER = np.array([[0, 255], [255, 0]], np.uint8)
COLUMN_2_5 = np.array([[2], [5]], np.uint8)


def test_pair_contribution_hand_values(orc):
    s, c = orc.pair_contribution(7, 7)
    assert not s.any() and not c.any()
    s, c = orc.pair_contribution(2, 5)
    assert [int(c[t]) for t in range(256)] == [1 if 2 <= t <= 4 else 0 for t in range(256)]
    assert (int(s[2]), int(s[3]), int(s[4])) == (0, 1, 1) and int(s.sum()) == 2
    s, c = orc.pair_contribution(0, 255)
    assert int(s.sum()) == 16256
    assert [int(x) for x in c] == [1] * 255 + [0]


def test_pair_contribution_totals_quarter_square(orc):
    for lo in range(0, 256, 17):
        for hi in range(lo, 256, 13):
            s, c = orc.pair_contribution(lo, hi)
            d = hi - lo
            assert int(c.sum()) == d
            assert int(s.sum()) == d * d // 4


def test_hand_curves(orc):
    assert not any(a.any() for a in orc.direct_curve(np.full((2, 2), 100, np.uint8)))
    for fn in (orc.direct_curve, orc.fast_curve):
        s, c = fn(COLUMN_2_5)
        assert [int(x) for x in c[:6]] == [0, 0, 1, 1, 1, 0]
        assert [int(x) for x in s[2:5]] == [0, 1, 1]
        s, c = fn(CHECKER)
        for t in range(256):
            assert int(c[t]) == (4 if t <= 254 else 0)
            assert int(s[t]) == (4 * min(t, 255 - t) if t <= 254 else 0)
        assert int(s[127]) == 508
        assert not any(a.any() for a in fn(np.array([[42]], np.uint8)))


def test_oracle_matches_reference_golden_corpus(orc, corpus):
    imgs, z = corpus
    for i, im in enumerate(imgs):
        s, c = orc.fast_curve(im)
        assert np.array_equal(s, z["sums"][i]) and np.array_equal(c, z["cards"][i]), i
        v, d = orc.mean_contrast(s, c)
        assert np.array_equal(v, z["values"][i]) and np.array_equal(d, z["defined"][i]), i
        assert orc.optimal_threshold(v, d) == z["t0"][i], i
        st, tk = orc.top_k(v, d, 6)
        assert st == z["status"][i], i
        assert tk == [int(t) for t in z["topk"][i] if t >= 0], i


def test_direct_equals_fast_and_blocks(orc, corpus):
    imgs, _ = corpus
    for im in imgs[:60]:
        f = orc.fast_curve(im)
        d = orc.direct_curve(im)
        assert all(np.array_equal(a, b) for a, b in zip(f, d))
        for blocks in (2, 3, 8):
            b = orc.fast_curve_blocks(im, blocks)
            assert all(np.array_equal(a, bb) for a, bb in zip(f, b))


def test_identities_and_invariances(orc, corpus):
    imgs, _ = corpus
    for im in imgs:
        s, c = orc.fast_curve(im)
        tv, qs = orc.identities(im)
        assert int(c.sum()) == tv and int(s.sum()) == qs
        assert int(c[255]) == 0
        assert np.all(s <= c * np.uint64(127))
        assert np.all((c > 0) | (s == 0))
        for t in (im[:, ::-1], im[::-1, :], im.T, im[::-1, ::-1]):
            s2, c2 = orc.fast_curve(np.ascontiguousarray(t))
            assert np.array_equal(s, s2) and np.array_equal(c, c2)


def test_row_partials_merge(orc, corpus):
    imgs, _ = corpus
    for im in imgs[:40]:
        h = im.shape[0]
        full = orc.fast_curve(im)
        cuts = sorted(set([0, h, h // 3, h // 2, max(h - 1, 0)]))
        acc = [np.zeros(256, np.uint64), np.zeros(256, np.uint64)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            if a < b:
                s, c = orc.curve_rows(im, a, b)
                acc[0] += s
                acc[1] += c
        assert np.array_equal(acc[0], full[0]) and np.array_equal(acc[1], full[1])


def _synthetic(values):
    v = np.zeros(256)
    d = np.zeros(256, np.uint8)
    for t, x in enumerate(values):
        if x >= 0:
            v[t] = x
            d[t] = 1
    return v, d


def test_selection_hand_cases(orc):
    v, d = orc.mean_contrast(*orc.fast_curve(CHECKER))
    assert orc.optimal_threshold(v, d) == 127
    assert orc.top_k(v, d, 1) == (0, [127])
    v, d = orc.mean_contrast(*orc.fast_curve(COLUMN_2_5))
    assert orc.optimal_threshold(v, d) == 3
    assert list(d[:6]) == [0, 0, 1, 1, 1, 0] and list(v[2:5]) == [0.0, 1.0, 1.0]
    v, d = orc.mean_contrast(*orc.fast_curve(np.full((3, 3), 42, np.uint8)))
    assert orc.optimal_threshold(v, d) == -1
    assert orc.top_k(v, d, 1)[0] == 1
    v, d = _synthetic([t if t < 12 else 24 - t for t in range(30)])
    for k in (1, 3, 10):
        assert orc.top_k(v, d, k) == (0, [12])
    assert orc.top_k(*_synthetic([1, 5, 5, 9, 0]), 10) == (0, [3])
    vals = [-1.0] * 10
    vals[0], vals[4], vals[8] = 3.0, 7.0, 2.0
    assert orc.top_k(*_synthetic(vals), 5) == (0, [4])
    rk = _synthetic([0, 8, 0, 6, 0, 8, 0])
    assert orc.top_k(*rk, 1) == (0, [1])
    assert orc.top_k(*rk, 2) == (0, [1, 5])
    assert orc.top_k(*rk, 3) == (0, [1, 3, 5])
    assert orc.top_k(*rk, 9) == (0, [1, 3, 5])
    assert orc.top_k(*_synthetic([]), 1)[0] == 1
    assert orc.top_k(*_synthetic([1.0]), 0)[0] == 2


def test_selection_golden(orc, selection):
    z = selection
    for i in range(z["values"].shape[0]):
        v, d = z["values"][i], z["defined"][i]
        assert orc.optimal_threshold(v, d) == z["t0"][i]
        for k in range(1, 9):
            st, tk = orc.top_k(v, d, k)
            assert st == z["status"][i, k - 1]
            assert tk == [int(t) for t in z["topk"][i, k - 1] if t >= 0]


def test_luma_oracle_against_reference_read_pnm(orc):
    """Colour ingest: the oracle's luma601 restatement against the reference's
    own read_pnm decoding of P6 / P3 streams (tests/golden/luma.npz)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "luma.npz"))
    s = g["samples"]
    assert np.array_equal(orc.rgb_to_gray(s[None]), g["sample_gray"][None])
    assert np.array_equal(orc.rgb_to_gray(g["rgb"]), g["gray"])
    assert np.array_equal(orc.rgb_to_gray(g["rgb"][:5, :7]), g["gray_p3"])
    # the closed form (what the GPU kernel computes), on every sample
    s64 = s.astype(np.int64)
    t = 299 * s64[:, 0] + 587 * s64[:, 1] + 114 * s64[:, 2] + 500
    assert np.array_equal(np.minimum(t // 1000, 255).astype(np.uint8), g["sample_gray"])
    r = orc.analyze(g["gray"], 6)
    assert np.array_equal(r["sum"], g["sums"]) and np.array_equal(r["card"], g["cards"])
    assert r["t0"] == int(g["t0"]) and r["topk"] == list(g["topk"])

"""The oracle against the reference library compiled from /root/reference
(oracle/_ref/libkohler_ref.so) on fresh seeded inputs — CPU only.  Skipped
when oracle/_ref was not built (the reference tree is not on the GPU box;
the built .so travels with the repo snapshot)."""
import numpy as np


def test_oracle_equals_reference_random(orc, ref):
    rng = np.random.default_rng(20240811)
    for i in range(80):
        w, h = int(rng.integers(1, 80)), int(rng.integers(1, 60))
        kind = i % 4
        if kind == 0:
            im = rng.integers(0, 256, (h, w), dtype=np.uint8)
        elif kind == 1:
            im = np.where(rng.random((h, w)) < 0.5, 17, 200).astype(np.uint8)
        elif kind == 2:
            im = np.clip(rng.normal(128, 5, (h, w)), 0, 255).astype(np.uint8)
        else:
            im = np.full((h, w), 9, np.uint8)
        a = orc.analyze(im, 6)
        for workers in (1, 3):
            b = ref.analyze(im, 6, workers)
            for key in ("sum", "card", "values", "defined"):
                assert np.array_equal(a[key], b[key]), (i, key)
            assert a["t0"] == b["t0"] and a["topk"] == b["topk"] and a["status"] == b["status"]


def test_reference_direct_equals_oracle(orc, ref):
    rng = np.random.default_rng(7)
    for _ in range(10):
        im = rng.integers(0, 256, (int(rng.integers(1, 20)), int(rng.integers(1, 20))), dtype=np.uint8)
        a = orc.direct_curve(im)
        b = ref.direct_curve(im)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

"""Generate the golden fixtures from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built by
``make -C oracle``):

    python tests/golden/make_golden.py

Writes tests/golden/corpus.npz: a seeded corpus of small images (the four
pixel distributions of the reference's test generator — uniform, two-level,
constant, gradient — at sizes 1x1 .. 64x48, mirroring
proj/tests/acceptance.cpp:86-103 and test_support.hpp:20-68) with the curves,
mean curves, optimal thresholds and top-6 maxima the reference library
computes for them, and tests/golden/selection.npz: synthetic mean curves
(plateaus, undefined gaps, ties) with the reference's optimal_threshold and
top_k_local_maxima for k in 1..8, and tests/golden/luma.npz (colour
ingest): RGB samples / a seeded RGB image encoded as P6 and P3 streams and
decoded by the reference's read_pnm (proj/src/pnm.cpp:87-139, luma601 at
:63-68), plus the reference pipeline on the decoded image
(``python tests/golden/make_golden.py --luma-only`` rewrites only this file).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def small_image(rng: np.random.Generator, w: int, h: int, dist: str) -> np.ndarray:
    if dist == "uniform":
        return rng.integers(0, 256, (h, w), dtype=np.uint8)
    if dist == "two_level":
        a, b = rng.integers(0, 256, 2)
        return np.where(rng.random((h, w)) < 0.5, a, b).astype(np.uint8)
    if dist == "constant":
        return np.full((h, w), rng.integers(0, 256), np.uint8)
    ys, xs = np.mgrid[0:h, 0:w]
    return ((xs + ys) * 255 // max(w + h - 2, 1)).astype(np.uint8)


def corpus(seed: int = 0xC0FFEE, count: int = 160):
    rng = np.random.default_rng(seed)
    dists = ["uniform", "two_level", "constant", "gradient"]
    imgs = [small_image(rng, 1, 1, "uniform"), small_image(rng, 64, 48, "uniform"),
            small_image(rng, 1, 48, "gradient"), small_image(rng, 64, 1, "two_level"),
            small_image(rng, 2, 2, "constant"), small_image(rng, 64, 48, "gradient"),
            np.array([[2], [5]], np.uint8), np.array([[0, 255], [255, 0]], np.uint8),
            small_image(rng, 17, 3, "uniform"), small_image(rng, 33, 5, "uniform")]
    i = 0
    while len(imgs) < count:
        w = int(rng.integers(1, 65))
        h = int(rng.integers(1, 49))
        imgs.append(small_image(rng, w, h, dists[i % 4]))
        i += 1
    return imgs


def synthetic_curves(seed: int = 0x5E1EC7, count: int = 300):
    """Mean curves built to stress the selection rules: few distinct values
    (plateaus and equal-valued maxima), undefined gaps, all-undefined."""
    rng = np.random.default_rng(seed)
    vals, defs = [], []
    for i in range(count):
        n = 256
        kind = i % 5
        if kind == 0:
            v = rng.integers(0, 6, n).astype(np.float64)          # many ties / plateaus
        elif kind == 1:
            v = rng.random(n) * 100.0
        elif kind == 2:
            v = np.round(rng.random(n) * 10.0) / 4.0
        elif kind == 3:
            v = np.repeat(rng.integers(0, 4, n // 8), 8).astype(np.float64)
        else:
            v = np.sin(np.arange(n) * rng.random() * 0.3) * 50 + 60
        p_def = [1.0, 0.7, 0.4, 0.9, 0.05][i % 5]
        d = (rng.random(n) < p_def).astype(np.uint8)
        if i % 37 == 0:
            d[:] = 0
        v = np.where(d > 0, v, 0.0)
        vals.append(v)
        defs.append(d)
    return np.array(vals), np.array(defs)


def luma_golden(ref) -> None:
    rng = np.random.default_rng(0x601)
    # edge samples: every {0, 1, 127, 128, 254, 255}^3 triple, the greys, and
    # triples whose weighted sum ends in exactly 500 (round half up)
    levels = [0, 1, 127, 128, 254, 255]
    samples = [(r, g, b) for r in levels for g in levels for b in levels]
    samples += [(v, v, v) for v in range(256)]
    half = []
    for r in range(0, 256, 3):
        for g in range(0, 256, 5):
            for b in range(256):
                if (299 * r + 587 * g + 114 * b) % 1000 == 500:
                    half.append((r, g, b))
                    break
    samples += half
    samples += [tuple(int(c) for c in t) for t in rng.integers(0, 256, (4000, 3))]
    samples = np.array(samples, np.uint8)
    n = len(samples)
    p6 = b"P6\n%d 1\n255\n" % n + samples.tobytes()
    sample_gray = ref.read_pnm(p6)[0]
    img = rng.integers(0, 256, (40, 48, 3), dtype=np.uint8)
    img[10:30, 12:40] = (200, 40, 90)  # a region, so the curve has structure
    gray = ref.read_pnm(b"P6\n48 40\n255\n" + img.tobytes())
    small = img[:5, :7]
    p3 = ("P3\n7 5\n255\n" + " ".join(str(int(v)) for v in small.ravel()) + "\n").encode()
    gray_p3 = ref.read_pnm(p3)
    r = ref.analyze(gray, k=6, workers=2)
    np.savez_compressed(os.path.join(HERE, "luma.npz"), samples=samples, sample_gray=sample_gray,
                        rgb=img, gray=gray, gray_p3=gray_p3, sums=r["sum"], cards=r["card"],
                        t0=np.int32(r["t0"]), topk=np.array(r["topk"], np.int32))
    print(f"wrote {n} luma samples and a 48x40 RGB image (reference read_pnm)")


def main():
    ref = oracle.Reference()
    if "--luma-only" in sys.argv:
        luma_golden(ref)
        return
    luma_golden(ref)
    imgs = corpus()
    shapes = np.array([im.shape for im in imgs], np.int32)
    flat = np.concatenate([im.ravel() for im in imgs]).astype(np.uint8)
    sums, cards, values, defined, t0s, topk, status = [], [], [], [], [], [], []
    for im in imgs:
        r = ref.analyze(im, k=6, workers=3)
        sums.append(r["sum"])
        cards.append(r["card"])
        values.append(r["values"])
        defined.append(r["defined"])
        t0s.append(r["t0"])
        tk = np.full(6, -1, np.int32)
        tk[: len(r["topk"])] = r["topk"]
        topk.append(tk)
        status.append(r["status"])
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), shapes=shapes, pixels=flat,
                        sums=np.array(sums), cards=np.array(cards), values=np.array(values),
                        defined=np.array(defined), t0=np.array(t0s, np.int32),
                        topk=np.array(topk), status=np.array(status, np.int32))

    vals, defs = synthetic_curves()
    t0 = np.array([ref.optimal_threshold(v, d) for v, d in zip(vals, defs)], np.int32)
    tk = np.full((len(vals), 8, 8), -1, np.int32)
    st = np.zeros((len(vals), 8), np.int32)
    for i, (v, d) in enumerate(zip(vals, defs)):
        for k in range(1, 9):
            s, ts = ref.top_k(v, d, k)
            st[i, k - 1] = s
            tk[i, k - 1, : len(ts)] = ts
    np.savez_compressed(os.path.join(HERE, "selection.npz"), values=vals, defined=defs, t0=t0,
                        topk=tk, status=st)
    print(f"wrote {len(imgs)} corpus images and {len(vals)} selection curves "
          f"(reference kernel: {ref.active_kernel()})")


if __name__ == "__main__":
    main()

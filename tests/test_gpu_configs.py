"""The five BASELINE.json configurations at FULL size on the GPU, checked
against the reference library (oracle/_ref) where it finishes in seconds and
through size-independent properties everywhere: the total-variation and
quarter-square identities (proj/tests/test_support.hpp:70-102), curve
invariants, determinism, and the no-boundary case."""
import numpy as np
import pytest
import torch

from paper_1707_05062_b200 import synth

pytestmark = pytest.mark.gpu

K = 6


def run_batch(ctx, x, k=K):
    """x: (n, h, w) uint8 CUDA tensor -> dict of host numpy outputs."""
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


def identities(x, chunk=64):
    """Per-image Σ|Δ| and Σ⌊Δ²/4⌋ over right and down pairs (torch, int64)."""
    tv, qs = [], []
    for s0 in range(0, x.shape[0], chunk):
        a = x[s0:s0 + chunk].to(torch.int32)
        t = torch.zeros(a.shape[0], dtype=torch.int64, device=x.device)
        q = torch.zeros_like(t)
        for d in ((a[:, :, 1:] - a[:, :, :-1]).abs(), (a[:, 1:, :] - a[:, :-1, :]).abs()):
            t += d.sum(dim=(1, 2), dtype=torch.int64)
            q += (d * d // 4).sum(dim=(1, 2), dtype=torch.int64)
        tv.append(t)
        qs.append(q)
    return torch.cat(tv).cpu().numpy(), torch.cat(qs).cpu().numpy()


def check_invariants(r, tv, qs):
    s, c = r["sums"], r["cards"]
    assert np.array_equal(c.sum(axis=1, dtype=np.uint64), tv.astype(np.uint64))
    assert np.array_equal(s.sum(axis=1, dtype=np.uint64), qs.astype(np.uint64))
    assert not c[:, 255].any()
    assert np.all(s <= c * np.uint64(127))
    assert np.all((c > 0) | (s == 0))
    # double curve = IEEE division of the integers
    with np.errstate(invalid="ignore", divide="ignore"):
        v = np.where(c > 0, s.astype(np.float64) / np.maximum(c, 1).astype(np.float64), 0.0)
    assert np.array_equal(r["values"], v)


def check_against_reference(r, exp, idx=None):
    idx = range(exp["sums"].shape[0]) if idx is None else idx
    for j, i in enumerate(idx):
        assert np.array_equal(r["sums"][i], exp["sums"][j]), i
        assert np.array_equal(r["cards"][i], exp["cards"][j]), i
        assert int(r["t0"][i]) == int(exp["t0"][j]), i
        cnt = int(exp["topk_count"][j])
        assert int(r["topk_count"][i]) == cnt
        assert list(r["topk"][i, :cnt]) == list(exp["topk"][j, :cnt]), i


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_single_image_configs_vs_reference(ctx, ref, name):
    x = synth.generate(name, device="cpu")
    r = run_batch(ctx, x.cuda())
    exp = ref.analyze_batch(x.numpy(), K, workers=8, threads=1)
    check_against_reference(r, exp)
    check_invariants(r, *identities(x.cuda()))
    assert r["status"][0] == 0 and r["topk_count"][0] == K


def test_c4_uniform_268mpx_vs_reference(ctx, ref):
    x = synth.generate("C4", device="cpu")
    r = run_batch(ctx, x.cuda())
    import os
    exp = ref.analyze_batch(x.numpy(), K, workers=os.cpu_count() or 8, threads=1)
    check_against_reference(r, exp)
    check_invariants(r, *identities(x.cuda()))


def test_c3_video_batch(ctx, ref):
    """All 512 frames bit-exact against the reference (frame-parallel on all
    host cores, workers = 1 per frame; proj/src/bench.cpp:263-277 runs the
    same per-frame pipeline sequentially)."""
    import os
    x = synth.generate("C3", device="cuda")
    r = run_batch(ctx, x)
    check_invariants(r, *identities(x, chunk=8))
    exp = ref.analyze_batch(x.cpu().numpy(), K, workers=1, threads=os.cpu_count() or 8)
    check_against_reference(r, exp)
    r2 = run_batch(ctx, x)
    for key in r:
        assert np.array_equal(r[key], r2[key])


def test_c5_small_images_vs_reference(ctx, ref):
    x = synth.generate("C5", device="cuda")
    r = run_batch(ctx, x)
    check_invariants(r, *identities(x, chunk=4096))
    exp = ref.analyze_batch(x.cpu().numpy(), K, workers=1)
    check_against_reference(r, exp)
    fam_b = np.arange(x.shape[0]) % 4 == 1
    assert np.all(r["status"][fam_b] == 1) and np.all(r["t0"][fam_b] == -1)
    assert not r["cards"][fam_b].any()
    assert np.all(r["status"][~fam_b] == 0)


def host_result(r):
    return {"sums": r.sums, "cards": r.cards, "values": r.values, "t0": r.t0,
            "topk": r.topk, "topk_count": r.topk_count, "status": r.status}


def test_host_api_chunked_single_image_vs_reference(ctx, ref):
    """Host API on C2: the upload is cut into row bands whose launches
    accumulate into one image (only the last finishes) — bit-exact."""
    x = synth.generate("C2", device="cpu").numpy()
    r = host_result(ctx.analyze_batch(x, K))
    exp = ref.analyze_batch(x, K, workers=8, threads=1)
    check_against_reference(r, exp)


@pytest.mark.parametrize("hw", [(2001, 1771), (1, 5_000_000), (4_200_000, 1)])
def test_host_api_chunked_ragged_and_degenerate(ctx, ref, hw):
    """Ragged width, a 1-pixel-wide column and a 1-row image through the
    chunked host path (bands of one row, halo rows at every chunk edge)."""
    h, w = hw
    rng = np.random.default_rng(h * 7 + w)
    x = rng.integers(0, 256, size=(1, h, w), dtype=np.uint8)
    x[0, : h // 2] //= 3  # two regimes
    r = host_result(ctx.analyze_batch(x, K))
    exp = ref.analyze_batch(x, K, workers=8, threads=1)
    check_against_reference(r, exp)


def test_host_api_chunked_batch_vs_reference(ctx, ref):
    """Host API on 24 C3 frames: image-range chunks, each its own launch."""
    x = synth.generate("C3", device="cuda")[:24].cpu().numpy()
    r = host_result(ctx.analyze_batch(x, K))
    exp = ref.analyze_batch(x, K, workers=1)
    check_against_reference(r, exp)


@pytest.mark.parametrize("depth", [2, 3, 4])
def test_pipelined_back_to_back_calls(ref, depth):
    """Pipeline depth d (kohler_cuda_set_pipeline_depth): d consecutive
    accumulation launches run side by side (sharing one accumulator buffer:
    each flush waits for the previous finish_kernel).  Back-to-back calls on
    different images must give exactly the depth-1 results (and the
    reference's on the C2 image)."""
    from paper_1707_05062_b200 import Context
    x = synth.generate("C2", device="cuda")[0]
    imgs = [x, x.flip(0).contiguous(), x.flip(1).contiguous(), (255 - x).contiguous(),
            x[:, :4000].contiguous(), x[::2].contiguous(), x.t().contiguous()]
    c1 = Context(0)
    want = [run_batch(c1, im[None]) for im in imgs]
    cp = Context(0)
    cp.set_pipeline_depth(depth)
    outs = []
    for rep in range(2):
        for im in imgs:  # no synchronisation between the calls
            h, w = im.shape
            o = {"sums": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
                 "cards": torch.zeros((1, 256), dtype=torch.int64, device="cuda"),
                 "values": torch.zeros((1, 256), dtype=torch.float64, device="cuda"),
                 "defined": torch.zeros((1, 256), dtype=torch.uint8, device="cuda"),
                 "t0": torch.zeros(1, dtype=torch.int32, device="cuda"),
                 "topk": torch.zeros((1, K), dtype=torch.int32, device="cuda"),
                 "topk_count": torch.zeros(1, dtype=torch.int32, device="cuda"),
                 "status": torch.zeros(1, dtype=torch.int32, device="cuda")}
            cp.analyze_batch_device(im, w, h, w, w * h, 1, K, o)
            outs.append(o)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        e = want[i % len(imgs)]
        for key in ("sums", "cards", "values", "t0", "topk", "topk_count", "status"):
            got = o[key].cpu().numpy()
            if key in ("sums", "cards"):
                got = got.view(np.uint64)
            assert np.array_equal(got, e[key]), (i, key)
    exp = ref.analyze_batch(x.cpu().numpy()[None], K)
    check_against_reference(want[0], exp)
    with pytest.raises(ValueError):
        cp.set_pipeline_depth(5)


def test_streaming_submit_collect(ctx, ref):
    """kohler_cuda_submit / kohler_cuda_collect: two tickets in flight, results
    identical to the synchronous host API and to the reference; a third
    submit before collecting fails; batches and ragged widths."""
    x = synth.generate("C2", device="cpu")[0]
    imgs = [x, x.flip(0), 255 - x, x[:, :5000], x[:777, :1231]]
    pinned = [im.contiguous().pin_memory() for im in imgs]
    want = [ctx.analyze_batch(im.numpy(), k=K) for im in imgs]
    t_prev = ctx.submit(pinned[0], K)
    got = []
    for i in range(1, len(pinned)):
        t = ctx.submit(pinned[i], K)
        got.append(ctx.collect(t_prev))
        t_prev = t
    got.append(ctx.collect(t_prev))
    for g, e in zip(got, want):
        assert np.array_equal(g.sums, e.sums) and np.array_equal(g.cards, e.cards)
        assert np.array_equal(g.values, e.values)
        assert g.thresholds(0) == e.thresholds(0) and int(g.t0[0]) == int(e.t0[0])
    ex = ref.analyze(x.numpy(), k=K, workers=8)
    assert np.array_equal(got[0].sums[0], ex["sum"]) and got[0].thresholds(0) == ex["topk"]
    a = ctx.submit(pinned[0], K)
    b = ctx.submit(pinned[1], K)
    with pytest.raises(ValueError):
        ctx.submit(pinned[2], K)
    ctx.collect(a)
    ctx.collect(b)
    batch = synth.generate("C5", device="cpu", n=64)
    t = ctx.submit(batch.numpy(), K)
    r = ctx.collect(t)
    w5 = ctx.analyze_batch(batch.numpy(), k=K)
    assert np.array_equal(r.sums, w5.sums) and np.array_equal(r.status, w5.status)


def test_image_larger_than_4_gib(ctx):
    """A 65600 x 65536 image (4.3 GB, > 2^32 bytes): 64-bit addressing in the
    walk, the border pass and the band split; checked through the identities
    (card total = total variation, sum total = Σ⌊Δ²/4⌋) and the invariants."""
    h, w = 65600, 65536
    g = torch.Generator(device="cuda")
    g.manual_seed(0x4B)
    x = torch.randint(0, 256, (h, w), dtype=torch.uint8, device="cuda", generator=g)
    x[: h // 3] //= 5
    r = run_batch(ctx, x[None])
    tv = qs = 0
    for y0 in range(0, h, 2048):
        a = x[y0:min(y0 + 2049, h)].to(torch.int32)
        dx = (a[:min(2048, h - y0), 1:] - a[:min(2048, h - y0), :-1]).abs()
        dy = (a[1:] - a[:-1]).abs()
        for d in (dx, dy):
            tv += int(d.sum(dtype=torch.int64))
            qs += int((d * d // 4).sum(dtype=torch.int64))
        del a, dx, dy
    check_invariants(r, np.array([tv]), np.array([qs]))
    assert int(r["status"][0]) == 0

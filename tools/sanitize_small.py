"""Small-shape workload for compute-sanitizer (racecheck / synccheck /
memcheck / initcheck): K1 walk_kernel (depth 1 and 3, grey and RGB fused, an
unaligned row width through the staging path, a band partial), K5
twalk_kernel (a batch of 128^2 and 64^2 images), finish_kernel and the
selection kernels; every result is checked against the oracle so a run
under the sanitizer is also a parity run.

  compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1707_05062_b200 import Context, synth  # noqa: E402

K = 6


def run(ctx, x, depth=1, rgb=None):
    n, h, w = x.shape
    out = {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
           "values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
           "defined": torch.zeros((n, 256), dtype=torch.uint8, device="cuda"),
           "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "topk": torch.zeros((n, K), dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(n, dtype=torch.int32, device="cuda")}
    ctx.set_pipeline_depth(depth)
    if rgb is None:
        ctx.analyze_batch_device(x, w, h, w, w * h, n, K, out)
    else:
        ctx.analyze_rgb_batch_device(rgb, w, h, 3 * w, 3 * w * h, n, K, out)
    torch.cuda.synchronize()
    return out


def check(out, x, orc, what):
    xs = x.cpu().numpy()
    for i in range(xs.shape[0]):
        e = orc.analyze(xs[i], K)
        s = out["sums"][i].cpu().numpy().view(np.uint64)
        c = out["cards"][i].cpu().numpy().view(np.uint64)
        assert np.array_equal(s, e["sum"]) and np.array_equal(c, e["card"]), (what, i)
        assert int(out["t0"][i]) == e["t0"], (what, i)


def main():
    orc = oracle.Oracle()
    ctx = Context(0)
    g = torch.Generator(device="cpu")
    g.manual_seed(7)
    # K1: one image, depth 1 and 3 (three launches in flight), grey
    x = synth.c1(device="cpu", w=384, h=256)[None].cuda()
    for depth in (1, 3):
        for _ in range(3):
            o = run(ctx, x, depth)
        check(o, x, orc, f"K1 depth {depth}")
    # K1 ragged width (staging + byte-load path) and a multi-image batch
    xr = torch.randint(0, 256, (3, 97, 203), generator=g, dtype=torch.uint8).cuda()
    check(run(ctx, xr), xr, orc, "K1 ragged batch")
    # K1 over RGB (fused: w % 16 == 0) and the two-pass path (w % 16 != 0)
    for w in (256, 200):
        grey = synth.c1(device="cpu", w=w, h=128)
        rgb = torch.stack([grey, grey, grey], dim=-1)[None].contiguous().cuda()
        luma = torch.from_numpy(orc.rgb_to_gray(rgb[0].cpu().numpy()))[None].cuda()
        check(run(ctx, luma, 1, rgb=rgb), luma, orc, f"K1 RGB w={w}")
    # band partial (the multi-GPU row decomposition)
    h = 256
    s = torch.zeros(256, dtype=torch.int64, device="cuda")
    c = torch.zeros(256, dtype=torch.int64, device="cuda")
    img = x[0]
    ctx.band_curve_device(img[100:].contiguous(), img.shape[1], img.shape[1], h, 100, 180, s, c)
    torch.cuda.synchronize()
    es, ec = orc.curve_rows(img.cpu().numpy(), 100, 180)
    assert np.array_equal(s.cpu().numpy().view(np.uint64), es)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), ec)
    # K5: small images (C5 families at 128^2, then 64^2)
    x5 = synth.c5(device="cpu", n=64)
    check(run(ctx, x5.cuda()), x5, orc, "K5 128^2")
    x6 = torch.randint(0, 256, (48, 64, 64), generator=g, dtype=torch.uint8)
    check(run(ctx, x6.cuda()), x6, orc, "K5 64^2")
    # selection on device curves (select256_kernel) and on host curves (select_kernel)
    out = {"values": torch.zeros((4, 256), dtype=torch.float64, device="cuda"),
           "defined": torch.zeros((4, 256), dtype=torch.uint8, device="cuda"),
           "t0": torch.zeros(4, dtype=torch.int32, device="cuda"),
           "topk": torch.zeros((4, K), dtype=torch.int32, device="cuda"),
           "topk_count": torch.zeros(4, dtype=torch.int32, device="cuda"),
           "status": torch.zeros(4, dtype=torch.int32, device="cuda")}
    o = run(ctx, x5[:4].cuda())
    ctx.select_device(o["sums"], o["cards"], 4, 256, K, out)
    torch.cuda.synchronize()
    assert torch.equal(out["t0"], o["t0"])
    mc = ctx.select_host(o["sums"][0].cpu().numpy().view(np.uint64),
                         o["cards"][0].cpu().numpy().view(np.uint64))
    if mc.defined.any():
        assert ctx.optimal_threshold(mc) == int(o["t0"][0])
    print("sanitize_small: all kernels ran, results match the oracle")


if __name__ == "__main__":
    main()

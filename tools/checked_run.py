"""Run the kernels of the bounds-checked build (lib/libkohler_cuda_checked.so,
-DKOHLER_CHECKED: every shared-memory counter event inside the counter block,
every other shared access inside the CTA's window, every cp.async source
inside the input buffer; a violation traps) over the shapes and paths that
stress the address arithmetic, and compare every result with the oracle.
The stand-in for compute-sanitizer, which the GPU pool does not allow.

    KOHLER_CUDA_LIB=paper_1707_05062_b200/lib/libkohler_cuda_checked.so python tools/checked_run.py

Prints one line per case and "CHECKED OK <n>" at the end (exit 0), or the
first mismatch / CUDA error (exit 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1707_05062_b200 import Context, _lib, synth  # noqa: E402

K = 6


def out(n):
    return {"sums": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
            "cards": torch.zeros((n, 256), dtype=torch.int64, device="cuda"),
            "values": torch.zeros((n, 256), dtype=torch.float64, device="cuda"),
            "defined": torch.zeros((n, 256), dtype=torch.uint8, device="cuda"),
            "t0": torch.zeros(n, dtype=torch.int32, device="cuda"),
            "topk": torch.zeros((n, K), dtype=torch.int32, device="cuda"),
            "topk_count": torch.zeros(n, dtype=torch.int32, device="cuda"),
            "status": torch.zeros(n, dtype=torch.int32, device="cuda")}


def check(o, imgs, orc, name):
    for i, x in enumerate(imgs):
        e = orc.analyze(x, K)
        s = o["sums"][i].cpu().numpy().view(np.uint64)
        c = o["cards"][i].cpu().numpy().view(np.uint64)
        if not (np.array_equal(s, e["sum"]) and np.array_equal(c, e["card"])):
            raise SystemExit(f"MISMATCH {name} image {i}")
        if int(o["t0"][i]) != e["t0"] or int(o["status"][i]) != e["status"]:
            raise SystemExit(f"MISMATCH {name} image {i} (thresholds)")


def main():
    assert os.path.basename(_lib.LIB_PATH) == "libkohler_cuda_checked.so", _lib.LIB_PATH
    orc = oracle.Oracle()
    rng = np.random.default_rng(2024)
    ctx = Context(0)
    cases = 0

    def run(name, imgs, pitch_pad=0, depth=1, rgb=False):
        nonlocal cases
        n = len(imgs)
        h, w = imgs[0].shape
        pitch = w + pitch_pad
        buf = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")
        for i, x in enumerate(imgs):
            buf[i, :, :w] = torch.from_numpy(x).cuda()
        ctx.set_pipeline_depth(depth)
        o = out(n)
        ctx.analyze_batch_device(buf, w, h, pitch, pitch * h, n, K, o)
        torch.cuda.synchronize()
        check(o, imgs, orc, name)
        ctx.set_pipeline_depth(1)
        cases += 1
        print(f"ok {name}: {n} x {w}x{h}", flush=True)

    # K1 single images: cluster (small), ticket (mid), finish_kernel (large);
    # widths off the 16-pixel grid (ragged segments), 1-row and 1-column images
    for (w, h) in [(1, 1), (16, 1), (1, 40), (17, 3), (100, 37), (511, 513), (512, 512),
                   (1000, 700), (2049, 1500), (5184, 3456)]:
        x = rng.integers(0, 256, (h, w), dtype=np.uint8)
        run(f"single {w}x{h}", [x])
    run("single padded pitch", [rng.integers(0, 256, (300, 200), dtype=np.uint8)], pitch_pad=24)
    run("C1 depth 3", [synth.c1(device="cpu").numpy()], depth=3)
    run("C2 depth 3", [synth.generate("C2", device="cpu")[0].numpy()], depth=3)
    # K1 batches (several images per CTA, epochs) and K5 batches (small images)
    run("K1 batch 5 x 300x257", [rng.integers(0, 256, (257, 300), dtype=np.uint8) for _ in range(5)])
    run("K5 batch 64 x 128x128", [rng.integers(0, 256, (128, 128), dtype=np.uint8) for _ in range(64)])
    run("K5 batch 40 x 45x30", [rng.integers(0, 256, (30, 45), dtype=np.uint8) for _ in range(40)])
    run("K5 batch 24 x 200x64", [rng.integers(0, 256, (64, 200), dtype=np.uint8) for _ in range(24)])
    fam = [np.full((128, 128), 7, np.uint8),
           (np.indices((128, 128)).sum(0) % 2 * 255).astype(np.uint8),
           np.repeat(rng.choice([0, 128, 255], (128, 1)), 128, 1).astype(np.uint8),
           np.clip(rng.normal(60, 15, (128, 128)), 0, 255).astype(np.uint8)]
    run("K5 C5 families", fam * 8)
    # one C3 frame batch slice through K1 with many images per launch
    c3 = synth.generate("C3", device="cpu")[:8].numpy()
    run("C3 8 frames", list(c3))
    # host API: chunked uploads (band + halo launches of one image)
    big = rng.integers(0, 256, (2100, 2048), dtype=np.uint8)
    r = ctx.analyze_batch(big[None], k=K)
    e = orc.analyze(big, K)
    if not (np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"])):
        raise SystemExit("MISMATCH host chunked upload")
    cases += 1
    print("ok host chunked 2048x2100", flush=True)
    # colour ingest fused into K1 (RGB rows read by the walk)
    rgb = rng.integers(0, 256, (2, 96, 160, 3), dtype=np.uint8)
    rr = ctx.analyze_rgb_batch(rgb, k=K)
    for i in range(2):
        e = orc.analyze(orc.rgb_to_gray(rgb[i]), K)
        if not np.array_equal(rr.sums[i], e["sum"]):
            raise SystemExit("MISMATCH rgb")
    cases += 1
    print("ok rgb batch", flush=True)
    print(f"CHECKED OK {cases}")


def negative():
    """The checks fire: with KOHLER_CHECKED_INJECT=1 the checked build's K1
    clamps its walks one row past the buffer end (a deliberate off-by-one);
    the cp.async source check must trap (violation 3) before the bad read."""
    assert os.path.basename(_lib.LIB_PATH) == "libkohler_cuda_checked.so", _lib.LIB_PATH
    assert os.environ.get("KOHLER_CHECKED_INJECT") == "1"
    ctx = Context(0)
    w, h = 256, 64
    buf = torch.zeros((h, w), dtype=torch.uint8, device="cuda")
    ctx.analyze_batch_device(buf, w, h, w, w * h, 1, K, out(1))
    torch.cuda.synchronize()
    print("NO VIOLATION")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--negative":
        try:
            negative()
        except RuntimeError as exc:
            print(f"CUDA ERROR {exc}")
            sys.exit(1)
        sys.exit(0)
    try:
        main()
    except RuntimeError as exc:  # a trapped violation surfaces as a CUDA error
        print(f"CUDA ERROR {exc}")
        sys.exit(1)

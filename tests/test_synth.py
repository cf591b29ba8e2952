"""Synthetic config generators (CPU, reduced sizes): shapes, determinism and
the value properties BASELINE.json states for each config."""
import torch

from paper_1707_05062_b200 import synth


def test_c1_levels_and_determinism():
    a = synth.c1(device="cpu", w=128, h=96)
    b = synth.c1(device="cpu", w=128, h=96)
    assert a.dtype == torch.uint8 and a.shape == (96, 128)
    assert torch.equal(a, b)
    assert not torch.equal(a, synth.c1(seed=1, device="cpu", w=128, h=96))


def test_c2_shape_small():
    x = synth.c2(device="cpu", w=300, h=200, n_ellipses=5)
    assert x.shape == (200, 300)
    assert int(x.float().std()) > 0


def test_c3_drift_and_noise():
    x = synth.c3(device="cpu", n=3, w=64, h=40)
    assert x.shape == (3, 40, 64)
    assert not torch.equal(x[0], x[1])


def test_c4_uniform():
    x = synth.c4(device="cpu", w=256, h=256)
    assert int(x.min()) == 0 and int(x.max()) == 255


def test_c5_families():
    x = synth.c5(device="cpu", n=64, size=32, chunk=16)
    assert x.shape == (64, 32, 32)
    for i in range(64):
        im = x[i]
        vals = set(torch.unique(im).tolist())
        fam = i % 4
        if fam == 0:
            assert vals <= {0, 128, 255}
            assert torch.equal(im, im[:, :1].expand_as(im))  # horizontal stripes
        elif fam == 1:
            assert len(vals) == 1
        elif fam == 2:
            assert vals == {0, 255}
        else:
            assert len(vals) > 10


def test_full_config_table():
    assert synth.CONFIGS["C2"].pixels == 5184 * 3456
    assert synth.CONFIGS["C5"].pixels == 65536 * 128 * 128

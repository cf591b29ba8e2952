"""The multi-GPU C ABI (kohler_cuda_multi_*, include/kohler_cuda.h "device
groups"): one host thread, one context per device.  Only one GPU is visible
to the tests: a group of that one device runs the NCCL all-reduce path
(world 1), and KOHLER_MULTI_VIRTUAL=1 groups of 3-8 members on the same GPU
run the B-way row-block split in both merge forms -- peer mode (the members'
band kernels add straight into the first member's accumulator, one
finish_kernel behind their events) and per-member partial curves merged on
the host (the stand-in for the all-reduce).  The band partials of every split
are also checked in test_gpu_parity.py and the N > 1 host logic in
test_bands_gloo.py.  Results must equal the oracle's bit for bit (reference
fast.cpp:36-62 for any split)."""
import numpy as np
import pytest

import oracle
from paper_1707_05062_b200 import DeviceGroup, synth
from paper_1707_05062_b200._lib import KOHLER_INVALID_ARGUMENT

pytestmark = pytest.mark.gpu
K = 6


@pytest.fixture(scope="module")
def group():
    g = DeviceGroup([0])
    yield g
    g.close()


def test_group_uses_nccl(group):
    assert group.size() == 1
    assert group.uses_nccl()  # the all-reduce path runs even for one member
    assert not group.uses_peer()


@pytest.mark.parametrize("w,h", [(1, 1), (16, 1), (129, 7), (512, 512), (5184, 3456)])
def test_group_curve_and_analyze(group, w, h):
    orc = oracle.Oracle()
    if (w, h) == (5184, 3456):
        x = synth.generate("C2", device="cpu")[0].numpy()
    else:
        x = np.random.default_rng(w * 7 + h).integers(0, 256, (h, w), dtype=np.uint8)
    e = orc.analyze(x, K)
    c = group.curve(x)
    assert np.array_equal(c.contrast_sum, e["sum"]) and np.array_equal(c.cardinality, e["card"])
    r = group.analyze(x, K)
    assert np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"])
    assert np.array_equal(r.values[0].view(np.uint64), np.asarray(e["values"]).view(np.uint64))
    assert int(r.t0[0]) == e["t0"] and int(r.status[0]) == e["status"]
    assert r.thresholds(0) == e["topk"]


def test_group_no_boundary(group):
    r = group.analyze(np.full((40, 30), 9, np.uint8), K)
    assert int(r.status[0]) == 1 and int(r.t0[0]) == -1 and int(r.topk_count[0]) == 0
    assert not r.cards[0].any()


def test_group_batch_shards(group):
    orc = oracle.Oracle()
    rng = np.random.default_rng(3)
    xs = rng.integers(0, 256, (7, 33, 48), dtype=np.uint8)
    xs[4] = 200  # one boundary-free image inside a shard
    r = group.analyze_batch(xs, K)
    for i in range(xs.shape[0]):
        e = orc.analyze(xs[i], K)
        assert np.array_equal(r.sums[i], e["sum"]) and np.array_equal(r.cards[i], e["card"])
        assert int(r.t0[i]) == e["t0"] and int(r.status[i]) == e["status"]
        assert r.thresholds(i) == e["topk"]


def test_group_argument_errors():
    with pytest.raises(ValueError):
        DeviceGroup([0, 0])  # a device listed twice
    with pytest.raises(Exception):
        DeviceGroup([])
    g = DeviceGroup([0])
    with pytest.raises(ValueError):
        g.analyze(np.zeros((4, 4), np.uint8), 0)  # k < 1
    g.close()
    assert KOHLER_INVALID_ARGUMENT == 2


@pytest.mark.parametrize("peer", [True, False])
@pytest.mark.parametrize("members,w,h", [(3, 129, 7), (5, 64, 2), (8, 1, 3), (4, 5184, 3456), (7, 300, 301)])
def test_virtual_group_row_blocks(members, w, h, peer, monkeypatch):
    """KOHLER_MULTI_VIRTUAL=1: a group of several members on the one visible
    GPU.  Exercises the row-block split of a B-device group -- uneven blocks,
    more members than rows (empty bands), the halo rows -- against the oracle,
    in both merge forms: peer mode (every member's band kernel adds straight
    into the first member's accumulator, system-scope REDs, one finish_kernel
    behind the members' events; the members' kernels run concurrently on
    their own streams) and, with KOHLER_MULTI_NO_PEER=1, per-member partial
    curves merged on the host (the stand-in for the NCCL all-reduce)."""
    monkeypatch.setenv("KOHLER_MULTI_VIRTUAL", "1")
    if not peer:
        monkeypatch.setenv("KOHLER_MULTI_NO_PEER", "1")
    g = DeviceGroup([0] * members)
    assert g.size() == members and not g.uses_nccl() and g.uses_peer() == peer
    orc = oracle.Oracle()
    if (w, h) == (5184, 3456):
        x = synth.generate("C2", device="cpu")[0].numpy()
    else:
        x = np.random.default_rng(members * 1000 + w + h).integers(0, 256, (h, w), dtype=np.uint8)
    e = orc.analyze(x, K)
    for _ in range(2):  # twice: the shared accumulator must be clean again after a call
        c = g.curve(x)
        assert np.array_equal(c.contrast_sum, e["sum"]) and np.array_equal(c.cardinality, e["card"])
        r = g.analyze(x, K)
        assert np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"])
        assert int(r.t0[0]) == e["t0"] and r.thresholds(0) == e["topk"]
        assert np.array_equal(r.values[0].view(np.uint64), np.asarray(e["values"]).view(np.uint64))
    g.close()


def test_virtual_peer_group_mixed_calls(monkeypatch):
    """Peer mode across different images and a boundary-free one: the one
    accumulator is reused call after call."""
    monkeypatch.setenv("KOHLER_MULTI_VIRTUAL", "1")
    g = DeviceGroup([0] * 4)
    assert g.uses_peer()
    orc = oracle.Oracle()
    rng = np.random.default_rng(77)
    for w, h in [(640, 480), (33, 5), (2000, 37), (16, 16)]:
        x = rng.integers(0, 256, (h, w), dtype=np.uint8)
        e = orc.analyze(x, K)
        r = g.analyze(x, K)
        assert np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"])
        assert int(r.t0[0]) == e["t0"] and r.thresholds(0) == e["topk"]
    r = g.analyze(np.full((40, 30), 9, np.uint8), K)
    assert int(r.status[0]) == 1 and int(r.t0[0]) == -1 and not r.cards[0].any()
    x = rng.integers(0, 256, (100, 100), dtype=np.uint8)
    e = orc.analyze(x, K)
    c = g.curve(x)
    assert np.array_equal(c.contrast_sum, e["sum"]) and np.array_equal(c.cardinality, e["card"])
    g.close()

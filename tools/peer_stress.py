"""Stress of the device groups' peer mode on one GPU (KOHLER_MULTI_VIRTUAL=1):
240 random images (1..1200 x 1..2000) through groups of 2, 5 and 8 members whose
band kernels add into the first member's accumulator concurrently, every
result compared with the oracle.  python tools/peer_stress.py"""
import os, sys, numpy as np
os.environ["KOHLER_MULTI_VIRTUAL"] = "1"
sys.path.insert(0, os.getcwd())
import oracle
from paper_1707_05062_b200 import DeviceGroup
rng = np.random.default_rng(1)
orc = oracle.Oracle()
bad = 0
for members in (2, 5, 8):
    g = DeviceGroup([0] * members)
    assert g.uses_peer()
    for it in range(80):
        h, w = int(rng.integers(1, 1200)), int(rng.integers(1, 2000))
        x = rng.integers(0, 256, (h, w), dtype=np.uint8)
        e = orc.analyze(x, 6)
        r = g.analyze(x, 6)
        ok = np.array_equal(r.sums[0], e["sum"]) and np.array_equal(r.cards[0], e["card"]) and int(r.t0[0]) == e["t0"] and r.thresholds(0) == e["topk"]
        if not ok:
            bad += 1
            print("MISMATCH", members, it, h, w)
    g.close()
print("peer stress done, mismatches:", bad)

"""The reference's own acceptance runner (proj/tests/acceptance.cpp:408-454,
compiled unchanged by oracle/Makefile `acceptance`) relinked against the
drop-in libkohler_b200.so — INTEGRATION.md option A exercised for real:

* acceptance_gpu      : fast_contrast_curve on the GPU, everything else from
                        the reference sources (its direct.cpp is the oracle of
                        criterion 1);
* acceptance_gpu_full : every drop-in function on the GPU;
* acceptance_ref      : the unmodified reference (CPU), the comparison.

Criterion 8 runs the reference CLI (tools/kohler_main.cpp), which needs the
absent CLI11.hpp; it is pointed at /bin/false and is expected to fail in all
three builds.  Every other criterion must PASS (timing criteria 5-7 compare
the implementations on the same host, as the reference runs them), except
criterion 5 in the all-GPU build: it times fast against DIRECT, and there
the definition-level direct curve is a GPU kernel too (measured 8x, not the
>= 5x / >= 10x a CPU direct scan gives; with the reference's CPU direct.cpp,
acceptance_gpu, it passes)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
EXPECT_PASS = {1, 2, 3, 4, 5, 6, 7, 9, 10}


def run_acceptance(name):
    exe = os.path.join(REF, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    res = {}
    for line in out.stdout.splitlines():
        m = re.match(r"\[(PASS|FAIL)\]\s+(\d+)\.", line)
        if m:
            res[int(m.group(2))] = m.group(1) == "PASS"
    assert set(res) == set(range(1, 11)), out.stdout
    return res, out.stdout


def test_reference_acceptance_cpu():
    res, text = run_acceptance("acceptance_ref")
    assert {c for c, ok in res.items() if ok} == EXPECT_PASS, text


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["acceptance_gpu", "acceptance_gpu_full"])
def test_reference_acceptance_relinked_on_gpu(name):
    res, text = run_acceptance(name)
    print(text)
    want = EXPECT_PASS if name == "acceptance_gpu" else EXPECT_PASS - {5}
    assert {c for c, ok in res.items() if ok} >= want, text
    assert not res[8]  # the CLI is absent

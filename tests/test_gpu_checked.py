"""The bounds-checked build (lib/libkohler_cuda_checked.so, -DKOHLER_CHECKED:
shared-memory counter events inside the counter block, other shared
accesses inside the CTA's window, cp.async sources inside the input buffer;
a violation traps) over the shapes and paths that stress the address
arithmetic, every result compared with the oracle (tools/checked_run.py).
compute-sanitizer is not available on the GPU pool; this is its stand-in."""
import os
import subprocess
import sys

import pytest

from paper_1707_05062_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean():
    assert os.path.exists(_lib.CHECKED_LIB_PATH), "build with __graft_entry__.build()"
    env = dict(os.environ, KOHLER_CUDA_LIB=_lib.CHECKED_LIB_PATH)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py")],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "KOHLER_CHECKED violation" not in r.stdout + r.stderr, tail
    assert r.stdout.strip().splitlines()[-1].startswith("CHECKED OK"), tail


def test_checked_build_catches_an_out_of_bounds_source():
    """Negative control: KOHLER_CHECKED_INJECT=1 makes the checked K1 clamp
    its walks one row past the buffer end; the cp.async source check must
    trap (violation 3) instead of reading past it."""
    env = dict(os.environ, KOHLER_CUDA_LIB=_lib.CHECKED_LIB_PATH, KOHLER_CHECKED_INJECT="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py"), "--negative"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 1, out[-3000:]
    assert "KOHLER_CHECKED violation 3" in out, out[-3000:]

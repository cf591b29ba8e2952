"""The C++ drop-in (libkohler_b200.so) exercised from C++ through the
reference-compatible headers (tests/cpp/dropin_test.cpp), on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1707_05062_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle", "_build")


def build(out):
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src,
                    "-L", LIB, "-lkohler_b200", "-L", ORACLE, "-lkohler_oracle",
                    f"-Wl,-rpath,{LIB}:{ORACLE}", "-o", out], check=True)


def test_dropin_test_compiles(tmp_path):
    """Builds against the headers and both libraries (no GPU needed)."""
    import oracle
    oracle.build(ref=False)
    build(str(tmp_path / "dropin_test"))


@pytest.mark.gpu
def test_dropin_cpp_on_gpu(tmp_path):
    import oracle
    oracle.build(ref=False)
    exe = str(tmp_path / "dropin_test")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.startswith("PASS")


@pytest.mark.gpu
def test_dropin_cpp_on_a_device_group(tmp_path):
    """The same C++ checks with KOHLER_CUDA_DEVICES set: fast_contrast_curve
    runs through the device-group path (row band per device, NCCL all-reduce
    of the partials; here a group of the one visible GPU)."""
    import oracle
    oracle.build(ref=False)
    exe = str(tmp_path / "dropin_test")
    build(exe)
    env = dict(os.environ, KOHLER_CUDA_DEVICES="0")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    # (NCCL prints its version line at communicator creation)
    assert r.stdout.strip().splitlines()[-1].startswith("PASS")

"""The C ABI library loads and exports everything include/kohler_cuda.h
declares; the C++ drop-in exports the reference API.  No compute calls:
runs without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1707_05062_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kohler_cuda.h")).read()
    return sorted(set(re.findall(r"\b(kohler_cuda_\w+)\s*\(", src)))


def test_library_built_in_tree():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"
    assert os.path.exists(_lib.DROPIN_PATH)


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes binding"
    assert set(_lib.SIGNATURES) == set(syms)
    assert lib.kohler_cuda_abi_version() == 104


def test_dropin_exports_reference_api():
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", _lib.DROPIN_PATH],
                         capture_output=True, text=True, check=True).stdout
    for sig in ["kohler::fast_contrast_curve(kohler::GrayImage const&, unsigned int)",
                "kohler::direct_contrast_curve(kohler::GrayImage const&)",
                "kohler::mean_contrast(kohler::ContrastCurve const&)",
                "kohler::optimal_threshold(kohler::MeanContrastCurve const&)",
                "kohler::top_k_local_maxima(kohler::MeanContrastCurve const&, int)",
                "kohler::merge_accumulators(std::span<kohler::ContrastCurve const, 18446744073709551615ul>)",
                "kohler::pair_contribution(unsigned char, unsigned char, kohler::ContrastCurve&)",
                "kohler::classify(kohler::GrayImage const&, kohler::ThresholdSet const&)",
                "kohler::quantize(kohler::GrayImage const&, kohler::ThresholdSet const&)"]:
        assert sig in out, sig


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "ATOMS.POPC.INC.32" in sass      # conflict-free striped pair (midpoint) events
    assert "ATOMS.ADD" in sass              # packed pixel-keyed count / sign-sum words
    assert "VIADDMNMX.S16x2.RELU" in sass   # the per-pair sign step, two pairs per instruction
    assert "LDGSTS" in sass                 # cp.async row ring of the column walks


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.kohler_cuda_create(0, ctypes.byref(h))
    assert rc != _lib.KOHLER_OK
    assert _lib.last_error() != ""
    from paper_1707_05062_b200 import api
    with pytest.raises((RuntimeError, ValueError)):
        api.Context(0)

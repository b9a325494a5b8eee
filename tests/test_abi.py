"""The C-ABI library loads and exports every declared symbol (no GPU needed)."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2510_16172_b200 import _lib


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib._SIGS, f"{name} has no ctypes signature"
    assert lib.fp_version() == 1


def test_error_strings_and_argument_validation():
    lib = _lib.load()
    assert lib.fp_error_string(0) == b"ok"
    assert b"unsupported" in lib.fp_error_string(2)
    # validation happens before any CUDA call: safe without a GPU
    null = None
    assert lib.fp_solve_f32(null, null, null, null, null, -1, 2, 10, 1, *([null] * 8), null) == 1
    assert lib.fp_solve_f32(null, null, null, null, null, 4, 2, 0, 1, *([null] * 8), null) == 1
    assert lib.fp_solve_f32(null, null, null, null, null, 4, 99, 10, 1, *([null] * 8), null) == 2
    assert lib.fp_vjp_f32(*([null] * 7), 1.0, 7, 4, 2, *([null] * 6), null) == 4
    with pytest.raises(NotImplementedError):
        _lib.check(2, "x")
    with pytest.raises(ValueError):
        _lib.check(1, "x")


def test_sass_is_sm100a():
    """The shipped kernels are native sm_100a code (cuobjdump lists the arch)."""
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout

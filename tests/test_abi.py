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
    assert lib.fp_solve_f32(null, null, null, null, null, -1, 2, 10, 1, *([null] * 9), null) == 1
    assert lib.fp_solve_f32(null, null, null, null, null, 4, 2, 0, 1, *([null] * 9), null) == 1
    assert lib.fp_solve_f32(null, null, null, null, null, 4, 99, 10, 1, *([null] * 9), null) == 2
    fate = np.zeros(8, np.uint8)
    assert lib.fp_solve_f32(null, null, null, null, null, 4, 2, 10, 1, *([null] * 7), fate.ctypes.data,
                            null, null) == 1  # fates need the trace
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


def test_host_entry_precision_follows_the_arrays():
    """solve_with_gradients_host never downcasts float64 arrays: DOUBLE is
    inferred, fp64 output buffers are required (checked before any CUDA call)."""
    from paper_2510_16172_b200 import ShapeMismatch
    from paper_2510_16172_b200.solver import Precision, host_buffers, solve_with_gradients_host

    B, K = 4, 2
    out64 = host_buffers(B, K, pinned=False, precision=Precision.DOUBLE)
    assert out64["d_basis"].dtype == np.float64 and out64["status"].dtype == np.uint8
    assert host_buffers(B, K, pinned=False)["T"].dtype == np.float32
    f8 = np.zeros
    args = (f8((B, K, 3, 2)), f8((B, K, 3)), f8((B, 3)), f8((B, 3)))
    with pytest.raises(ShapeMismatch):  # float64 inputs with fp32 outputs
        solve_with_gradients_host(*args, out=host_buffers(B, K, pinned=False))
    lib = _lib.load()
    null = None
    for fn in (lib.fp_solve_vjp_host_f32, lib.fp_solve_vjp_host_f64):
        assert fn(*([null] * 5), -1, K, 20, 1, 1.0, 0, *([null] * 8), 0, 3) == 1
        assert fn(*([null] * 5), B, K, 20, 1, 1.0, 0, *([null] * 8), 0, 9) == 1  # depth > 8
        assert fn(*([null] * 5), 0, K, 20, 1, 1.0, 0, *([null] * 8), 0, 3) == 0  # empty batch
        # a NULL required input is rejected before any copy or launch (T0 may
        # be NULL: zero initialisation)
        assert fn(*([null] * 5), B, K, 20, 1, 1.0, 0, *([null] * 8), 0, 3) == 1
        buf = np.zeros(64)
        p = buf.ctypes.data
        for missing in range(4):
            ins = [p] * 4
            ins[missing] = null
            assert fn(*ins, null, B, K, 20, 1, 1.0, 0, *([null] * 8), 0, 3) == 1, missing
        assert fn(null, null, p, p, null, B, 0, 20, 1, 1.0, 0, *([null] * 8), 0, 9) == 1  # K = 0, depth
        assert fn(p, p, p, p, null, B, K, 20, 1, 1.0, 7, *([null] * 8), 0, 3) == 4  # bad mode


def test_enumerate_candidates_argument_checks():
    """Range and order validation happen on the host (no GPU needed)."""
    from paper_2510_16172_b200 import enumerate_candidates

    with pytest.raises(ValueError):
        enumerate_candidates(5, 4)
    with pytest.raises(ValueError):
        enumerate_candidates(5, 2, begin=0, end=5 * 4 + 1)
    with pytest.raises(ValueError):
        enumerate_candidates(5, 2, exclude_repeats=False, begin=3, end=2)


def test_host_submit_and_wait_argument_checks():
    lib = _lib.load()
    null = None
    # a submit needs somewhere to put its ticket; empty batches complete at once
    assert lib.fp_solve_vjp_host_submit_f32(*([null] * 5), 4, 2, 20, 1, 1.0, 0, *([null] * 8), 0, 3,
                                            null) == 1
    assert lib.fp_host_wait(0) == 0
    assert lib.fp_host_wait(1 << 40) == 1  # never issued
    assert lib.fp_host_wait(70 << 56 | 1) == 1  # no such device


def test_host_outputs_are_selectable():
    """host_buffers(outputs=...) allocates only the chosen results; the
    others are passed as NULL (neither computed into host memory nor copied)."""
    from paper_2510_16172_b200 import ShapeMismatch
    from paper_2510_16172_b200.solver import HOST_OUTPUTS, host_buffers, solve_with_gradients_host

    out = host_buffers(8, 3, pinned=False, outputs=("T", "length", "status"))
    assert sorted(out) == ["T", "length", "status"]
    assert set(host_buffers(8, 3, pinned=False)) == set(HOST_OUTPUTS)
    f4 = np.zeros
    args = (f4((8, 3, 3, 2), np.float32), f4((8, 3, 3), np.float32), f4((8, 3), np.float32),
            f4((8, 3), np.float32))
    with pytest.raises(ValueError):
        solve_with_gradients_host(*args, out={"bogus": np.zeros(8, np.float32)})
    with pytest.raises(ShapeMismatch):
        solve_with_gradients_host(*args, out={"T": np.zeros((8, 3, 3), np.float32)})

"""ctypes binding of the C ABI in include/fermat_b200.h.

The shared library is the product: there is no CPU fallback. If it is
missing, every entry point raises ExtensionMissing (build it with
``python -m paper_2510_16172_b200.build``).
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import FermatPathError

LIB_PATH = os.environ.get("FERMAT_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libfermat_b200.so")
HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "fermat_b200.h")

FP_OK = 0
FP_ERR_INVALID_ARGUMENT = 1
FP_ERR_UNSUPPORTED_ORDER = 2
FP_ERR_CUDA = 3
FP_ERR_UNSUPPORTED_MODE = 4
FP_MAX_ORDER = 64  # orders 9..64: warp-per-path solver (csrc/fp_wide.cu)

STATUS_DEGENERATE_ENTRY = 0x01
STATUS_ZERO_DIRECTION = 0x02
STATUS_NOT_STATIONARY = 0x04
STATUS_NONFINITE = 0x08
STATUS_DEGENERATE_FINAL = 0x10
STATUS_SINGULAR = 0x20
STATUS_OUT_OF_BOUNDS = 0x40
STATUS_SHORT_SEGMENT = 0x80
VIS_BLOCKED = 0x01      # fp_visibility_f64 flags
VIS_WRONG_SIDE = 0x02
STATUS_UNCONVERGED_MASK = (STATUS_DEGENERATE_ENTRY | STATUS_NOT_STATIONARY
                           | STATUS_NONFINITE | STATUS_DEGENERATE_FINAL)

FATE_CURVATURE_SKIP = 0x01  # trace_fate bits (per BFGS iteration)
FATE_NONFINITE_SKIP = 0x02
FATE_ZERO_DIRECTION = 0x04
FATE_ENTRY_CHECK = 0x08  # diagnostic: the H' magnitude bound was inconclusive, every entry checked

VJP_FULL = 0
VJP_ENVELOPE = 1
VJP_MIXED = 2


class ExtensionMissing(RuntimeError):
    """The CUDA library is not built (or cannot be loaded)."""


class CudaCallError(FermatPathError):
    """A C-ABI call returned an error code."""


_P = C.c_void_p
_I64 = C.c_int64
_I = C.c_int
_F = C.c_float
_D = C.c_double

_SIGS = {
    "fp_solve_f32": [_P] * 5 + [_I64, _I, _I, _I] + [_P] * 9 + [_P],
    "fp_solve_f64": [_P] * 5 + [_I64, _I, _I, _I] + [_P] * 9 + [_P],
    "fp_vjp_f32": [_P] * 7 + [_F, _I, _I64, _I] + [_P] * 6 + [_P],
    "fp_vjp_f64": [_P] * 7 + [_D, _I, _I64, _I] + [_P] * 6 + [_P],
    "fp_solve_vjp_f32": [_P] * 5 + [_I64, _I, _I, _I, _P, _F, _I] + [_P] * 8 + [_P],
    "fp_solve_vjp_f64": [_P] * 5 + [_I64, _I, _I, _I, _P, _D, _I] + [_P] * 8 + [_P],
    "fp_solve_vjp_host_f32": [_P] * 5 + [_I64, _I, _I, _I, _F, _I] + [_P] * 8 + [_I64, _I],
    "fp_solve_vjp_host_f64": [_P] * 5 + [_I64, _I, _I, _I, _D, _I] + [_P] * 8 + [_I64, _I],
    "fp_solve_vjp_host_submit_f32": [_P] * 5 + [_I64, _I, _I, _I, _F, _I] + [_P] * 8 + [_I64, _I, _P],
    "fp_solve_vjp_host_submit_f64": [_P] * 5 + [_I64, _I, _I, _I, _D, _I] + [_P] * 8 + [_I64, _I, _P],
    "fp_host_wait": [C.c_uint64],
    "fp_objective_f64": [_P] * 5 + [_I64, _I] + [_P] * 4 + [_P],
    "fp_line_search_f64": [_P] * 7 + [_I64, _I, _I] + [_P] * 2 + [_P],
    "fp_init_params_f64": [_P] * 4 + [_I64, _I, _P, _P],
    "fp_peak_ffma": [_I, _I, _P, _P],
    "fp_peak_ffma_reg": [_I, _I, _P, _P],
    "fp_gate_wait": [_P, _D, _P],
    "fp_enum_pattern_count": [_I, _I, _I, C.c_uint],
    "fp_enum_decode": [_P, _I, _P, _I, _I, _I, C.c_uint, _I64, _I64, _P, _P, _P],
    "fp_enum_trace_f32": [_P, _P, _P, _I, _P, _I, _P, _P, _I, _I, C.c_uint, _I64, _I64, _I, _I,
                          _P, _I64] + [_P] * 9 + [_P],
    "fp_vertex_chain_f32": [_P, _I, _P, _P, _P, _P],
    "fp_visibility_f64": [_P, _I, _P, _P, _P, _P, _P, _P, _P, _I, _I64, _I, _D, _P, _P, _P],
    "fp_newton_f32": [_P] * 5 + [_I64, _I, _I] + [_P] * 3 + [_P],
    "fp_newton_f64": [_P] * 5 + [_I64, _I, _I] + [_P] * 3 + [_P],
    "fp_image_method_f64": [_P] * 4 + [_I64, _I, _P, _P, _P],
    "fp_gd_f32": [_P] * 5 + [_I64, _I, _I, _P, _P, _P],
    "fp_gd_f64": [_P] * 5 + [_I64, _I, _I, _P, _P, _P],
    "fp_set_kernel_policy": [_I],
    "fp_launch_count": [],
    "fp_last_cuda_error": [],
    "fp_error_string": [_I],
    "fp_version": [],
}
_RESTYPES = {"fp_launch_count": C.c_uint64, "fp_error_string": C.c_char_p,
             "fp_enum_pattern_count": C.c_int64}

_lib = None


def declared_symbols() -> list[str]:
    """Function names declared in include/fermat_b200.h."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(fp_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load the library (once); raises ExtensionMissing if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} is not built; run `python -m paper_2510_16172_b200.build` "
            "(the solver has no CPU fallback)")
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - environment specific
        raise ExtensionMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, args in _SIGS.items():
        if os.environ.get("FERMAT_B200_LIB") and not hasattr(lib, name):
            continue  # an experimental library (A/B builds of older sources) may lack newer entries
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == FP_OK:
        return
    lib = load()
    msg = lib.fp_error_string(rc).decode()
    if rc == FP_ERR_UNSUPPORTED_ORDER:
        raise NotImplementedError(f"{what}: {msg} (max order {FP_MAX_ORDER})")
    if rc == FP_ERR_INVALID_ARGUMENT:
        raise ValueError(f"{what}: {msg}")
    raise CudaCallError(f"{what}: {msg} (code {rc})")


POLICY_AUTO = 0
POLICY_DENSE = 1
POLICY_AUTO_SERIAL = 2
POLICY_BUCKET = 3
POLICY_TILE = 4
TILE_MAX_ORDER = 5  # fp_abi.cu kAutoTileMaxOrder: orders with a host-sync-free dispatch


def set_kernel_policy(policy: str) -> None:
    """'auto' (kind-mask specialised kernels, default) or 'dense' (uniform 2K kernel)."""
    code = {"auto": POLICY_AUTO, "dense": POLICY_DENSE, "serial": POLICY_AUTO_SERIAL,
            "bucket": POLICY_BUCKET, "tile": POLICY_TILE}[policy]
    check(load().fp_set_kernel_policy(code), "fp_set_kernel_policy")


def launch_count() -> int:
    return int(load().fp_launch_count())

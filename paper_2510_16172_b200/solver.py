"""Batched Fermat path solve on the GPU — drop-in for fermatpath.solver.

Mirrors /root/reference/pkg/src/fermatpath/solver.py:33-252: the same
Precision / SolveOptions / SolveReport types, `init_params`,
`line_search_alpha`, `bfgs_solve`, `batch_solve` and the batched kernel
entry `_bfgs_kernel`, plus tensor-level entry points (`solve`,
`solve_with_gradients`) that keep everything in HBM. All arithmetic runs in
the sm_100a kernels of libfermat_b200.so (include/fermat_b200.h).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .batching import BatchScene, device, params_tensor, ptr, stack_params, stream_ptr, to_device
from .errors import DegenerateSegment, ShapeMismatch, ZeroDirection
from .geometry import PathSpec, check_params


class Precision(Enum):
    SINGLE = "single"
    DOUBLE = "double"

    @property
    def dtype(self):
        return np.float32 if self is Precision.SINGLE else np.float64


@dataclass(frozen=True)
class SolveOptions:
    iterations: int = 100
    fixed_point_iters: int = 1
    precision: Precision = Precision.DOUBLE
    record_trace: bool = False
    grad_tol: float | None = None  # scalar-mode early stop only (solver.py:48-49)

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.fixed_point_iters < 1:
            raise ValueError("fixed_point_iters must be >= 1")


@dataclass(frozen=True)
class SolveReport:
    solution: np.ndarray
    final_length: float
    final_grad_norm: float
    iterations: int
    trace: list | None = None


@dataclass
class SolveResult:
    """Device-resident outputs of one batched solve."""

    T: torch.Tensor            # (B, K, 2)
    g: torch.Tensor | None     # (B, K, 2) clamped-norm gradient at T
    points: torch.Tensor | None  # (B, K, 3)
    length: torch.Tensor | None  # (B,)
    status: torch.Tensor       # (B,) uint8, FP_STATUS_* bits
    trace_len: torch.Tensor | None = None    # (I, B)
    trace_gnorm: torch.Tensor | None = None  # (I, B)
    H: torch.Tensor | None = None            # (B, 2K, 2K)
    trace_fate: torch.Tensor | None = None   # (I, B) uint8 FATE_* bits of each BFGS update

    @property
    def converged(self) -> torch.Tensor:
        """Finite, non-degenerate and |g| < 1e-5 (1 + L) (implicit_diff.py:25,30-36)."""
        return (self.status & _lib.STATUS_UNCONVERGED_MASK) == 0


@dataclass
class SceneGradients:
    """Batched SceneGradient fields (objective.py:67-86), one row per path."""

    basis: torch.Tensor   # (B, K, 3, 2)
    anchor: torch.Tensor  # (B, K, 3)
    start: torch.Tensor   # (B, 3)
    end: torch.Tensor     # (B, 3)


_MODES = {"full": _lib.VJP_FULL, "envelope": _lib.VJP_ENVELOPE, "mixed": _lib.VJP_MIXED}


def _empty(shape, dt, dev):
    return torch.empty(shape, dtype=dt, device=dev)


def solve(scene: BatchScene, T0=None, opts: SolveOptions = SolveOptions(), *,
          return_state: bool = False, want_grad: bool = True, want_points: bool = True) -> SolveResult:
    """Fixed-iteration batch BFGS (solver._bfgs_kernel, solver.py:146-215) on the GPU."""
    lib = _lib.load()
    sc = scene.astype(opts.precision.dtype)
    B, K = sc.size, sc.n
    dt, dev = sc.basis.dtype, sc.basis.device
    T0 = torch.zeros(B, K, 2, dtype=dt, device=dev) if T0 is None else params_tensor(sc, T0)
    I = opts.iterations
    res = SolveResult(
        T=_empty((B, K, 2), dt, dev),
        g=_empty((B, K, 2), dt, dev) if want_grad else None,
        points=_empty((B, K, 3), dt, dev) if want_points else None,
        length=_empty((B,), dt, dev),
        status=_empty((B,), torch.uint8, dev),
        # order 0 runs no iterations: empty per-path traces (solver.py:160-164)
        trace_len=_empty((I if K else 0, B), dt, dev) if opts.record_trace else None,
        trace_gnorm=_empty((I if K else 0, B), dt, dev) if opts.record_trace else None,
        H=_empty((B, 2 * K, 2 * K), dt, dev) if return_state else None,
        trace_fate=_empty((I if K else 0, B), torch.uint8, dev) if opts.record_trace else None,
    )
    fn = lib.fp_solve_f32 if dt == torch.float32 else lib.fp_solve_f64
    rc = fn(ptr(sc.basis), ptr(sc.anchor), ptr(sc.start), ptr(sc.end), ptr(T0), B, K, I,
            opts.fixed_point_iters, ptr(res.T), ptr(res.g), ptr(res.points), ptr(res.length),
            ptr(res.status), ptr(res.trace_len), ptr(res.trace_gnorm), ptr(res.trace_fate), ptr(res.H),
            stream_ptr())
    _lib.check(rc, "fp_solve")
    if K == 0:
        res.T.zero_()
        if res.g is not None:
            res.g.zero_()
    return res


def solve_with_gradients(scene: BatchScene, T0=None, opts: SolveOptions = SolveOptions(
        precision=Precision.SINGLE), weight=1.0, mode: str = "full"):
    """Fused forward solve + implicit VJP of sum_b w_b L*_b (one kernel).

    fp32 or fp64 per `opts.precision`. Returns (SolveResult without g,
    SceneGradients). `weight` is a scalar or a (B,) tensor of cotangents on
    the optimal lengths. `mode` is "full" or "envelope".
    """
    single = opts.precision is Precision.SINGLE
    lib = _lib.load()
    sc = scene.astype(opts.precision.dtype)
    B, K = sc.size, sc.n
    dt, dev = (torch.float32 if single else torch.float64), sc.basis.device
    T0 = torch.zeros(B, K, 2, dtype=dt, device=dev) if T0 is None else params_tensor(sc, T0)
    wt = None
    scale = 1.0
    if isinstance(weight, torch.Tensor) and weight.dim() > 0:
        wt = to_device(weight, dt)
    else:
        scale = float(weight)
    res = SolveResult(T=_empty((B, K, 2), dt, dev), g=None, points=_empty((B, K, 3), dt, dev),
                      length=_empty((B,), dt, dev), status=_empty((B,), torch.uint8, dev))
    grads = SceneGradients(_empty((B, K, 3, 2), dt, dev), _empty((B, K, 3), dt, dev),
                           _empty((B, 3), dt, dev), _empty((B, 3), dt, dev))
    name = "fp_solve_vjp_f32" if single else "fp_solve_vjp_f64"
    rc = getattr(lib, name)(ptr(sc.basis), ptr(sc.anchor), ptr(sc.start), ptr(sc.end), ptr(T0),
                            B, K, opts.iterations, opts.fixed_point_iters, ptr(wt), scale,
                            _MODES[mode], ptr(res.T), ptr(res.points), ptr(res.length),
                            ptr(grads.basis), ptr(grads.anchor), ptr(grads.start),
                            ptr(grads.end), ptr(res.status), stream_ptr())
    _lib.check(rc, name)
    return res, grads


class HostJob:
    """A submitted host-buffer step (`submit_with_gradients_host`); `wait()`
    blocks until its outputs are in host memory and returns them."""

    def __init__(self, ticket: int, out: dict, keep: tuple):
        self.ticket, self.out, self._keep = ticket, out, keep  # keep inputs alive until waited

    def wait(self) -> dict:
        if self._keep is not None:
            _lib.check(_lib.load().fp_host_wait(self.ticket), "fp_host_wait")
            self._keep = None
        return self.out


def _host_call(submit: bool, basis, anchor, start, end, T0, iterations, fixed_point_iters, weight,
               mode, chunk, depth, out, precision):
    lib = _lib.load()
    if precision is None:
        precision = Precision.DOUBLE if np.asarray(basis).dtype == np.float64 else Precision.SINGLE
    ft = precision.dtype
    basis = np.ascontiguousarray(basis, ft)
    B, K = basis.shape[0], basis.shape[1]
    anchor = np.ascontiguousarray(anchor, ft)
    start = np.ascontiguousarray(start, ft)
    end = np.ascontiguousarray(end, ft)
    # T0 = None: zero initialisation on the device (no host-to-device copy)
    T0 = None if T0 is None else np.ascontiguousarray(T0, ft)
    if (anchor.shape != (B, K, 3) or start.shape != (B, 3) or end.shape != (B, 3)
            or (T0 is not None and T0.shape != (B, K, 2))):
        raise ShapeMismatch("host arrays must be basis (B,K,3,2), anchor (B,K,3), start/end (B,3), T0 (B,K,2)")
    if iterations < 1 or fixed_point_iters < 1:
        raise ValueError("iterations and fixed_point_iters must be >= 1")
    out = out if out is not None else host_buffers(B, K, pinned=False, precision=precision)
    unknown = set(out) - set(HOST_OUTPUTS)
    if unknown:
        raise ValueError(f"unknown outputs {sorted(unknown)}; choose from {HOST_OUTPUTS}")
    for k, v in out.items():
        want = np.uint8 if k == "status" else ft
        if v.dtype != want or not v.flags.c_contiguous or v.shape != _host_shape(k, B, K):
            raise ShapeMismatch(f"out[{k!r}] must be a C-contiguous {np.dtype(want).name} array "
                                f"of shape {_host_shape(k, B, K)}")
    # outputs absent from `out` are passed as NULL: neither computed nor copied
    P = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    O = lambda k: P(out.get(k))  # noqa: E731
    single = precision is Precision.SINGLE
    args = (P(basis), P(anchor), P(start), P(end), P(T0), B, K, iterations, fixed_point_iters,
            float(weight), _MODES[mode], O("T"), O("points"), O("length"), O("d_basis"),
            O("d_anchor"), O("d_start"), O("d_end"), O("status"), int(chunk), int(depth))
    if not submit:
        name = "fp_solve_vjp_host_f32" if single else "fp_solve_vjp_host_f64"
        _lib.check(getattr(lib, name)(*args), name)
        return out
    import ctypes

    ticket = ctypes.c_uint64(0)
    name = "fp_solve_vjp_host_submit_f32" if single else "fp_solve_vjp_host_submit_f64"
    _lib.check(getattr(lib, name)(*args, ctypes.addressof(ticket)), name)
    return HostJob(int(ticket.value), out, (basis, anchor, start, end, T0))


def solve_with_gradients_host(basis, anchor, start, end, T0=None, iterations: int = 20,
                              fixed_point_iters: int = 1, weight: float = 1.0, mode: str = "full",
                              chunk: int = 1 << 19, depth: int = 3, out=None,
                              precision: Precision | None = None):
    """solve_with_gradients for host (numpy) arrays in the reference layout.

    One call of fp_solve_vjp_host_f32 / _f64: the batch streams through the
    GPU in chunks (copy-in, compute and copy-out streams over a ring of
    `depth` device chunk slots), so both PCIe directions and compute overlap.
    `precision` defaults to the dtype of `basis` (float64 arrays run the fp64
    kernels, never a silent fp32 downcast). Pinned (page-locked) arrays
    transfer fastest: pass `out` from `host_buffers` to reuse pinned outputs.
    Returns a dict of numpy arrays: T, points, length, status, d_basis,
    d_anchor, d_start, d_end (the keys of `out` when given: a missing key is
    an output that is skipped). T0 = None is zero initialisation, done on
    the device.
    """
    return _host_call(False, basis, anchor, start, end, T0, iterations, fixed_point_iters, weight,
                      mode, chunk, depth, out, precision)


def submit_with_gradients_host(basis, anchor, start, end, T0=None, iterations: int = 20,
                               fixed_point_iters: int = 1, weight: float = 1.0, mode: str = "full",
                               chunk: int = 1 << 19, depth: int = 3, out=None,
                               precision: Precision | None = None) -> HostJob:
    """solve_with_gradients_host without the final wait: returns a HostJob.

    Consecutive submits (same order and chunk) chain through one ring of
    device chunk slots, so step i + 1's host-to-device copies overlap step
    i's device-to-host copies (fp_solve_vjp_host_submit_*). The input and
    output arrays must stay untouched until `job.wait()` returns; use one
    `out` set per step in flight.
    """
    return _host_call(True, basis, anchor, start, end, T0, iterations, fixed_point_iters, weight,
                      mode, chunk, depth, out, precision)


HOST_OUTPUTS = ("T", "points", "length", "status", "d_basis", "d_anchor", "d_start", "d_end")


def _host_shape(name: str, B: int, K: int) -> tuple:
    return {"T": (B, K, 2), "points": (B, K, 3), "length": (B,), "status": (B,),
            "d_basis": (B, K, 3, 2), "d_anchor": (B, K, 3), "d_start": (B, 3), "d_end": (B, 3)}[name]


def host_buffers(B: int, K: int, pinned: bool = True, precision: Precision = Precision.SINGLE,
                 outputs=HOST_OUTPUTS) -> dict:
    """Output arrays for solve_with_gradients_host (page-locked when pinned).

    `outputs` selects which results the call returns; the others are not
    computed into host memory and cost no device-to-host copy (e.g. leave
    out "points", which the reference derives on the host from T).
    """
    def mk(shape, dt):
        if pinned:
            return torch.empty(shape, dtype=dt, pin_memory=True).numpy()
        return np.empty(shape, dtype=torch.empty(0, dtype=dt).numpy().dtype)
    f = torch.float32 if precision is Precision.SINGLE else torch.float64
    return {k: mk(_host_shape(k, B, K), torch.uint8 if k == "status" else f) for k in outputs}


def init_params_batch(scene: BatchScene) -> torch.Tensor:
    """(B, K, 2) fp64 midpoint projections (solver.init_params, solver.py:67-81)."""
    lib = _lib.load()
    sc = scene.astype(np.float64)
    out = torch.zeros(sc.size, sc.n, 2, dtype=torch.float64, device=sc.basis.device)
    rc = lib.fp_init_params_f64(ptr(sc.basis), ptr(sc.anchor), ptr(sc.start), ptr(sc.end), sc.size,
                                sc.n, ptr(out), stream_ptr())
    _lib.check(rc, "fp_init_params_f64")
    return out


def init_params(spec: PathSpec) -> np.ndarray:
    """Deterministic initial guess (solver.py:67-81)."""
    if spec.n == 0:
        return np.zeros((0, 2))
    return init_params_batch(BatchScene.from_specs([spec]))[0].cpu().numpy()


def line_search_alpha(spec: PathSpec, T, P, alpha0: float = 0.0, k: int = 1) -> float:
    """Fixed-point step size after k iterations from alpha0 (solver.py:115-143)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    T = check_params(spec, T)
    P = check_params(spec, P)
    lib = _lib.load()
    sc = BatchScene.from_specs([spec]).astype(np.float64)
    dev = sc.basis.device
    Tt = to_device(T[None], torch.float64)
    Pt = to_device(P[None], torch.float64)
    a0 = torch.full((1,), float(alpha0), dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.uint8, device=dev)
    rc = lib.fp_line_search_f64(ptr(sc.basis), ptr(sc.anchor), ptr(sc.start), ptr(sc.end), ptr(Tt),
                                ptr(Pt), ptr(a0), 1, sc.n, k, ptr(out), ptr(st), stream_ptr())
    _lib.check(rc, "fp_line_search_f64")
    status = int(st.item())
    if status & _lib.STATUS_DEGENERATE_ENTRY and not status & _lib.STATUS_ZERO_DIRECTION:
        raise DegenerateSegment("step-size denominator segment collapsed")
    if status & _lib.STATUS_ZERO_DIRECTION:
        if status & _lib.STATUS_DEGENERATE_ENTRY:
            raise DegenerateSegment("coincident consecutive path points")
        raise ZeroDirection("direction moves no interaction point")
    return float(out.item())


def _traces_from(res: SolveResult, n_rows: int):
    if res.trace_len is None:
        return None
    L = res.trace_len.double().cpu().numpy()
    G = res.trace_gnorm.double().cpu().numpy()
    return [[(it, float(L[it, b]), float(G[it, b])) for it in range(L.shape[0])]
            for b in range(n_rows)]


def _raise_entry(res: SolveResult):
    if bool(((res.status & _lib.STATUS_DEGENERATE_ENTRY) != 0).any()):
        raise DegenerateSegment("coincident consecutive path points in batch")


def _bfgs_kernel(sc: BatchScene, T0, opts: SolveOptions, return_state: bool = False):
    """Drop-in for solver._bfgs_kernel (solver.py:146-215): numpy in/out.

    Returns (T, g, traces) or (T, g, traces, H) in the working dtype;
    raises DegenerateSegment when any entry segment is degenerate, like the
    reference's whole-batch check (solver.py:166).
    """
    if not isinstance(sc, BatchScene):
        sc = BatchScene(sc.basis, sc.anchor, sc.start, sc.end)
    res = solve(sc, T0, SolveOptions(opts.iterations, opts.fixed_point_iters, opts.precision,
                                     opts.record_trace), return_state=return_state,
                want_points=False)
    if sc.n > 0:
        _raise_entry(res)
    T = res.T.cpu().numpy()
    g = res.g.cpu().numpy()
    traces = _traces_from(res, sc.size)
    if return_state:
        return T, g, traces, res.H.cpu().numpy()
    return T, g, traces


def _reports(res: SolveResult, n_rows: int, iterations: int, traces) -> list[SolveReport]:
    T = res.T.cpu().numpy()
    L = res.length.cpu().numpy()
    G = np.linalg.norm(res.g.cpu().numpy().reshape(n_rows, -1), axis=1)
    return [SolveReport(solution=np.asarray(T[b], dtype=float), final_length=float(L[b]),
                        final_grad_norm=float(G[b]), iterations=iterations,
                        trace=traces[b] if traces is not None else None)
            for b in range(n_rows)]


def bfgs_solve(spec: PathSpec, T0, opts: SolveOptions = SolveOptions()) -> SolveReport:
    """Scalar solve = batch of one (solver.py:235-240); honours grad_tol."""
    T0 = check_params(spec, T0)
    sc = BatchScene.from_specs([spec])
    if opts.grad_tol is None:
        res = solve(sc, T0[None], opts)
        if spec.n > 0:
            _raise_entry(res)
        return _reports(res, 1, opts.iterations, _traces_from(res, 1))[0]
    # Scalar early stop (solver.py:208-211): the run is deterministic, so the
    # state at the first iteration meeting the test is a shorter fixed run.
    probe = solve(sc, T0[None], SolveOptions(opts.iterations, opts.fixed_point_iters,
                                             opts.precision, True))
    if spec.n > 0:
        _raise_entry(probe)
    L = probe.trace_len[:, 0].double().cpu().numpy()
    G = probe.trace_gnorm[:, 0].double().cpu().numpy()
    hit = np.nonzero(G < opts.grad_tol * (1.0 + L))[0]
    stop = int(hit[0]) + 1 if hit.size else opts.iterations
    res = solve(sc, T0[None], SolveOptions(stop, opts.fixed_point_iters, opts.precision,
                                           opts.record_trace))
    return _reports(res, 1, opts.iterations, _traces_from(res, 1))[0]


def batch_solve(specs: Sequence[PathSpec], T0s, opts: SolveOptions = SolveOptions()) -> list[SolveReport]:
    """Uniform-schedule batch solve (solver.py:243-252)."""
    if opts.grad_tol is not None:
        raise ValueError("grad_tol is a scalar-mode option; batches run fixed iterations")
    sc = BatchScene.from_specs(specs)
    T0 = stack_params(specs, T0s)
    res = solve(sc, T0, opts)
    if sc.n > 0:
        _raise_entry(res)
    return _reports(res, sc.size, opts.iterations, _traces_from(res, sc.size))

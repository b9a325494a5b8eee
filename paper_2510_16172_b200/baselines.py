"""Comparison solvers on the GPU — drop-in for the reference's fermatpath.baselines.

Mirrors /root/reference/pkg/src/fermatpath/baselines.py: the exact image
method (baselines.py:48-80) and the masked damped Newton solver
(baselines.py:152-201) — config 1's comparator — run as sm_100a kernels
(csrc/fp_baselines.cu) behind fp_image_method_f64 / fp_newton_f32/f64.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .batching import BatchScene, params_tensor, ptr, stream_ptr
from .errors import NoIntersection, NotAllPlanes
from .geometry import PathSpec, SurfaceKind, check_params
from .solver import Precision, SolveOptions, SolveReport


def image_points_batch(sc: BatchScene) -> torch.Tensor:
    """(B, K, 3) exact reflection points for all-plane scenes (baselines.py:48-71)."""
    lib = _lib.load()
    s64 = sc.astype(np.float64)
    B, K = s64.size, s64.n
    pts = torch.empty(B, K, 3, dtype=torch.float64, device=s64.basis.device)
    st = torch.empty(B, dtype=torch.uint8, device=s64.basis.device)
    rc = lib.fp_image_method_f64(ptr(s64.basis), ptr(s64.anchor), ptr(s64.start), ptr(s64.end), B, K,
                                 ptr(pts), ptr(st), stream_ptr())
    _lib.check(rc, "fp_image_method_f64")
    if B and K and bool((st != 0).any()):
        raise NoIntersection("mirrored sight line parallel to its plane")
    return pts


def image_method(spec: PathSpec) -> np.ndarray:
    """Exact reflection points (n, 3) via successive mirroring (baselines.py:74-80)."""
    if any(s.kind is not SurfaceKind.PLANE for s in spec.surfaces):
        raise NotAllPlanes("image method handles planar reflections only")
    if spec.n == 0:
        return np.zeros((0, 3))
    return image_points_batch(BatchScene.from_specs([spec]))[0].cpu().numpy()


def newton_batch(sc: BatchScene, T0, opts: SolveOptions = SolveOptions(), trace: bool = False):
    """Masked damped Newton with step halving (baselines._newton_kernel, baselines.py:152-193).

    Returns (T, g[, trace_gnorm (I, B)]) as device tensors.
    """
    lib = _lib.load()
    s = sc.astype(opts.precision.dtype)
    B, K = s.size, s.n
    dt, dev = s.basis.dtype, s.basis.device
    T0 = torch.zeros(B, K, 2, dtype=dt, device=dev) if T0 is None else params_tensor(s, T0)
    if K == 0:
        out = (T0.clone(), torch.zeros_like(T0))
        return out + ((torch.zeros(opts.iterations, B, dtype=dt, device=dev),) if trace else ())
    T = torch.empty_like(T0)
    g = torch.empty_like(T0)
    tg = torch.empty(opts.iterations, B, dtype=dt, device=dev) if trace else None
    fn = lib.fp_newton_f32 if dt == torch.float32 else lib.fp_newton_f64
    rc = fn(ptr(s.basis), ptr(s.anchor), ptr(s.start), ptr(s.end), ptr(T0), B, K, opts.iterations,
            ptr(T), ptr(g), ptr(tg), stream_ptr())
    _lib.check(rc, "fp_newton")
    return (T, g, tg) if trace else (T, g)


def newton_solve(spec: PathSpec, T0, opts: SolveOptions = SolveOptions()) -> SolveReport:
    """Damped Newton on active coordinates with step halving (baselines.py:196-201)."""
    T0 = check_params(spec, T0)
    sc = BatchScene.from_specs([spec])
    T, g = newton_batch(sc, T0[None], opts)
    from .batching import objective_batch

    L = float(objective_batch(sc.astype(opts.precision.dtype), T)[0].item())
    if opts.precision is Precision.SINGLE:
        L = float(np.float32(L))
    return SolveReport(solution=T[0].double().cpu().numpy(), final_length=L,
                       final_grad_norm=float(np.linalg.norm(g[0].cpu().numpy())),
                       iterations=opts.iterations)


def gd_batch(sc: BatchScene, T0, opts: SolveOptions = SolveOptions()):
    """Fixed-step gradient descent (baselines._gd_kernel, baselines.py:87-101) -> (T, g)."""
    lib = _lib.load()
    s = sc.astype(opts.precision.dtype)
    B, K = s.size, s.n
    dt, dev = s.basis.dtype, s.basis.device
    T0 = torch.zeros(B, K, 2, dtype=dt, device=dev) if T0 is None else params_tensor(s, T0)
    if K == 0:
        return T0.clone(), torch.zeros_like(T0)
    T = torch.empty_like(T0)
    g = torch.empty_like(T0)
    fn = lib.fp_gd_f32 if dt == torch.float32 else lib.fp_gd_f64
    rc = fn(ptr(s.basis), ptr(s.anchor), ptr(s.start), ptr(s.end), ptr(T0), B, K, opts.iterations,
            ptr(T), ptr(g), stream_ptr())
    _lib.check(rc, "fp_gd")
    return T, g


def gradient_descent(spec: PathSpec, T0, opts: SolveOptions = SolveOptions()) -> SolveReport:
    """Fixed-step gradient descent baseline (baselines.py:104-111)."""
    T0 = check_params(spec, T0)
    sc = BatchScene.from_specs([spec])
    T, g = gd_batch(sc, T0[None], opts)
    from .batching import objective_batch

    L = float(objective_batch(sc, T.double())[0].item())
    if opts.precision is Precision.SINGLE:
        L = float(np.float32(L))
    return SolveReport(solution=T[0].double().cpu().numpy(), final_length=L,
                       final_grad_norm=float(np.linalg.norm(g[0].cpu().numpy())),
                       iterations=opts.iterations)


# High-precision reference (baselines.py:204-249)
REFERENCE_GRAD_TOL = 1e-12
REFERENCE_BFGS_ITERS = 1000
REFERENCE_FP_ITERS = 64
REFERENCE_POLISH_ITERS = 64


def _converged(sc64: BatchScene, T: torch.Tensor) -> torch.Tensor:
    """|g| < 1e-12 (1 + L) with clamped-norm g (baselines.py:236-240)."""
    from .batching import objective_batch

    L, g, _, _ = objective_batch(sc64, T)
    return torch.linalg.vector_norm(g.reshape(len(L), -1), dim=1) < REFERENCE_GRAD_TOL * (1.0 + L)


def reference_solve_batch(specs, T0s=None):
    """Ground truth: 1000 fp64 BFGS iterations (64 fixed-point steps) from the
    midpoint projection, then up to 64 single Newton steps on the paths still
    above |g| < 1e-12 (1 + L) (baselines.py:208-233). Returns (T numpy (B,n,2),
    converged numpy (B,))."""
    from .batching import stack_params
    from .solver import init_params_batch, solve

    sc = BatchScene.from_specs(specs).astype(np.float64)
    T0 = init_params_batch(sc) if T0s is None else params_tensor(sc, stack_params(specs, T0s))
    if sc.n == 0:
        return T0.cpu().numpy(), np.ones(sc.size, dtype=bool)
    res = solve(sc, T0, SolveOptions(REFERENCE_BFGS_ITERS, REFERENCE_FP_ITERS, Precision.DOUBLE),
                want_points=False)
    T = res.T
    conv = _converged(sc, T)
    polish = SolveOptions(iterations=1, precision=Precision.DOUBLE)
    for _ in range(REFERENCE_POLISH_ITERS):
        todo = torch.nonzero(~conv).flatten()
        if todo.numel() == 0:
            break
        sub = BatchScene(sc.basis[todo], sc.anchor[todo], sc.start[todo], sc.end[todo])
        Tn, _ = newton_batch(sub, T[todo], polish)
        T = T.clone()
        T[todo] = Tn
        conv = _converged(sc, T)
    return T.cpu().numpy(), conv.cpu().numpy()


def reference_solve(spec: PathSpec, T0=None) -> np.ndarray:
    """High-precision parameters for one path; NoConvergence on failure (baselines.py:243-249)."""
    from .errors import NoConvergence

    T, conv = reference_solve_batch([spec], None if T0 is None else [check_params(spec, T0)])
    if not conv[0]:
        raise NoConvergence("reference solver missed its gradient tolerance")
    return T[0]

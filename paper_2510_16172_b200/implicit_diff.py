"""Scene-parameter gradients by implicit differentiation, on the GPU.

Drop-in for /root/reference/pkg/src/fermatpath/implicit_diff.py:25-106 plus
the batched forms the reference lacks. One kernel per batch assembles the
exact block-tridiagonal Hessian at T* (objective.py:48-64), restricts it to
the active coordinates, solves it by block elimination in registers (with the
reference's Tikhonov retry, implicit_diff.py:55-71) and contracts the
solution with the mixed derivative (objective.py:101-135).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .batching import BatchScene, params_tensor, ptr, stream_ptr, to_device
from .errors import DegenerateSegment, NotStationary, SingularSystem
from .geometry import PathSpec, check_params
from .objective import SceneGradient
from .solver import SceneGradients

STATIONARITY_TOL = 1e-5  # implicit_diff.py:25
TIKHONOV_SCALE = 1e-12   # implicit_diff.py:26
RESIDUAL_TOL = 1e-8      # implicit_diff.py:27 (fp64 LAPACK residual)

_MODES = {"full": _lib.VJP_FULL, "envelope": _lib.VJP_ENVELOPE, "mixed": _lib.VJP_MIXED}


def vjp_batch(scene: BatchScene, T, v_T=None, w_L=None, mode: str = "full", return_u: bool = False):
    """Batched VJP at the (stationary) parameters T.

    mode "full":     w_L (dL/dtheta + vjp_solution(grad)) + vjp_solution(v_T)
    mode "envelope": w_L dL/dtheta + vjp_solution(v_T)
    mode "mixed":    w_L dL/dtheta + param_vjp(T, v_T)   (no solve, no gate)
    w_L is None (0), a scalar, or a (B,) tensor. Returns (SceneGradients,
    status (B,) uint8, u (B,K,2) or None).
    """
    lib = _lib.load()
    sc = scene
    dt = sc.basis.dtype
    B, K = sc.size, sc.n
    dev = sc.basis.device
    T = params_tensor(sc, T)
    vt = None if v_T is None else params_tensor(sc, v_T)
    wt, scale = None, 0.0
    if isinstance(w_L, torch.Tensor) and w_L.dim() > 0:
        wt = to_device(w_L, dt)
    elif isinstance(w_L, np.ndarray) and w_L.ndim > 0:
        wt = to_device(w_L, dt)
    elif w_L is not None:
        scale = float(w_L)
    out = SceneGradients(torch.empty(B, K, 3, 2, dtype=dt, device=dev),
                         torch.empty(B, K, 3, dtype=dt, device=dev),
                         torch.empty(B, 3, dtype=dt, device=dev),
                         torch.empty(B, 3, dtype=dt, device=dev))
    u = torch.empty(B, K, 2, dtype=dt, device=dev) if return_u else None
    st = torch.empty(B, dtype=torch.uint8, device=dev)
    fn = lib.fp_vjp_f32 if dt == torch.float32 else lib.fp_vjp_f64
    rc = fn(ptr(sc.basis), ptr(sc.anchor), ptr(sc.start), ptr(sc.end), ptr(T), ptr(vt), ptr(wt),
            scale, _MODES[mode], B, K, ptr(out.basis), ptr(out.anchor), ptr(out.start), ptr(out.end),
            ptr(u), ptr(st), stream_ptr())
    _lib.check(rc, "fp_vjp")
    return out, st, u


def _one(spec: PathSpec, Tstar, v=None, w_L=None, mode="full", gate=True, want_u=False):
    Tstar = check_params(spec, Tstar)
    sc = BatchScene.from_specs([spec]).astype(np.float64)
    vv = None if v is None else check_params(spec, v)[None]
    grads, st, u = vjp_batch(sc, Tstar[None], vv, w_L, mode, return_u=want_u)
    status = int(st.item())
    if status & _lib.STATUS_DEGENERATE_FINAL:
        raise DegenerateSegment("consecutive path points (nearly) coincide")
    if gate and status & _lib.STATUS_NOT_STATIONARY:
        raise NotStationary("gradient norm exceeds the stationarity gate")
    if status & _lib.STATUS_SINGULAR:
        raise SingularSystem("active Hessian singular even with Tikhonov")
    sg = SceneGradient(grads.basis[0].cpu().numpy(), grads.anchor[0].cpu().numpy(),
                       grads.start[0].cpu().numpy(), grads.end[0].cpu().numpy())
    return sg, (u[0].cpu().numpy() if want_u else None)


def solve_stationary_system(spec: PathSpec, Tstar, v) -> np.ndarray:
    """Solve H u = -v on active coordinates; inert entries are zero (implicit_diff.py:39-52)."""
    if spec.n == 0:
        check_params(spec, Tstar)
        return np.zeros((0, 2))
    _, u = _one(spec, Tstar, v, None, "envelope", gate=True, want_u=True)
    return u


def vjp_solution(spec: PathSpec, Tstar, v) -> SceneGradient:
    """v^T dT*/dtheta (implicit_diff.py:74-77)."""
    sg, _ = _one(spec, Tstar, v, None, "envelope", gate=True)
    return sg


def grad_length_wrt_params(spec: PathSpec, Tstar, debug_check: bool = False) -> SceneGradient:
    """Total derivative of the optimal length (implicit_diff.py:80-106)."""
    partial, _ = _one(spec, Tstar, None, 1.0, "envelope", gate=True)
    if debug_check:
        full, _ = _one(spec, Tstar, None, 1.0, "full", gate=True)
        gap = np.linalg.norm(full.flat() - partial.flat())
        if gap > 1e-6 * (1.0 + partial.norm()):
            raise AssertionError(f"envelope cross-check failed: |full - partial| = {gap:.3e}")
    return partial


def full_length_gradient(spec: PathSpec, Tstar) -> SceneGradient:
    """partial + vjp_solution(grad): the chain-rule total derivative (implicit_diff.py:92-100)."""
    sg, _ = _one(spec, Tstar, None, 1.0, "full", gate=True)
    return sg

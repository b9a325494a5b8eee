"""Path-length objective and its derivatives — drop-in for fermatpath.objective.

Mirrors /root/reference/pkg/src/fermatpath/objective.py:20-135. The scalar
functions are batches of one through the fp64 kernels: `path_length`,
`gradient`, `hessian` use fp_objective_f64; `length_param_gradient` and
`param_vjp` use the VJP kernel in its "mixed" mode (no stationarity solve).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DegenerateSegment
from .geometry import PathSpec, check_params


def seg_epsilon(spec: PathSpec) -> float:
    """Segment floor 1e-12 (1 + |end - start|) (objective.py:20-22)."""
    return 1e-12 * (1.0 + spec.scene_scale)


@dataclass(frozen=True)
class SceneGradient:
    """Derivatives of a scalar w.r.t. every scene parameter (objective.py:67-86)."""

    basis: np.ndarray   # (n, 3, 2)
    anchor: np.ndarray  # (n, 3)
    start: np.ndarray   # (3,)
    end: np.ndarray     # (3,)

    def flat(self) -> np.ndarray:
        return np.concatenate([np.ravel(self.basis), np.ravel(self.anchor), self.start, self.end])

    def norm(self) -> float:
        return float(np.linalg.norm(self.flat()))

    @classmethod
    def zeros(cls, n: int) -> "SceneGradient":
        return cls(np.zeros((n, 3, 2)), np.zeros((n, 3)), np.zeros(3), np.zeros(3))


def _objective(spec: PathSpec, T, hessian: bool):
    from .batching import BatchScene, objective_batch

    T = check_params(spec, T)
    sc = BatchScene.from_specs([spec])
    L, g, H, st = objective_batch(sc, T[None], hessian=hessian)
    return (float(L.item()), g[0].cpu().numpy(), None if H is None else H[0].cpu().numpy(),
            int(st.item()))


def path_length(spec: PathSpec, T) -> float:
    """Total Euclidean length of the embedded path (objective.py:34-37)."""
    if spec.n == 0:
        check_params(spec, T)
        return float(np.linalg.norm(spec.end - spec.start))
    return _objective(spec, T, False)[0]


def gradient(spec: PathSpec, T) -> np.ndarray:
    """dL/dT (n, 2); raises DegenerateSegment like objective.py:40-45."""
    if spec.n == 0:
        check_params(spec, T)
        return np.zeros((0, 2))
    _, g, _, st = _objective(spec, T, False)
    if st & _lib.STATUS_DEGENERATE_FINAL:
        raise DegenerateSegment("consecutive path points (nearly) coincide")
    return g


def hessian(spec: PathSpec, T) -> np.ndarray:
    """Exact 2n x 2n block-tridiagonal Hessian (objective.py:48-64)."""
    if spec.n == 0:
        check_params(spec, T)
        return np.zeros((0, 0))
    _, _, H, st = _objective(spec, T, True)
    if st & _lib.STATUS_DEGENERATE_FINAL:
        raise DegenerateSegment("consecutive path points (nearly) coincide")
    return H


def _mixed(spec: PathSpec, T, u, w_L):
    from .implicit_diff import _one

    if spec.n == 0:
        check_params(spec, T)
        e = (spec.end - spec.start) / np.linalg.norm(spec.end - spec.start)
        return SceneGradient(np.zeros((0, 3, 2)), np.zeros((0, 3)), -w_L * e, w_L * e)
    sg, _ = _one(spec, T, u, w_L, "mixed", gate=False)
    return sg


def length_param_gradient(spec: PathSpec, T) -> SceneGradient:
    """dL/dtheta at fixed T (objective.py:89-98)."""
    return _mixed(spec, T, None, 1.0)


def param_vjp(spec: PathSpec, T, u) -> SceneGradient:
    """u^T d(grad_T L)/dtheta (objective.py:101-135)."""
    check_params(spec, u)
    return _mixed(spec, T, u, 0.0)

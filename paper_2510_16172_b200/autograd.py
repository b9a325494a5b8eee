"""Differentiable batched path solve for PyTorch (autograd over the implicit VJP).

`fermat_paths(basis, anchor, start, end)` solves every path on the GPU
(fp_solve_f32 / _f64) and returns the optimal parameters T*, the lengths L*
and the interaction points; their backward is the implicit-differentiation
VJP of the reference (implicit_diff.vjp_solution + length_param_gradient,
implicit_diff.py:74-106, objective.py:89-135) in one kernel (fp_vjp_*), not
autograd through the BFGS iterations. Cotangents:

    on L*:      w_L = dLoss/dL*            -> full gradient dL*/dtheta
    on T*:      v_T = dLoss/dT*            -> vjp_solution(v_T)
    on points:  x_i = A_i t_i + b_i        -> direct terms (dA_i += g t_i^T,
                                              db_i += g) plus A_i^T g into v_T

T0 receives no gradient (the optimum does not depend on the start point).
The VJP is exact at stationary points only; `status` (returned, not
differentiable) marks the others (FP_STATUS_UNCONVERGED_MASK), whose
gradient rows the caller should mask. Precision follows the inputs' dtype.
"""

from __future__ import annotations

import torch

from .batching import BatchScene
from .implicit_diff import vjp_batch
from .solver import Precision, SolveOptions, solve


class _FermatPaths(torch.autograd.Function):
    @staticmethod
    def forward(ctx, basis, anchor, start, end, T0, iterations, fixed_point_iters):
        sc = BatchScene(basis.detach(), anchor.detach(), start.detach(), end.detach())
        prec = Precision.SINGLE if sc.basis.dtype == torch.float32 else Precision.DOUBLE
        res = solve(sc, None if T0 is None else T0.detach(),
                    SolveOptions(iterations=iterations, fixed_point_iters=fixed_point_iters,
                                 precision=prec), want_grad=False, want_points=True)
        ctx.save_for_backward(sc.basis, sc.anchor, sc.start, sc.end, res.T)
        ctx.mark_non_differentiable(res.status)
        return res.T, res.length, res.points, res.status

    @staticmethod
    def backward(ctx, gT, gL, gP, _gst):
        basis, anchor, start, end, T = ctx.saved_tensors
        sc = BatchScene(basis, anchor, start, end)
        v_T = None if gT is None else gT.contiguous()
        if gP is not None:
            # points x_i = A_i t_i + b_i: A_i^T g_i joins the cotangent on T*
            aTg = torch.einsum("bkrc,bkr->bkc", basis, gP)
            v_T = aTg if v_T is None else v_T + aTg
        w_L = None if gL is None else gL.contiguous()
        if v_T is None and w_L is None:
            return None, None, None, None, None, None, None
        grads, _, _ = vjp_batch(sc, T, v_T=v_T, w_L=w_L, mode="full")
        d_basis, d_anchor = grads.basis, grads.anchor
        if gP is not None:
            d_basis = d_basis + gP.unsqueeze(-1) * T.unsqueeze(-2)
            d_anchor = d_anchor + gP
        return d_basis, d_anchor, grads.start, grads.end, None, None, None


def fermat_paths(basis: torch.Tensor, anchor: torch.Tensor, start: torch.Tensor, end: torch.Tensor,
                 T0: torch.Tensor | None = None, iterations: int = 20, fixed_point_iters: int = 1):
    """Differentiable batched solve: (T* (B,K,2), L* (B,), points (B,K,3), status (B,) uint8).

    Inputs are CUDA tensors in the reference layout (basis (B,K,3,2), anchor
    (B,K,3), start/end (B,3)), float32 or float64; gradients flow to all four
    through the implicit VJP kernel (see the module docstring).
    """
    return _FermatPaths.apply(basis, anchor, start, end, T0, int(iterations), int(fixed_point_iters))

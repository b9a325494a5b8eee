"""torch.autograd over the solve: backward = the implicit VJP kernel.

Checks (1) d(sum L*)/dtheta through autograd equals the fused solve + VJP
kernel bit for bit, and (2) a loss mixing L*, T* and the interaction points
against central finite differences of the fp64 solve (paths are independent,
so one perturbed solve gives the difference quotient of every path at once).
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200 import _lib, datagen, fermat_paths
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve_with_gradients

pytestmark = pytest.mark.gpu


def _tensors(b, dt):
    return [torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt).requires_grad_(True)
            for x in (b.basis, b.anchor, b.start, b.end)]


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_length_gradient_equals_fused_kernel(dt):
    b = datagen.gen_batch(21, datagen.all_orderings(3), 64)
    basis, anchor, start, end = _tensors(b, dt)
    T, L, P, st = fermat_paths(basis, anchor, start, end, iterations=20)
    L.sum().backward()
    prec = Precision.SINGLE if dt == torch.float32 else Precision.DOUBLE
    res, g = solve_with_gradients(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0,
                                  SolveOptions(iterations=20, precision=prec), weight=1.0)
    assert torch.equal(T.detach(), res.T) and torch.equal(L.detach(), res.length)
    for x, y in ((basis.grad, g.basis), (anchor.grad, g.anchor), (start.grad, g.start),
                 (end.grad, g.end)):
        assert torch.equal(x, y)


def test_mixed_loss_matches_finite_differences():
    b = datagen.gen_batch(22, ["RD", "DR", "RR", "DD"], 64)
    dt = torch.float64
    iters = 200
    basis, anchor, start, end = _tensors(b, dt)
    gen = torch.Generator(device="cuda").manual_seed(0)
    B, K = b.size, 2
    wL = torch.rand(B, device="cuda", dtype=dt, generator=gen)
    wT = torch.randn(B, K, 2, device="cuda", dtype=dt, generator=gen)
    wP = torch.randn(B, K, 3, device="cuda", dtype=dt, generator=gen)
    edge = torch.from_numpy(np.all(b.basis[..., 1] == 0, axis=-1)).cuda()
    wT[..., 1][edge] = 0.0  # inert coordinates of edges carry no cotangent

    def per_path(bs, an, s0, s1):
        T, L, P, st = fermat_paths(bs, an, s0, s1, iterations=iters)
        return wL * L + (wT * T).sum((1, 2)) + (wP * P).sum((1, 2)), st

    loss, st = per_path(basis, anchor, start, end)
    loss.sum().backward()
    # finite differences resolve the optimum only where the solve converged
    # tightly (|g| far below the 1e-5 gate): perturbed solves then land on
    # the same stationary point to ~1e-12
    from paper_2510_16172_b200.solver import solve
    ref = solve(BatchScene(b.basis, b.anchor, b.start, b.end), None,
                SolveOptions(iterations=iters, precision=Precision.DOUBLE))
    gn = torch.linalg.vector_norm(ref.g.reshape(B, -1), dim=1)
    conv = (((st & _lib.STATUS_UNCONVERGED_MASK) == 0) & (gn < 1e-10)).cpu().numpy()
    assert conv.mean() > 0.4
    h = 1e-5
    leaves = (basis, anchor, start, end)
    checks = [(2, (0,)), (3, (2,)), (1, (0, 1)), (1, (1, 2)), (0, (0, 2, 0)), (0, (1, 0, 0))]
    for k, idx in checks:
        t = leaves[k]
        with torch.no_grad():
            ins = [x.detach().clone() for x in leaves]
            plus = [x.clone() for x in ins]
            minus = [x.clone() for x in ins]
            plus[k][(slice(None),) + idx] += h
            minus[k][(slice(None),) + idx] -= h
            lp, _ = per_path(*plus)
            lm, _ = per_path(*minus)
        fd = ((lp - lm) / (2 * h)).cpu().numpy()
        ad = t.grad[(slice(None),) + idx].cpu().numpy()
        err = np.abs(ad - fd) / np.maximum(np.abs(fd), 1e-3)
        assert np.all(err[conv] < 1e-4), (k, idx, float(err[conv].max()))


def test_implicit_gradient_matches_autodiff_through_iterations():
    """Independent check of the VJP kernel: autograd through the same BFGS
    written in torch ops (tools/implicit_vs_ad.py) agrees with the implicit
    gradient on converged paths (fp64, 50 iterations)."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "implicit_vs_ad", os.path.join(os.path.dirname(__file__), "..", "tools", "implicit_vs_ad.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    b = datagen.gen_batch(23, datagen.all_orderings(2), 512)
    xs = [torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.float64).requires_grad_(True)
          for x in (b.basis, b.anchor, b.start, b.end)]
    _, L = mod.bfgs_torch(*xs, 50)
    L.sum().backward()
    res, g = solve_with_gradients(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0,
                                  SolveOptions(iterations=50, precision=Precision.DOUBLE))
    conv = (res.status & _lib.STATUS_UNCONVERGED_MASK) == 0
    fin = torch.isfinite(xs[1].grad.reshape(b.size, -1)).all(1)
    m = conv & fin
    assert m.float().mean() > 0.4
    for ad, im in ((xs[0].grad, g.basis), (xs[1].grad, g.anchor), (xs[2].grad, g.start), (xs[3].grad, g.end)):
        a, i = ad[m].reshape(int(m.sum()), -1), im[m].reshape(int(m.sum()), -1)
        rel = torch.linalg.vector_norm(a - i, dim=1) / torch.linalg.vector_norm(i, dim=1)
        assert float(rel.median()) < 1e-6 and float(torch.quantile(rel, 0.9)) < 1e-3

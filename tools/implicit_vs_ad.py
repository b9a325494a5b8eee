"""The paper's gradient claim on B200: implicit differentiation at the optimum
vs automatic differentiation through the unrolled solver iterations.

AD baseline: the same fixed-iteration BFGS with the fixed-point step size
(solver.py:84-215: dense 2K formulation, curvature skip, F = 1) written in
torch ops over the batch, differentiated by torch.autograd through every
iteration. Implicit: the fused forward + VJP kernel (one launch). Prints the
time of each per iteration count and the gradient agreement on converged
paths (the AD gradient of the unrolled solve tends to the implicit one as the
iterations converge).

    python tools/implicit_vs_ad.py [--paths 65536] [--order 3]
"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve_with_gradients  # noqa: E402


def bfgs_torch(basis, anchor, start, end, iters):
    """Batched BFGS in torch ops (differentiable), zero init, F = 1."""
    B, K = basis.shape[:2]
    eps = 1e-12 * (1 + torch.linalg.vector_norm(end - start, dim=-1))

    def points(T):
        x = torch.einsum("bkrc,bkc->bkr", basis, T) + anchor
        return torch.cat([start[:, None], x, end[:, None]], 1)

    def grad(T):
        s = torch.diff(points(T), dim=1)
        n = torch.clamp(torch.linalg.vector_norm(s, dim=-1), min=eps[:, None])
        u = s / n[..., None]
        return torch.einsum("bkrc,bkr->bkc", basis, u[:, :-1] - u[:, 1:]).reshape(B, 2 * K), s, n

    T = torch.zeros(B, K, 2, dtype=basis.dtype, device=basis.device)
    g, s, n = grad(T)
    H = torch.eye(2 * K, dtype=basis.dtype, device=basis.device).expand(B, 2 * K, 2 * K)
    for _ in range(iters):
        p = -torch.einsum("bij,bj->bi", H, g)
        w = torch.einsum("bkrc,bkc->bkr", basis, p.reshape(B, K, 2))
        zero = torch.zeros_like(w[:, :1])
        d = torch.diff(torch.cat([zero, w, zero], 1), dim=1)
        a2 = (d * d).sum(-1)
        c = (d * s).sum(-1)
        den = (a2 / n).sum(-1)
        alpha = -(c / n).sum(-1) / torch.where(den > 0, den, torch.ones_like(den))
        alpha = torch.where(torch.isfinite(alpha) & (a2.sum(-1) > 0), alpha, torch.zeros_like(alpha))
        sg = alpha[:, None] * p
        T = T + sg.reshape(B, K, 2)
        gn, s, n = grad(T)
        y = gn - g
        sy = (sg * y).sum(-1)
        # the curvature test is a branch, not part of the derivative (and the
        # norm of a zero step has no gradient): evaluate it on detached values
        ok = sy.detach() > 1e-12 * torch.linalg.vector_norm(sg.detach(), dim=-1) * torch.linalg.vector_norm(
            y.detach(), dim=-1)
        rho = torch.where(ok, 1 / torch.where(ok, sy, torch.ones_like(sy)), torch.zeros_like(sy))
        Hy = torch.einsum("bij,bj->bi", H, y)
        yHy = (y * Hy).sum(-1)
        upd = (-rho[:, None, None] * (sg[:, :, None] * Hy[:, None, :] + Hy[:, :, None] * sg[:, None, :])
               + ((rho * rho * yHy + rho)[:, None, None]) * sg[:, :, None] * sg[:, None, :])
        H = H + torch.where(ok[:, None, None], upd, torch.zeros_like(upd))
        g = gn
    return T, torch.linalg.vector_norm(s, dim=-1).sum(-1)


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--paths", type=int, default=1 << 16)
    ap.add_argument("--order", type=int, default=3)
    args = ap.parse_args()
    K = args.order
    b = datagen.gen_batch(5, datagen.all_orderings(K), args.paths // 2 ** K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    leaves = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (b.basis, b.anchor, b.start, b.end)]
    for iters in (10, 20, 50):
        opts = SolveOptions(iterations=iters, precision=Precision.SINGLE)

        def ad():
            xs = [x.clone().requires_grad_(True) for x in leaves]
            _, L = bfgs_torch(*xs, iters)
            L.sum().backward()
            return xs

        def implicit():
            return solve_with_gradients(sc, b.T0, opts)

        t_ad = timed(ad, 3)
        t_im = timed(implicit, 10)
        xs = ad()
        res, g = implicit()
        conv = ((res.status & _lib.STATUS_UNCONVERGED_MASK) == 0)
        # AD through overflowing BFGS updates (which the kernel skips,
        # solver.py:196-199) can return NaN: compare where it is finite
        fin = torch.isfinite(xs[1].grad.reshape(b.size, -1)).all(1)
        m = conv & fin
        da, di = xs[1].grad[m].reshape(int(m.sum()), -1), g.anchor[m].reshape(int(m.sum()), -1)
        rel = (torch.linalg.vector_norm(da - di, dim=1) / torch.linalg.vector_norm(di, dim=1)).median()
        print(f"K={K} I={iters} B={b.size}: AD through iterations {t_ad:8.2f} ms, implicit VJP kernel "
              f"(fused with the solve) {t_im:6.3f} ms, ratio {t_ad / t_im:7.1f}x; converged "
              f"{float(conv.float().mean()):.2f}, median rel. diff of dL/d(anchor) {float(rel):.1e} "
              f"({int(m.sum())} converged paths with a finite AD gradient)", flush=True)


if __name__ == "__main__":
    main()

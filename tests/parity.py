"""Parity helpers shared by the GPU tests (test infrastructure; uses the oracle).

Contract (BASELINE.json north_star):
  * a path is CONVERGED per the oracle when its reference result is finite,
    |grad_T L| < 1e-5 (1 + L) recomputed in fp64 at the reference T
    (implicit_diff.py:25,30-36), and its shortest segment exceeds 1e-3 m;
  * on converged paths, interaction points and lengths agree within 1e-5
    relative or 1e-4 m absolute; gradients within 1e-3 relative (norm-wise
    per path, as bench.py:510);
  * on unconverged paths only the agreement fraction is reported (the fp32
    reference moves by more than that under a 1-ulp input change).
"""

from __future__ import annotations

import os

import numpy as np

from oracle import fermat_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

POINT_REL, POINT_ABS = 1e-5, 1e-4
GRAD_REL = 1e-3


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def converged_mask(basis, anchor, start, end, T):
    """Oracle classification at reference T (fp64 recompute)."""
    f = np.float64
    b, a, x0, x1, t = (np.asarray(z, f) for z in (basis, anchor, start, end, T))
    eps = O.seg_floor(x0, x1, f)
    s, n = O.seg_and_norm(O.path_points(b, a, x0, x1, t))
    u = s / np.maximum(n, eps[:, None])[..., None]
    g = np.einsum("bnij,bni->bnj", b, u[:, :-1] - u[:, 1:])
    gn = np.sqrt(np.einsum("bnj,bnj->b", g, g))
    L = n.sum(axis=1)
    fin = np.isfinite(t).all(axis=(1, 2)) & np.isfinite(L)
    return fin & (gn < 1e-5 * (1.0 + L)) & (n.min(axis=1) > 1e-3)


def points_ok(p, p_ref):
    """Per path: every interaction point within 1e-5 rel or 1e-4 abs."""
    d = np.linalg.norm(np.asarray(p, np.float64) - p_ref, axis=-1)
    lim = np.maximum(POINT_REL * np.linalg.norm(p_ref, axis=-1), POINT_ABS)
    return np.all(d <= lim, axis=-1)


def lengths_ok(L, L_ref):
    L = np.asarray(L, np.float64)
    return np.abs(L - L_ref) <= np.maximum(POINT_REL * np.abs(L_ref), POINT_ABS)


def flat_grad(db, da, d0, d1):
    n = db.shape[0]
    return np.concatenate([np.reshape(db, (n, -1)), np.reshape(da, (n, -1)),
                           np.reshape(d0, (n, -1)), np.reshape(d1, (n, -1))], axis=1)


def grad_rel_err(g, g_ref):
    g = np.asarray(g, np.float64)
    return np.linalg.norm(g - g_ref, axis=1) / np.maximum(np.linalg.norm(g_ref, axis=1), 1e-30)


def self_agreement(basis, anchor, start, end, T0, iterations, fp_iters, dtype):
    """The reference's own agreement on its UNCONVERGED paths under a 1-ulp
    change of the inputs (start nudged to the next representable value):
    the fraction whose points and lengths stay within the contract
    tolerance (99.98% RD/10 it, 94.1% RDR/20 it, 90.5%
    RRR/20 it in fp32). Returns (fraction, count of unconverged paths)."""
    dt = np.dtype(dtype).type
    ref = O.solve_outputs(basis, anchor, start, end, T0, iterations, fp_iters, dt)
    nudged = np.nextafter(np.asarray(start, dt), np.asarray(np.inf, dt))
    pert = O.solve_outputs(basis, anchor, nudged, end, T0, iterations, fp_iters, dt)
    conv = converged_mask(basis, anchor, start, end, ref["T"])
    ok = points_ok(pert["points"], ref["points"]) & lengths_ok(pert["L"], ref["L"])
    n = int((~conv).sum())
    return (float(ok[~conv].mean()) if n else 1.0), n


def agreement_floor(basis, anchor, start, end, T0, iterations, fp_iters, dtype):
    """Floor for the GPU's agreement with the reference on unconverged paths:
    the reference's 1-ulp self-agreement less two binomial standard errors
    of the sample (and never above 1)."""
    p, n = self_agreement(basis, anchor, start, end, T0, iterations, fp_iters, dtype)
    if n == 0:
        return 0.0
    return max(0.0, p - 2.0 * np.sqrt(max(p * (1 - p), 1.0 / n) / n))

"""numpy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

This module is the CPU oracle (see oracle/__init__.py for who may import
it). Every function cites the reference code it restates; the restatement
keeps the reference's numpy contraction structure so that, run in the same
numpy build, it reproduces the reference bit for bit (pinned by
tests/test_oracle_pin.py against tests/golden/*.npz).

Array conventions (reference batching.py:20-25): basis (B,K,3,2),
anchor (B,K,3), start (B,3), end (B,3), parameters T (B,K,2).
"""

from __future__ import annotations

import numpy as np

# implicit_diff.py:25-27
STATIONARITY_TOL = 1e-5
TIKHONOV_SCALE = 1e-12
RESIDUAL_TOL = 1e-8
# solver.py:169
CURVATURE_TOL = 1e-12


class OracleDegenerate(Exception):
    """Stands in for the reference's DegenerateSegment (errors.py:16)."""


class OracleNotStationary(Exception):
    """Stands in for the reference's NotStationary (errors.py:44)."""


class OracleSingular(Exception):
    """Stands in for the reference's SingularSystem (errors.py:48)."""


# ---------------------------------------------------------------------------
# Batched geometry (reference batching.py)


def seg_floor(start, end, dtype):
    """Per-path segment floor 1e-12(1+|end-start|), fp64 then cast (batching.py:67-72)."""
    d = np.asarray(end, np.float64) - np.asarray(start, np.float64)
    return (1e-12 * (1.0 + np.linalg.norm(d, axis=1))).astype(dtype)


def path_points(basis, anchor, start, end, T):
    """[start, A_i t_i + b_i, end] per path (batching.py:83-86)."""
    inner = np.einsum("bnij,bnj->bni", basis, T) + anchor
    return np.concatenate([start[:, None], inner, end[:, None]], axis=1)


def seg_and_norm(pts):
    """Segments and their Euclidean norms (batching.py:89-92)."""
    s = pts[:, 1:] - pts[:, :-1]
    return s, np.sqrt(np.einsum("bki,bki->bk", s, s))


def clamped(basis, anchor, start, end, T, eps):
    """Segments with norms floored at eps (batching.py:117-120)."""
    s, nrm = seg_and_norm(path_points(basis, anchor, start, end, T))
    return s, np.maximum(nrm, eps[:, None])


def grad_batch(basis, anchor, start, end, T, eps):
    """Clamped-norm gradient A_i^T (u_{i-1} - u_i) (batching.py:95-104)."""
    s, nrm = clamped(basis, anchor, start, end, T, eps)
    u = s / nrm[..., None]
    return np.einsum("bnij,bni->bnj", basis, u[:, :-1] - u[:, 1:])


def length_batch(basis, anchor, start, end, T):
    """Unclamped total length (batching.py:123-126)."""
    _, nrm = seg_and_norm(path_points(basis, anchor, start, end, T))
    return np.einsum("bk->b", nrm)


def degenerate_rows(basis, anchor, start, end, T, eps):
    """Rows whose entry segments fail the checked_segments test (batching.py:107-114)."""
    _, nrm = seg_and_norm(path_points(basis, anchor, start, end, T))
    return np.any(nrm <= eps[:, None], axis=1)


# ---------------------------------------------------------------------------
# Forward solver (reference solver.py)


def fixed_point_step(basis, s, P, iters, eps):
    """Paper Eq. 6 fixed-point step size from alpha=0 (solver.py:84-112)."""
    dt = s.dtype
    B = P.shape[0]
    w = np.einsum("bnij,bnj->bni", basis, P)
    z = np.zeros((B, 1, 3), dtype=dt)
    d = np.diff(np.concatenate([z, w, z], axis=1), axis=1)
    a2 = np.einsum("bki,bki->bk", d, d)
    c = np.einsum("bki,bki->bk", d, s)
    zero = np.einsum("bk->b", a2) <= np.finfo(dt).tiny
    alpha = np.zeros(B, dtype=dt)
    for _ in range(iters):
        trial = s + alpha[:, None, None] * d
        den = np.maximum(np.sqrt(np.einsum("bki,bki->bk", trial, trial)), eps[:, None])
        num = np.einsum("bk->b", c / den)
        dsum = np.einsum("bk->b", a2 / den)
        cand = -num / np.where(zero, np.ones_like(dsum), dsum)
        alpha = np.where(zero | ~np.isfinite(cand), alpha, cand)
    return alpha, zero


def bfgs(basis, anchor, start, end, T0, iterations, fp_iters=1, dtype=np.float32,
         trace=False, return_H=False):
    """Fixed-iteration batch BFGS (solver.py:146-215).

    Returns a dict with T, g, and optionally trace_len/trace_gnorm (I,B), H,
    and (with trace) the fate of every update, trace_fate (I,B) uint8: bit 0
    the curvature test failed (solver.py:182-184), bit 1 H' was not finite
    and the update was skipped (solver.py:196-199), bit 2 the step size met
    a zero direction (solver.py:100,110-111). Not a reference output: the
    reference computes the same masks internally.
    Raises OracleDegenerate when any entry segment is degenerate, like the
    reference's whole-batch DegenerateSegment (solver.py:166).
    """
    basis = np.asarray(basis).astype(dtype)
    anchor = np.asarray(anchor).astype(dtype)
    start = np.asarray(start).astype(dtype)
    end = np.asarray(end).astype(dtype)
    T = np.ascontiguousarray(T0, dtype=dtype)
    B, K = T.shape[0], T.shape[1]
    m = 2 * K
    eps = seg_floor(start, end, dtype)
    out = {}
    if K == 0:
        out.update(T=T, g=np.zeros((B, 0, 2), dtype))
        return out
    if np.any(degenerate_rows(basis, anchor, start, end, T, eps)):
        raise OracleDegenerate("coincident consecutive path points in batch")
    H = np.broadcast_to(np.eye(m, dtype=dtype), (B, m, m)).copy()
    g = grad_batch(basis, anchor, start, end, T, eps).reshape(B, m)
    tol = dtype(CURVATURE_TOL)
    tl, tg, tf = [], [], []
    for _ in range(iterations):
        p = -np.einsum("bij,bj->bi", H, g)
        s, _ = clamped(basis, anchor, start, end, T, eps)
        alpha, zero = fixed_point_step(basis, s, p.reshape(B, K, 2), fp_iters, eps)
        sigma = alpha[:, None] * p
        T = T + sigma.reshape(B, K, 2)
        g1 = grad_batch(basis, anchor, start, end, T, eps).reshape(B, m)
        y = g1 - g
        sy = np.einsum("bi,bi->b", sigma, y)
        sn = np.sqrt(np.einsum("bi,bi->b", sigma, sigma))
        yn = np.sqrt(np.einsum("bi,bi->b", y, y))
        ok = sy > tol * sn * yn
        rho = np.where(ok, np.ones_like(sy) / np.where(ok, sy, np.ones_like(sy)), 0.0)
        with np.errstate(over="ignore", invalid="ignore"):
            Hy = np.einsum("bij,bj->bi", H, y)
            yHy = np.einsum("bi,bi->b", y, Hy)
            cross = np.einsum("bi,bj->bij", sigma, Hy)
            outer = np.einsum("bi,bj->bij", sigma, sigma)
            Hn = (H - rho[:, None, None] * (cross + np.swapaxes(cross, 1, 2))
                  + (rho * rho * yHy + rho)[:, None, None] * outer)
        curv = ok
        ok = ok & np.all(np.isfinite(Hn), axis=(1, 2))
        H = np.where(ok[:, None, None], Hn, H)
        g = g1
        if trace:
            tl.append(length_batch(basis, anchor, start, end, T))
            tg.append(np.sqrt(np.einsum("bi,bi->b", g, g)))
            tf.append(np.where(curv, 0, 1).astype(np.uint8) | np.where(curv & ~ok, 2, 0).astype(np.uint8)
                      | np.where(zero, 4, 0).astype(np.uint8))
    out.update(T=T, g=g.reshape(B, K, 2))
    if trace:
        out.update(trace_len=np.stack(tl), trace_gnorm=np.stack(tg), trace_fate=np.stack(tf))
    if return_H:
        out["H"] = H
    return out


def solve_outputs(basis, anchor, start, end, T0, iterations, fp_iters=1, dtype=np.float32):
    """T, g, final length in T's dtype, points in fp64 (solver.py:218-232, bench.py:313-314)."""
    r = bfgs(basis, anchor, start, end, T0, iterations, fp_iters, dtype)
    T = r["T"]
    bd = basis.astype(dtype)
    r["L"] = length_batch(bd, anchor.astype(dtype), start.astype(dtype), end.astype(dtype), T)
    r["points"] = path_points(basis.astype(np.float64), anchor.astype(np.float64),
                              start.astype(np.float64), end.astype(np.float64),
                              T.astype(np.float64))[:, 1:-1]
    return r


def line_search(basis, anchor, start, end, T, P, alpha0=0.0, k=1):
    """Scalar fixed-point line search with caller's alpha0 (solver.py:115-143).

    Single path (arrays without the batch axis), fp64.
    """
    b1 = basis[None].astype(np.float64)
    a1 = anchor[None].astype(np.float64)
    x0 = np.asarray(start, np.float64)[None]
    xe = np.asarray(end, np.float64)[None]
    eps = seg_floor(x0, xe, np.float64)
    s, nrm = seg_and_norm(path_points(b1, a1, x0, xe, np.asarray(T, np.float64)[None]))
    if np.any(nrm <= eps[:, None]):
        raise OracleDegenerate("entry segment collapsed")
    w = np.einsum("bnij,bnj->bni", b1, np.asarray(P, np.float64)[None])
    z = np.zeros((1, 1, 3))
    d = np.diff(np.concatenate([z, w, z], axis=1), axis=1)
    a2 = np.einsum("bki,bki->bk", d, d)
    if float(a2.sum()) <= np.finfo(np.float64).tiny:
        raise ZeroDivisionError("zero direction")
    c = np.einsum("bki,bki->bk", d, s)
    alpha = np.full(1, alpha0, dtype=np.float64)
    for _ in range(k):
        trial = s + alpha[:, None, None] * d
        den = np.sqrt(np.einsum("bki,bki->bk", trial, trial))
        if np.any(den <= eps[:, None]):
            raise OracleDegenerate("denominator segment collapsed")
        alpha = -np.einsum("bk->b", c / den) / np.einsum("bk->b", a2 / den)
    return float(alpha[0])


def init_guess(basis, anchor, start, end):
    """Least-squares projection of the midpoint onto each active span (solver.py:67-81).

    Single path, fp64.
    """
    mid = 0.5 * (np.asarray(start, float) + np.asarray(end, float))
    K = basis.shape[0]
    T = np.zeros((K, 2))
    for i in range(K):
        act = np.linalg.norm(basis[i], axis=0) > 0.0
        A = basis[i][:, act]
        T[i, act] = np.linalg.solve(A.T @ A, A.T @ (mid - anchor[i]))
    return T


# ---------------------------------------------------------------------------
# Scalar calculus in fp64 (reference objective.py)


def _scalar_segments(basis, anchor, start, end, T):
    """Points, segments, norms; raises on degenerate segments (objective.py:25-31)."""
    pts = np.empty((basis.shape[0] + 2, 3))
    pts[0], pts[-1] = start, end
    if basis.shape[0]:
        pts[1:-1] = np.einsum("nij,nj->ni", basis, T) + anchor
    s = np.diff(pts, axis=0)
    nrm = np.linalg.norm(s, axis=1)
    if np.any(nrm <= 1e-12 * (1.0 + np.linalg.norm(np.asarray(end) - np.asarray(start)))):
        raise OracleDegenerate("consecutive path points (nearly) coincide")
    return pts, s, nrm


def scalar_length(basis, anchor, start, end, T):
    """objective.path_length (objective.py:34-37)."""
    pts = np.empty((basis.shape[0] + 2, 3))
    pts[0], pts[-1] = start, end
    if basis.shape[0]:
        pts[1:-1] = np.einsum("nij,nj->ni", basis, T) + anchor
    return float(np.linalg.norm(np.diff(pts, axis=0), axis=1).sum())


def scalar_gradient(basis, anchor, start, end, T):
    """objective.gradient (objective.py:40-45)."""
    _, s, nrm = _scalar_segments(basis, anchor, start, end, T)
    u = s / nrm[:, None]
    return np.einsum("nij,ni->nj", basis, u[:-1] - u[1:])


def scalar_hessian(basis, anchor, start, end, T):
    """Exact block-tridiagonal Hessian (objective.py:48-64)."""
    _, s, nrm = _scalar_segments(basis, anchor, start, end, T)
    K = basis.shape[0]
    u = s / nrm[:, None]
    M = (np.eye(3)[None] - np.einsum("ki,kj->kij", u, u)) / nrm[:, None, None]
    H = np.zeros((2 * K, 2 * K))
    for i in range(K):
        H[2 * i:2 * i + 2, 2 * i:2 * i + 2] = basis[i].T @ (M[i] + M[i + 1]) @ basis[i]
        if i + 1 < K:
            off = -basis[i].T @ M[i + 1] @ basis[i + 1]
            H[2 * i:2 * i + 2, 2 * i + 2:2 * i + 4] = off
            H[2 * i + 2:2 * i + 4, 2 * i:2 * i + 2] = off.T
    return H


def partial_gradient(basis, anchor, start, end, T):
    """dL/dtheta at fixed T -> (basis (K,3,2), anchor (K,3), start, end) (objective.py:89-98)."""
    _, s, nrm = _scalar_segments(basis, anchor, start, end, T)
    u = s / nrm[:, None]
    q = u[:-1] - u[1:]
    return (np.einsum("ni,nj->nij", q, T), q.copy(), -u[0], u[-1].copy())


def mixed_vjp(basis, anchor, start, end, T, U):
    """U^T d(grad_T L)/d(theta) (objective.py:101-135)."""
    _, s, nrm = _scalar_segments(basis, anchor, start, end, T)
    uh = s / nrm[:, None]
    K = basis.shape[0]
    dx = np.zeros((K + 2, 3))
    if K:
        dx[1:-1] = np.einsum("nij,nj->ni", basis, U)
    ds = np.diff(dx, axis=0)
    w = (ds - uh * np.einsum("ki,ki->k", uh, ds)[:, None]) / nrm[:, None]
    z = w[:-1] - w[1:]
    q = uh[:-1] - uh[1:]
    return (np.einsum("ni,nj->nij", z, T) + np.einsum("ni,nj->nij", q, U),
            z, -w[0], w[-1].copy())


def _active(basis):
    return np.linalg.norm(basis, axis=1) > 0.0  # (K, 2)


def require_stationary(basis, anchor, start, end, T):
    """Gate |g| < 1e-5 (1 + L) (implicit_diff.py:30-36)."""
    g = scalar_gradient(basis, anchor, start, end, T)
    L = scalar_length(basis, anchor, start, end, T)
    if np.linalg.norm(g) >= STATIONARITY_TOL * (1.0 + L):
        raise OracleNotStationary(f"gradient norm {np.linalg.norm(g):.3e}")


def is_stationary(basis, anchor, start, end, T):
    try:
        require_stationary(basis, anchor, start, end, T)
    except (OracleNotStationary, OracleDegenerate):
        return False
    return True


def _solve_sym(Ha, rhs):
    """LAPACK solve with residual check and Tikhonov fallback (implicit_diff.py:55-71)."""
    if Ha.size == 0:
        return rhs.copy()
    try:
        x = np.linalg.solve(Ha, rhs)
        if np.linalg.norm(Ha @ x - rhs) <= RESIDUAL_TOL * (1.0 + np.linalg.norm(rhs)):
            return x
    except np.linalg.LinAlgError:
        pass
    lam = TIKHONOV_SCALE * np.trace(Ha)
    try:
        x = np.linalg.solve(Ha + lam * np.eye(Ha.shape[0]), rhs)
    except np.linalg.LinAlgError as exc:
        raise OracleSingular("active Hessian singular") from exc
    if not np.all(np.isfinite(x)):
        raise OracleSingular("non-finite regularised solve")
    return x


def stationary_solve(basis, anchor, start, end, T, v):
    """Solve H_a u_a = -v_a on active coordinates (implicit_diff.py:39-52)."""
    require_stationary(basis, anchor, start, end, T)
    H = scalar_hessian(basis, anchor, start, end, T)
    act = _active(basis).ravel()
    ua = _solve_sym(H[np.ix_(act, act)], -np.asarray(v, float).ravel()[act])
    u = np.zeros(2 * basis.shape[0])
    u[act] = ua
    return u.reshape(-1, 2)


def solution_vjp(basis, anchor, start, end, T, v):
    """v^T dT*/dtheta (implicit_diff.py:74-77)."""
    return mixed_vjp(basis, anchor, start, end, T,
                     stationary_solve(basis, anchor, start, end, T, v))


def envelope_gradient(basis, anchor, start, end, T):
    """grad_length_wrt_params return value (implicit_diff.py:80-106)."""
    require_stationary(basis, anchor, start, end, T)
    return partial_gradient(basis, anchor, start, end, T)


def full_gradient(basis, anchor, start, end, T):
    """partial + vjp_solution(grad) — the debug_check 'full' formula (implicit_diff.py:92-100)."""
    part = envelope_gradient(basis, anchor, start, end, T)
    g = scalar_gradient(basis, anchor, start, end, T)
    corr = solution_vjp(basis, anchor, start, end, T, g)
    return tuple(a + b for a, b in zip(part, corr))


def flat(sg):
    """SceneGradient.flat ordering: basis, anchor, start, end (objective.py:76-79)."""
    return np.concatenate([np.ravel(a) for a in sg])


def full_gradient_rows(basis, anchor, start, end, T, rows, weights=None):
    """Full formula for selected rows in fp64; returns stacked arrays + stationary mask.

    Rows that fail the gate (or are degenerate/singular) get NaN gradients.
    """
    K = basis.shape[1]
    n = len(rows)
    db = np.full((n, K, 3, 2), np.nan)
    da = np.full((n, K, 3), np.nan)
    d0 = np.full((n, 3), np.nan)
    d1 = np.full((n, 3), np.nan)
    ok = np.zeros(n, dtype=bool)
    f64 = np.float64
    for j, r in enumerate(rows):
        args = (basis[r].astype(f64), anchor[r].astype(f64), start[r].astype(f64),
                end[r].astype(f64), T[r].astype(f64))
        try:
            sg = full_gradient(*args)
        except (OracleNotStationary, OracleDegenerate, OracleSingular):
            continue
        w = 1.0 if weights is None else float(weights[j])
        db[j], da[j], d0[j], d1[j] = (w * x for x in sg)
        ok[j] = True
    return db, da, d0, d1, ok


# ---------------------------------------------------------------------------
# Comparison solvers (reference baselines.py)

NEWTON_DAMPING = 1e-10      # baselines.py:127
NEWTON_MAX_HALVINGS = 20    # baselines.py:128


def hessian_batched(basis, anchor, start, end, T, eps):
    """(B, 2K, 2K) Hessian with clamped norms (baselines.py:131-149)."""
    s, nrm = clamped(basis, anchor, start, end, T, eps)
    B, K = T.shape[0], T.shape[1]
    u = s / nrm[..., None]
    M = (np.eye(3, dtype=s.dtype)[None, None] - np.einsum("bki,bkj->bkij", u, u)) / nrm[..., None, None]
    H = np.zeros((B, 2 * K, 2 * K), dtype=s.dtype)
    for i in range(K):
        H[:, 2 * i:2 * i + 2, 2 * i:2 * i + 2] = np.einsum(
            "bri,brs,bsj->bij", basis[:, i], M[:, i] + M[:, i + 1], basis[:, i])
        if i + 1 < K:
            off = -np.einsum("bri,brs,bsj->bij", basis[:, i], M[:, i + 1], basis[:, i + 1])
            H[:, 2 * i:2 * i + 2, 2 * i + 2:2 * i + 4] = off
            H[:, 2 * i + 2:2 * i + 4, 2 * i:2 * i + 2] = np.swapaxes(off, 1, 2)
    return H


def newton(basis, anchor, start, end, T0, iterations, dtype=np.float32, trace=False):
    """Masked damped Newton with step halving (baselines.py:152-193)."""
    basis, anchor, start, end = (np.asarray(x).astype(dtype) for x in (basis, anchor, start, end))
    T = np.ascontiguousarray(T0, dtype=dtype)
    B, K = T.shape[0], T.shape[1]
    m = 2 * K
    eps = seg_floor(start, end, dtype)
    active = (np.linalg.norm(basis, axis=2) > 0.0).reshape(B, m)
    dim = active.sum(axis=1).astype(dtype)
    g = grad_batch(basis, anchor, start, end, T, eps)
    tg = []
    for _ in range(iterations):
        H = hessian_batched(basis, anchor, start, end, T, eps)
        gm = np.where(active, g.reshape(B, m), 0.0)
        H = np.where(active[:, :, None] & active[:, None, :], H, 0.0)
        diag = np.arange(m)
        tr = np.einsum("bii->b", H)
        lam = NEWTON_DAMPING * tr / np.maximum(dim, 1.0)
        H[:, diag, diag] = np.where(active, H[:, diag, diag] + lam[:, None], 1.0)
        step = -np.linalg.solve(H, gm[..., None])[..., 0]
        L0 = length_batch(basis, anchor, start, end, T)
        scale = np.ones(B, dtype=dtype)
        cand = T + step.reshape(B, K, 2)
        Lc = length_batch(basis, anchor, start, end, cand)
        for _ in range(NEWTON_MAX_HALVINGS):
            worse = Lc > L0
            if not np.any(worse):
                break
            scale = np.where(worse, scale * 0.5, scale)
            cand = T + scale[:, None, None] * step.reshape(B, K, 2)
            Lc = length_batch(basis, anchor, start, end, cand)
        T = np.where((Lc <= L0)[:, None, None], cand, T)
        g = grad_batch(basis, anchor, start, end, T, eps)
        if trace:
            tg.append(np.sqrt(np.einsum("bnj,bnj->b", g, g)))
    out = dict(T=T, g=g)
    if trace:
        out["trace_gnorm"] = np.stack(tg)
    return out


def image_points(basis, anchor, start, end):
    """Exact reflection points of all-plane paths (baselines.py:48-71), fp64."""
    basis, anchor, start, end = (np.asarray(x, np.float64) for x in (basis, anchor, start, end))
    B, K = basis.shape[0], basis.shape[1]
    nrm = np.cross(basis[..., 0], basis[..., 1])
    nrm = nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)
    imgs = np.empty((B, K, 3))
    m = start.copy()
    for i in range(K):
        d = np.einsum("bi,bi->b", m - anchor[:, i], nrm[:, i])
        m = m - 2.0 * d[:, None] * nrm[:, i]
        imgs[:, i] = m
    pts = np.empty((B, K, 3))
    y = end.copy()
    parallel = np.zeros(B, dtype=bool)
    for i in range(K - 1, -1, -1):
        dirv = y - imgs[:, i]
        den = np.einsum("bi,bi->b", dirv, nrm[:, i])
        parallel |= np.abs(den) <= 1e-12 * np.linalg.norm(dirv, axis=1)
        t = np.einsum("bi,bi->b", anchor[:, i] - imgs[:, i], nrm[:, i]) / den
        y = imgs[:, i] + t[:, None] * dirv
        pts[:, i] = y
    return pts, parallel

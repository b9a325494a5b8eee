"""CPU oracle for the visibility post-processing — TEST INFRASTRUCTURE ONLY.

No reference code exists (SPEC.md:11 puts occlusion out of the reference's
scope; PAPER.md:32,67 describes it as the step after the solve), so this
restatement of csrc/fp_visibility.cu's specification is the oracle ("parity
unpinned" against the reference). It evaluates every float64 operation in the
kernel's order without fused multiply-adds (numpy never fuses), so flags are
compared bit for bit; tests/test_visibility.py pins it with known answers.
"""

from __future__ import annotations

import numpy as np

BLOCKED = 0x01
WRONG_SIDE = 0x02


def crosses(P, D, blk, e):
    """Segments P -> P + D (n, 3) against blockers (Q, 3, 3) -> (n, Q) bool (Moller-Trumbore).

    e: (n,) or scalar fraction of the segment excluded at each end."""
    e = np.asarray(e, np.float64)
    e = e[:, None] if e.ndim == 1 else e
    P = np.asarray(P, np.float64)[:, None, :]
    D = np.asarray(D, np.float64)[:, None, :]
    blk = np.asarray(blk, np.float64)
    O, U, V = blk[None, :, 0], blk[None, :, 1], blk[None, :, 2]
    h0 = D[..., 1] * V[..., 2] - D[..., 2] * V[..., 1]
    h1 = D[..., 2] * V[..., 0] - D[..., 0] * V[..., 2]
    h2 = D[..., 0] * V[..., 1] - D[..., 1] * V[..., 0]
    det = U[..., 0] * h0 + U[..., 1] * h1 + U[..., 2] * h2
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        f = 1.0 / det
        w0, w1, w2 = P[..., 0] - O[..., 0], P[..., 1] - O[..., 1], P[..., 2] - O[..., 2]
        a = f * (w0 * h0 + w1 * h1 + w2 * h2)
        q0 = w1 * U[..., 2] - w2 * U[..., 1]
        q1 = w2 * U[..., 0] - w0 * U[..., 2]
        q2 = w0 * U[..., 1] - w1 * U[..., 0]
        b = f * (D[..., 0] * q0 + D[..., 1] * q1 + D[..., 2] * q2)
        s = f * (V[..., 0] * q0 + V[..., 1] * q1 + V[..., 2] * q2)
        return ((det != 0.0) & (a >= 0.0) & (a <= 1.0) & (b >= 0.0) & (b <= 1.0)
                & (s > e) & (s < 1.0 - e))


def visibility(blockers, tx, rx, rec_rx, points, rec_seq=None, obj_basis=None, obj_plane=None,
               eps=1e-4, chunk=4096):
    """(flags uint8 (n,), first_blocker int32 (n,)) for n traced paths of order K.

    eps: metres excluded at each end of a segment (e = eps / |segment|)."""
    pts = np.asarray(points, np.float32).astype(np.float64)
    n, K = pts.shape[0], pts.shape[1]
    X = np.empty((n, K + 2, 3))
    X[:, 0] = np.asarray(tx, np.float32).astype(np.float64)
    X[:, 1:K + 1] = pts
    X[:, K + 1] = np.asarray(rx, np.float32).astype(np.float64)[np.asarray(rec_rx)]
    flags = np.zeros(n, np.uint8)
    first = np.full(n, -1, np.int32)
    if rec_seq is not None:
        seq = np.asarray(rec_seq)
        A = np.asarray(obj_basis, np.float32).astype(np.float64)
        plane = np.asarray(obj_plane).astype(bool)
        for i in range(K):
            o = seq[:, i]
            a0, a1, a2 = A[o, 0, 0], A[o, 1, 0], A[o, 2, 0]
            b0, b1, b2 = A[o, 0, 1], A[o, 1, 1], A[o, 2, 1]
            n0 = a1 * b2 - a2 * b1
            n1 = a2 * b0 - a0 * b2
            n2 = a0 * b1 - a1 * b0
            xp, x, xn = X[:, i], X[:, i + 1], X[:, i + 2]
            din = (xp[:, 0] - x[:, 0]) * n0 + (xp[:, 1] - x[:, 1]) * n1 + (xp[:, 2] - x[:, 2]) * n2
            dout = (xn[:, 0] - x[:, 0]) * n0 + (xn[:, 1] - x[:, 1]) * n1 + (xn[:, 2] - x[:, 2]) * n2
            wrong = plane[o] & ~(din * dout > 0.0)
            flags[wrong] |= WRONG_SIDE
    blk = np.asarray(blockers, np.float64)
    blocked = np.zeros(n, bool)
    for k in range(K + 1):
        P, D = X[:, k], X[:, k + 1] - X[:, k]
        e = eps / np.sqrt(D[:, 0] * D[:, 0] + D[:, 1] * D[:, 1] + D[:, 2] * D[:, 2])
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            live = np.nonzero(~blocked[lo:hi])[0] + lo
            if live.size == 0 or blk.shape[0] == 0:
                continue
            hit = crosses(P[live], D[live], blk, e[live])
            any_hit = hit.any(axis=1)
            idx = live[any_hit]
            blocked[idx] = True
            first[idx] = np.argmax(hit[any_hit], axis=1).astype(np.int32)
    flags[blocked] |= BLOCKED
    return flags, first

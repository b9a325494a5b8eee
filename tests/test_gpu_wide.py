"""Orders 9..64 on the warp-per-path solver (csrc/fp_wide.cu) against the
reference's golden vectors (tests/golden/fwd_wide_k*.npz, make_golden.py --wide).

The reference accepts up to 64 interactions (geometry.py:23); these paths use
100 iterations from zero init; parity per tests/parity.py on the paths the
reference converges, agreement fractions elsewhere.
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.implicit_diff import vjp_batch
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients
from oracle import fermat_oracle as O

from parity import GRAD_REL, converged_mask, flat_grad, golden, grad_rel_err, lengths_ok, points_ok

pytestmark = pytest.mark.gpu

ORDERS = [9, 12, 16, 33, 64]


def _ref_points(d, T):
    f = np.float64
    return O.path_points(d["basis"].astype(f), d["anchor"].astype(f), d["start"].astype(f),
                         d["end"].astype(f), np.asarray(T, f))[:, 1:-1]


@pytest.mark.parametrize("K", ORDERS)
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_wide_forward_matches_reference(K, prec):
    d = golden(f"fwd_wide_k{K}")
    dt = np.float32 if prec == "f32" else np.float64
    sc = BatchScene(d["basis"], d["anchor"], d["start"], d["end"])
    opts = SolveOptions(iterations=int(d["iterations"]), fixed_point_iters=1,
                        precision=Precision.SINGLE if prec == "f32" else Precision.DOUBLE)
    res = solve(sc, d["T0"], opts)
    torch.cuda.synchronize()
    T_ref = d["T_" + prec]
    conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], T_ref)
    assert conv.sum() >= 4
    pts = res.points.double().cpu().numpy()
    ok = points_ok(pts, _ref_points(d, T_ref)) & lengths_ok(res.length.cpu().numpy(), d["L_" + prec])
    assert ok[conv].all(), f"{(~ok[conv]).sum()} converged paths out of tolerance"
    # inert (edge) coordinates never move
    edge = np.all(d["basis"][..., 1] == 0, axis=-1)
    T = res.T.cpu().numpy()
    assert np.array_equal(T[..., 1][edge], d["T0"][..., 1][edge].astype(dt))
    # the device gate agrees with the oracle's classification on converged paths
    assert res.converged.cpu().numpy()[conv].mean() > 0.99
    if prec == "f64":
        assert np.abs(T - T_ref)[conv].max() < 1e-7


@pytest.mark.parametrize("K", ORDERS)
def test_wide_gradients_match_reference(K):
    d = golden(f"fwd_wide_k{K}")
    sc = BatchScene(d["basis"], d["anchor"], d["start"], d["end"])
    opts = SolveOptions(iterations=int(d["iterations"]), precision=Precision.SINGLE)
    res, grads = solve_with_gradients(sc, d["T0"], opts)
    conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T_f32"])
    stat = d["grad_stationary"] & conv & (res.status.cpu().numpy() == 0)
    assert stat.sum() >= 3
    got = flat_grad(*(g.double().cpu().numpy() for g in (grads.basis, grads.anchor, grads.start, grads.end)))
    ref = flat_grad(d["grad_full_basis"], d["grad_full_anchor"], d["grad_full_start"], d["grad_full_end"])
    assert grad_rel_err(got[stat], ref[stat]).max() < GRAD_REL
    # fp64 VJP of an arbitrary cotangent at the reference solution (vjp_solution)
    sc64 = sc.astype(np.float64)
    T = torch.as_tensor(d["T_f32"].astype(np.float64), device="cuda")
    v = torch.as_tensor(d["grad_v"], device="cuda")
    g64, st, u = vjp_batch(sc64, T, v_T=v, w_L=0.0, mode="full", return_u=True)
    ok = d["grad_stationary"]
    got = flat_grad(*(g.cpu().numpy() for g in (g64.basis, g64.anchor, g64.start, g64.end)))
    ref = flat_grad(d["grad_vjp_basis"], d["grad_vjp_anchor"], d["grad_vjp_start"], d["grad_vjp_end"])
    assert grad_rel_err(got[ok], ref[ok]).max() < 1e-8
    assert np.allclose(u.cpu().numpy()[ok], d["grad_u"][ok], rtol=1e-8, atol=1e-10)


def test_wide_fused_equals_solve_then_vjp():
    d = golden("fwd_wide_k16")
    sc = BatchScene(d["basis"], d["anchor"], d["start"], d["end"])
    opts = SolveOptions(iterations=30, precision=Precision.SINGLE)
    res, grads = solve_with_gradients(sc, d["T0"], opts)
    sep = solve(sc, d["T0"], opts)
    g2, st2, _ = vjp_batch(sc, sep.T, w_L=1.0, mode="full")
    assert torch.equal(res.T, sep.T) and torch.equal(res.length, sep.length)
    for a, b in ((grads.basis, g2.basis), (grads.anchor, g2.anchor), (grads.start, g2.start),
                 (grads.end, g2.end)):
        assert torch.equal(torch.nan_to_num(a, 7.0), torch.nan_to_num(b, 7.0))


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_two_paths_per_warp_are_independent(prec):
    """Orders up to 15 (fp32) / 11 (fp64) run two paths per warp, 16 lanes
    each (csrc/fp_wide.cu), with every shuffle, vote and barrier masked to the
    path's half. Neighbouring paths that take different branches (a NaN row
    whose updates are all skipped next to healthy rows, all-edge next to
    mixed orderings) still get exactly the bits each gets alone — in a batch
    of one, where the other half-warp has no path and leaves at once."""
    from paper_2510_16172_b200 import datagen

    b = datagen.gen_batch(31, ["RDRRDRDDR", "DDDDDDDDD"], 6)
    basis, anchor, start, end, T0 = (np.array(x) for x in (b.basis, b.anchor, b.start, b.end, b.T0))
    anchor[3, 2, 0] = np.nan
    opts = SolveOptions(iterations=30, precision=Precision.SINGLE if prec == "f32" else Precision.DOUBLE)
    res, grads = solve_with_gradients(BatchScene(basis, anchor, start, end), T0, opts)
    torch.cuda.synchronize()
    assert int(res.status[3]) & 0x08  # the NaN row is flagged non-finite
    for i in range(b.size):
        r1, g1 = solve_with_gradients(BatchScene(basis[i:i + 1], anchor[i:i + 1], start[i:i + 1], end[i:i + 1]),
                                      T0[i:i + 1], opts)
        for x, y in ((res.T[i:i + 1], r1.T), (res.length[i:i + 1], r1.length), (res.status[i:i + 1], r1.status),
                     (grads.basis[i:i + 1], g1.basis), (grads.anchor[i:i + 1], g1.anchor),
                     (grads.start[i:i + 1], g1.start), (grads.end[i:i + 1], g1.end)):
            assert torch.equal(torch.nan_to_num(x.double(), 7.0), torch.nan_to_num(y.double(), 7.0)), i


def test_order_above_64_rejected():
    from paper_2510_16172_b200 import datagen

    b = datagen.gen_batch(1, ["D" * 65], 2)
    with pytest.raises((NotImplementedError, ValueError)):
        solve(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0, SolveOptions(iterations=2))

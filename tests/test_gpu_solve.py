"""GPU forward-solve parity against the reference's golden vectors and the oracle.

All calls go through the package API -> C ABI (libfermat_b200.so) -> sm_100a
kernels. Tolerances are stated in tests/parity.py.
"""

import numpy as np
import pytest
import torch

import paper_2510_16172_b200 as fp
from paper_2510_16172_b200 import _lib, datagen
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve
from oracle import fermat_oracle as O

from parity import (GRAD_REL, agreement_floor, converged_mask, flat_grad, golden, grad_rel_err,
                    lengths_ok, points_ok)

pytestmark = pytest.mark.gpu


def _solve(d, dtype, iters=None, fp_iters=None, T0=None, **kw):
    sc = BatchScene(d["basis"], d["anchor"], d["start"], d["end"])
    prec = Precision.SINGLE if dtype == np.float32 else Precision.DOUBLE
    opts = SolveOptions(iterations=int(iters if iters is not None else d["iterations"]),
                        fixed_point_iters=int(fp_iters if fp_iters is not None else d["fp_iters"]),
                        precision=prec, **kw)
    res = solve(sc, d["T0"] if T0 is None else T0, opts)
    torch.cuda.synchronize()
    return res


def _check_against(res, T_ref, L_ref, basis, anchor, start, end, min_agree):
    """Converged paths in tolerance; unconverged ones agree at least as often
    as the reference agrees with itself under a 1-ulp input change
    (min_agree: parity.agreement_floor on the same inputs)."""
    T = res.T.cpu().numpy()
    pts = res.points.double().cpu().numpy()
    L = res.length.cpu().numpy()
    f = np.float64
    ref_pts = O.path_points(basis.astype(f), anchor.astype(f), start.astype(f), end.astype(f),
                            T_ref.astype(f))[:, 1:-1]
    conv = converged_mask(basis, anchor, start, end, T_ref)
    ok = points_ok(pts, ref_pts) & lengths_ok(L, L_ref)
    assert conv.any()
    assert ok[conv].all(), f"{(~ok[conv]).sum()} converged paths out of tolerance"
    if (~conv).any():
        print(f"unconverged agreement {ok[~conv].mean():.4f} (floor {min_agree:.4f}, {(~conv).sum()} paths)")
        assert ok[~conv].mean() >= min_agree, (ok[~conv].mean(), min_agree)
    return conv, ok


def _floor(d, dt, T0=None, iters=None, fp_iters=None):
    return agreement_floor(d["basis"], d["anchor"], d["start"], d["end"], d["T0"] if T0 is None else T0,
                           int(iters if iters is not None else d["iterations"]),
                           int(fp_iters if fp_iters is not None else d["fp_iters"]), dt)


def test_config0_matches_reference():
    d = golden("fwd_config0")
    res = _solve(d, np.float32)
    conv, ok = _check_against(res, d["T"], d["L"], d["basis"], d["anchor"], d["start"], d["end"],
                              _floor(d, np.float32))
    # device gate agrees with the oracle classification on the clear cases
    dev_conv = res.converged.cpu().numpy()
    assert (dev_conv[conv]).mean() > 0.99


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_mixed_orderings_fp32(K):
    d = golden(f"fwd_mixed_k{K}")
    res = _solve(d, np.float32)
    _check_against(res, d["T_f32"], d["L_f32"], d["basis"], d["anchor"], d["start"], d["end"],
                   _floor(d, np.float32))


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_mixed_orderings_fp64(K):
    d = golden(f"fwd_mixed_k{K}")
    res = _solve(d, np.float64)
    _check_against(res, d["T_f64"], d["L_f64"], d["basis"], d["anchor"], d["start"], d["end"],
                   _floor(d, np.float64))
    # fp64 on converged paths is far tighter than the fp32 contract
    conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T_f64"])
    T = res.T.cpu().numpy()
    assert np.abs(T - d["T_f64"])[conv].max() < 1e-8


@pytest.mark.parametrize("kinds", ["reflections", "diffractions", "mixed"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_reference_generator_scenes(kinds, n):
    """Reference gen_scenes + init_params start, F=4, 50 iterations, both precisions."""
    d = golden(f"refgen_{kinds}_n{n}")
    for dt, suf in ((np.float64, "_f64"), (np.float32, "_f32")):
        res = _solve(d, dt)
        T = res.T.cpu().numpy()
        _check_against(res, d["T" + suf], d["L" + suf], d["basis"], d["anchor"], d["start"],
                       d["end"], _floor(d, dt))
        if kinds == "diffractions":
            # inert coordinates come back bitwise untouched (test_acceptance.py:120-134)
            assert np.array_equal(T[..., 1], d["T0"][..., 1].astype(dt))


def test_trace_matches_reference():
    d = golden("fwd_trace")
    res = _solve(d, np.float32, record_trace=True)
    tl = res.trace_len.cpu().numpy()
    tg = res.trace_gnorm.cpu().numpy()
    assert tl.shape == d["trace_len"].shape
    conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T"])
    # lengths are smooth in T: compare per iteration on converged paths
    rel = np.abs(tl - d["trace_len"]) / d["trace_len"]
    assert np.all(rel[:, conv] < 1e-5)
    # gradient norms agree to fp32 rounding of the gradient itself
    assert np.all(np.abs(tg - d["trace_gnorm"])[:, conv] < 1e-5 * (1 + d["trace_len"][:, conv]))


def test_known_answers():
    d = golden("known_answers")
    spec = fp.PathSpec(start=d["vpath_start"], end=d["vpath_end"],
                       surfaces=(fp.make_plane(d["vpath_anchor"][0], d["vpath_basis"][0][:, 0],
                                               d["vpath_basis"][0][:, 1]),))
    rep = fp.bfgs_solve(spec, d["vpath_T0"])
    assert rep.final_length == pytest.approx(2.0, abs=1e-9)
    assert rep.final_grad_norm < 1e-9
    assert np.allclose(rep.solution, d["vpath_T"], atol=1e-12)
    a = fp.line_search_alpha(spec, np.array([[0.0, 2.0]]), np.array([[0.0, -1.0]]), k=1)
    assert a == pytest.approx(float(d["linesearch_alpha"]), abs=1e-12)
    assert a == pytest.approx(2.0, abs=1e-12)
    with pytest.raises(fp.ZeroDirection):
        fp.line_search_alpha(spec, np.array([[0.0, 2.0]]), np.zeros((1, 2)))


@pytest.mark.parametrize("prec", [Precision.SINGLE, Precision.DOUBLE])
def test_batch_invariance_bitwise(prec):
    """Results per path do not depend on batch size, order or alignment,
    in fp32 and in fp64 (a permuted batch is a scattered layout: bucketed dispatch)."""
    b = datagen.gen_batch(7, datagen.all_orderings(3), 300)  # 2400 rows: ragged last CTA
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    opts = SolveOptions(iterations=20, precision=prec)
    full = solve(sc, b.T0, opts)
    perm = np.random.default_rng(0).permutation(b.size)
    scp = BatchScene(b.basis[perm], b.anchor[perm], b.start[perm], b.end[perm])
    permuted = solve(scp, b.T0[perm], opts)
    assert torch.equal(full.T[perm], permuted.T)
    assert torch.equal(full.length[perm], permuted.length)
    assert torch.equal(full.status[perm], permuted.status)
    # an odd offset breaks 16-byte alignment: the non-TMA staging path must agree
    sub = solve(sc.slice(1, 1 + 517), full.T.new_tensor(b.T0[1:518]), opts)
    assert torch.equal(full.T[1:518], sub.T)
    assert torch.equal(full.points[1:518], sub.points)
    one = solve(sc.slice(5, 6), full.T.new_tensor(b.T0[5:6]), opts)
    assert torch.equal(full.T[5:6], one.T)


def test_batch_solve_matches_scalar_bitwise():
    d = golden("refgen_mixed_n3")
    specs = _specs(d)
    opts = SolveOptions(iterations=50, fixed_point_iters=4)
    reps = fp.batch_solve(specs, list(d["T0"]), opts)
    for spec, T0, br in zip(specs, d["T0"], reps):
        sr = fp.bfgs_solve(spec, T0, opts)
        assert np.array_equal(sr.solution, br.solution)


def test_inert_coordinates_never_move():
    b = datagen.gen_batch(3, ["DDD", "RDR", "DRD"], 200)
    T0 = b.T0.copy()
    edge = np.all(b.basis[..., 1] == 0, axis=-1)
    noise = np.random.default_rng(1).normal(size=T0[..., 1].shape).astype(np.float32) * 10
    T0[..., 1] = np.where(edge, noise, 0.0)  # scramble inert coordinates only
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    res = solve(sc, T0, SolveOptions(iterations=20, precision=Precision.SINGLE))
    T = res.T.cpu().numpy()
    assert np.array_equal(T[..., 1][edge], T0[..., 1][edge])
    ref = solve(sc, b.T0, SolveOptions(iterations=20, precision=Precision.SINGLE)).T.cpu().numpy()
    assert np.array_equal(T[..., 0], ref[..., 0])


def test_edge_cases_empty_order0_and_errors():
    sc = BatchScene(np.zeros((0, 2, 3, 2), np.float32), np.zeros((0, 2, 3), np.float32),
                    np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32))
    res = solve(sc, None, SolveOptions(iterations=3, precision=Precision.SINGLE))
    assert res.T.shape == (0, 2, 2)
    x0 = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 2.0]])
    x1 = np.array([[3.0, 4.0, 0.0], [1.0, 2.0, 3.0]])
    sc0 = BatchScene(np.zeros((2, 0, 3, 2)), np.zeros((2, 0, 3)), x0, x1)
    r0 = solve(sc0, None, SolveOptions(iterations=3))
    assert np.allclose(r0.length.cpu().numpy(), [5.0, 1.0])
    # order 0 with record_trace: empty per-path traces like the reference
    # (solver.py:160-164), also through the scalar grad_tol early stop
    from paper_2510_16172_b200.solver import _bfgs_kernel
    T, g, traces = _bfgs_kernel(sc0, np.zeros((2, 0, 2)), SolveOptions(iterations=3, record_trace=True))
    assert T.shape == (2, 0, 2) and g.shape == (2, 0, 2) and traces == [[], []]
    spec0 = fp.PathSpec(start=x0[0], end=x1[0], surfaces=())
    rep = fp.bfgs_solve(spec0, np.zeros((0, 2)), SolveOptions(iterations=3, record_trace=True, grad_tol=1e-6))
    assert rep.trace == [] and rep.final_length == pytest.approx(5.0)
    big = datagen.gen_batch(1, ["R" * 65], 4)  # above MAX_INTERACTIONS (geometry.py:23)
    with pytest.raises(NotImplementedError):
        solve(BatchScene(big.basis, big.anchor, big.start, big.end), big.T0, SolveOptions(iterations=2))
    # degenerate entry: plane through the start point (test_objective.py:46-55)
    spec = fp.PathSpec(start=[0.0, 0.0, 0.0], end=[0.0, 0.0, 2.0],
                       surfaces=(fp.make_plane([0.0, 0.0, 0.0], [1, 0, 0], [0, 1, 0]),))
    with pytest.raises(fp.DegenerateSegment):
        fp.bfgs_solve(spec, np.zeros((1, 2)))


def _specs(d):
    specs = []
    for b in range(d["start"].shape[0]):
        surfs = []
        for i in range(d["basis"].shape[1]):
            A = d["basis"][b, i]
            if np.all(A[:, 1] == 0):
                surfs.append(fp.make_edge(d["anchor"][b, i], A[:, 0]))
            else:
                surfs.append(fp.make_plane(d["anchor"][b, i], A[:, 0], A[:, 1]))
        specs.append(fp.PathSpec(start=d["start"][b], end=d["end"][b], surfaces=tuple(surfs)))
    return specs


def test_init_params_matches_reference():
    d = golden("refgen_mixed_n4")
    specs = _specs(d)
    for spec, T0 in zip(specs, d["T0"]):
        assert np.allclose(fp.init_params(spec), T0, atol=1e-12)


def test_launch_counter_advances():
    before = _lib.launch_count()
    b = datagen.config0(256)
    solve(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0,
          SolveOptions(iterations=10, precision=Precision.SINGLE))
    torch.cuda.synchronize()
    assert _lib.launch_count() >= before + 1


@pytest.mark.parametrize("K", [2, 3, 5])
def test_specialised_kernels_match_dense(K):
    """Kind-mask specialised kernels (bucketed dispatch) agree with the uniform 2K kernel.

    Both compute the same IEEE operations per coordinate, but the specialised
    kernels pair the compressed unknowns for FFMA2 differently from the 2K
    layout, so reductions associate differently: agreement is to rounding on
    converged paths (the parity contract), not bitwise. Inert coordinates and
    the dense kernel's own determinism stay bitwise (other tests).
    """
    from paper_2510_16172_b200.solver import solve_with_gradients

    b = datagen.interleave(datagen.gen_batch(21, datagen.all_orderings(K), 97), seed=K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    opts = SolveOptions(iterations=20, precision=Precision.SINGLE, record_trace=True)
    try:
        _lib.set_kernel_policy("dense")
        dense = solve(sc, b.T0, opts)
        dres, dgrad = solve_with_gradients(sc, b.T0, SolveOptions(iterations=20, precision=Precision.SINGLE))
        _lib.set_kernel_policy("auto")
        spec = solve(sc, b.T0, opts)
        sres, sgrad = solve_with_gradients(sc, b.T0, SolveOptions(iterations=20, precision=Precision.SINGLE))
    finally:
        _lib.set_kernel_policy("auto")
    T = dense.T.double().cpu().numpy()
    conv = converged_mask(b.basis, b.anchor, b.start, b.end, T)
    assert conv.mean() > 0.05  # K=5 mixed: ~0.13 at 20 iterations (SURVEY.md key fact 4)
    assert points_ok(spec.points.cpu().numpy()[conv], dense.points.double().cpu().numpy()[conv]).all()
    assert lengths_ok(spec.length.cpu().numpy()[conv], dense.length.double().cpu().numpy()[conv]).all()
    st_d, st_s = dense.status.cpu().numpy(), spec.status.cpu().numpy()
    assert np.mean(st_d[conv] == st_s[conv]) > 0.99
    gd = flat_grad(*(x.double().cpu().numpy() for x in (dgrad.basis, dgrad.anchor, dgrad.start, dgrad.end)))
    gs = flat_grad(*(x.double().cpu().numpy() for x in (sgrad.basis, sgrad.anchor, sgrad.start, sgrad.end)))
    both = conv & (dres.status.cpu().numpy() == 0) & (sres.status.cpu().numpy() == 0)
    assert grad_rel_err(gs[both], gd[both]).max() < GRAD_REL
    # unconverged paths: most still land on the same answer
    agree = points_ok(spec.points.cpu().numpy(), dense.points.double().cpu().numpy())
    assert agree.mean() > 0.8


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("layout", ["ordered", "interleaved"])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_tile_and_bucketed_dispatch_bitwise_equal(K, layout, prec):
    """Every non-dense policy runs each path through its own kind-mask variant:
    the tile kernel (per-warp dispatch, mixed warps diverge) and the bucketed
    path (fp32: per-mask kernels; fp64: the tile kernel over a mask-sorted
    permutation) give the same bits, for ordering-major and scattered layouts
    (include/fermat_b200.h, FP_POLICY_*), so results never depend on the
    policy's layout history."""
    from paper_2510_16172_b200.solver import solve_with_gradients

    b = datagen.gen_batch(40 + K, datagen.all_orderings(K), 300)
    if layout == "interleaved":
        b = datagen.interleave(b, seed=K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    opts = SolveOptions(iterations=20, precision=Precision.SINGLE if prec == "single" else Precision.DOUBLE)
    out = {}
    try:
        for pol in ("tile", "bucket", "serial", "auto"):
            _lib.set_kernel_policy(pol)
            res, grads = solve_with_gradients(sc, b.T0, opts)
            fwd = solve(sc, b.T0, opts)
            out[pol] = (res, grads, fwd)
    finally:
        _lib.set_kernel_policy("auto")
    ref_res, ref_g, ref_f = out["bucket"]
    for pol, (res, grads, fwd) in out.items():
        for x, y in ((res.T, ref_res.T), (res.points, ref_res.points), (res.length, ref_res.length),
                     (res.status, ref_res.status), (grads.basis, ref_g.basis), (grads.anchor, ref_g.anchor),
                     (grads.start, ref_g.start), (grads.end, ref_g.end), (fwd.T, ref_f.T),
                     (fwd.g, ref_f.g), (fwd.points, ref_f.points), (fwd.status, ref_f.status)):
            assert torch.equal(x, y), pol


@pytest.mark.parametrize("prec", [Precision.SINGLE, Precision.DOUBLE])
def test_repeat_runs_bitwise_identical(prec):
    """Every order 1..8: two runs of the fused step on the same inputs return
    the same bits in every output (no read of an undefined register lane or
    of stale shared memory can go unnoticed)."""
    from paper_2510_16172_b200.solver import solve_with_gradients

    for K in range(1, 9):
        orders = datagen.all_orderings(K) if K <= 5 else datagen.all_orderings(K)[:8]
        b = datagen.gen_batch(700 + K, orders, 4096 // len(orders))
        sc = BatchScene(b.basis, b.anchor, b.start, b.end)
        opts = SolveOptions(iterations=20, precision=prec)
        runs = [solve_with_gradients(sc, b.T0, opts) for _ in range(2)]
        (r1, g1), (r2, g2) = runs
        for x, y in ((r1.T, r2.T), (r1.length, r2.length), (r1.status, r2.status), (r1.points, r2.points),
                     (g1.basis, g2.basis), (g1.anchor, g2.anchor), (g1.start, g2.start), (g1.end, g2.end)):
            assert torch.equal(x.view(torch.uint8), y.view(torch.uint8)), K

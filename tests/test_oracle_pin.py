"""Pin the CPU oracle against the reference's golden vectors (no GPU).

tests/golden/*.npz were produced by tests/golden/make_golden.py, which runs
the reference package itself. The numpy restatement reproduces it bit for
bit in the same numpy build; across numpy builds a tight tolerance applies.
"""

import numpy as np
import pytest

from oracle import fermat_oracle as O

from parity import converged_mask, golden

SAME_NUMPY = None


def _same_numpy(d):
    return str(d["numpy_version"]) == np.__version__


def _eq(a, b, exact):
    if exact:
        return np.array_equal(a, b, equal_nan=True)
    return np.allclose(a, b, rtol=1e-6, atol=1e-7, equal_nan=True)


def test_config0_forward():
    d = golden("fwd_config0")
    r = O.solve_outputs(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], 10, 1, np.float32)
    ex = _same_numpy(d)
    conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T"])
    if ex:
        for k in ("T", "g", "L", "points"):
            assert np.array_equal(r[k], d[k]), k
    else:
        assert np.allclose(r["T"][conv], d["T"][conv], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_mixed_forward_both_precisions(K):
    d = golden(f"fwd_mixed_k{K}")
    ex = _same_numpy(d)
    for dt, suf in ((np.float32, "_f32"), (np.float64, "_f64")):
        r = O.bfgs(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], 20, 1, dt, return_H=True)
        conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T" + suf])
        if ex:
            assert np.array_equal(r["T"], d["T" + suf])
            assert np.array_equal(r["g"], d["g" + suf])
            assert np.array_equal(r["H"], d["H" + suf])
        else:
            assert np.allclose(r["T"][conv], d["T" + suf][conv], rtol=1e-5, atol=1e-5)


def test_trace_forward():
    d = golden("fwd_trace")
    r = O.bfgs(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], 20, 2, np.float32, trace=True)
    assert _eq(r["trace_len"], d["trace_len"], _same_numpy(d))
    assert _eq(r["trace_gnorm"], d["trace_gnorm"], _same_numpy(d))


@pytest.mark.parametrize("kinds", ["reflections", "diffractions", "mixed"])
@pytest.mark.parametrize("n", [1, 3, 5])
def test_reference_generator_forward(kinds, n):
    d = golden(f"refgen_{kinds}_n{n}")
    ex = _same_numpy(d)
    for dt, suf in ((np.float64, "_f64"), (np.float32, "_f32")):
        r = O.solve_outputs(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], 50, 4, dt)
        for k in ("T", "g", "L"):
            assert _eq(r[k], d[k + suf], ex), (k, suf)


@pytest.mark.parametrize("K", [1, 2, 3])
def test_implicit_gradients(K):
    d = golden(f"fwd_mixed_k{K}")
    rows = np.arange(d["T_f32"].shape[0])[:40]
    db, da, d0, d1, ok = O.full_gradient_rows(d["basis"], d["anchor"], d["start"], d["end"],
                                              d["T_f32"], rows)
    assert np.array_equal(ok, d["grad_stationary"][rows])
    for name, arr in (("basis", db), ("anchor", da), ("start", d0), ("end", d1)):
        assert _eq(arr[ok], d["grad_full_" + name][rows][ok], _same_numpy(d))


@pytest.mark.parametrize("kinds", ["reflections", "mixed"])
def test_scalar_pieces_at_reference_optimum(kinds):
    d = golden(f"refgen_{kinds}_n3")
    ex = _same_numpy(d)
    for j in range(d["Tref"].shape[0]):
        args = (d["basis"][j], d["anchor"][j], d["start"][j], d["end"][j], d["Tref"][j])
        if not d["grad_stationary"][j]:
            continue
        env = O.envelope_gradient(*args)
        assert _eq(O.flat(env), np.concatenate([d["grad_env_basis"][j].ravel(),
                                                 d["grad_env_anchor"][j].ravel(),
                                                 d["grad_env_start"][j], d["grad_env_end"][j]]), ex)
        u = O.stationary_solve(*args, d["grad_v"][j])
        assert _eq(u, d["grad_u"][j], ex)
        assert _eq(O.scalar_hessian(*args), d["grad_hess"][j], ex)


def test_known_answers():
    d = golden("known_answers")
    a = O.line_search(d["vpath_basis"], d["vpath_anchor"], d["vpath_start"], d["vpath_end"],
                      np.array([[0.0, 2.0]]), np.array([[0.0, -1.0]]), k=1)
    assert a == float(d["linesearch_alpha"]) == pytest.approx(2.0, abs=1e-12)
    r = O.bfgs(d["vpath_basis"][None], d["vpath_anchor"][None], d["vpath_start"][None],
               d["vpath_end"][None], d["vpath_T0"][None], 100, 1, np.float64)
    assert np.allclose(r["T"][0], d["vpath_T"], atol=1e-14)


def test_init_guess():
    d = golden("refgen_mixed_n4")
    for j in range(d["T0"].shape[0]):
        assert np.allclose(O.init_guess(d["basis"][j], d["anchor"][j], d["start"][j], d["end"][j]),
                           d["T0"][j], atol=1e-13)


def test_degenerate_entry_raises():
    basis = np.array([[[[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]]]])
    with pytest.raises(O.OracleDegenerate):
        O.bfgs(basis, np.zeros((1, 1, 3)), np.zeros((1, 3)), np.array([[0.0, 0.0, 2.0]]),
               np.zeros((1, 1, 2)), 3, 1, np.float64)


@pytest.mark.parametrize("K", [1, 2, 3])
def test_newton_config1(K):
    d = golden(f"config1_k{K}")
    for it in (5, 10, 20):
        r = O.newton(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], it, np.float32)
        assert _eq(r["T"], d[f"newton_T_{it}"], _same_numpy(d))
        assert _eq(r["g"], d[f"newton_g_{it}"], _same_numpy(d))


@pytest.mark.parametrize("kinds", ["reflections", "diffractions", "mixed"])
def test_newton_and_image_reference_scenes(kinds):
    for n in (1, 3, 5):
        d = golden(f"refgen_{kinds}_n{n}")
        r = O.newton(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], 10, np.float64)
        assert _eq(r["T"], d["newton_T_f64"], _same_numpy(d))
        if kinds == "reflections":
            pts, par = O.image_points(d["basis"], d["anchor"], d["start"], d["end"])
            assert not par.any()
            assert _eq(pts, d["image_points"], _same_numpy(d))


def test_enumeration_oracle_self_consistent():
    from oracle import enumerate_oracle as E
    kinds = np.array([True, True, False, True, False])
    planes, edges = np.nonzero(kinds)[0], np.nonzero(~kinds)[0]
    for order in (1, 2, 3):
        got = set()
        for p in E.patterns(order):
            seqs = E.pattern_sequences(planes, edges, order, p)
            assert len({tuple(s) for s in seqs}) == len(seqs)
            assert all(kinds[s[j]] == bool((p >> j) & 1) for s in seqs for j in range(order))
            got |= {tuple(s) for s in seqs}
        assert got == E.brute_force_sequences(kinds, order)
        assert len(got) == len(kinds) * (len(kinds) - 1) ** (order - 1)


@pytest.mark.parametrize("K", [9, 16, 64])
def test_wide_orders_forward(K):
    """Orders 9..64 (geometry.py:23 MAX_INTERACTIONS): the oracle restatement
    reproduces the reference there too."""
    d = golden(f"fwd_wide_k{K}")
    ex = _same_numpy(d)
    for dt, suf in ((np.float32, "_f32"), (np.float64, "_f64")):
        r = O.bfgs(d["basis"], d["anchor"], d["start"], d["end"], d["T0"], int(d["iterations"]), 1, dt)
        conv = converged_mask(d["basis"], d["anchor"], d["start"], d["end"], d["T" + suf])
        assert conv.sum() >= 4
        if ex:
            assert np.array_equal(r["T"], d["T" + suf])
            assert np.array_equal(r["g"], d["g" + suf])
        else:
            assert np.allclose(r["T"][conv], d["T" + suf][conv], rtol=1e-5, atol=1e-5)


def test_near_singular_fallback():
    """_solve_sym's residual-check Tikhonov fallback (implicit_diff.py:55-71):
    the oracle reproduces the reference's u bit for bit on grazing
    reflections with cond(H) from 1e4 to 1e11, and where the fallback fired
    (cond >= 1e10) its u differs from the plain LAPACK solution."""
    d = golden("near_singular_k1")
    assert d["fired"].sum() >= 3 and (~d["fired"]).sum() >= 3
    for j in range(len(d["fired"])):
        args = (d["basis"][j], d["anchor"][j], d["start"][j], d["end"][j], d["T"][j])
        u = O.stationary_solve(*args, d["v"][j])
        assert np.array_equal(u, d["u"][j]), j
        H = O.scalar_hessian(*args)
        plain = np.linalg.solve(H, -d["v"][j].ravel())
        gap = np.linalg.norm(u.ravel() - plain) / np.linalg.norm(plain)
        assert (gap > 1e-3) == bool(d["fired"][j]), (j, gap)


def test_installed_reference_agrees_with_the_port():
    """bench.py --impl reference times the genuine reference from oracle/_ref
    (oracle/build_ref.py); on the same sample its forward solve equals the
    numpy port bit for bit, and the per-path gradient gate accepts the same
    paths."""
    import sys

    from oracle.cpu_baseline import REF_DIR, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not installed (python oracle/build_ref.py)")
    sys.path.insert(0, REF_DIR)
    try:
        from fermatpath.batching import BatchScene
        from fermatpath.solver import Precision, SolveOptions, _bfgs_kernel
    finally:
        sys.path.remove(REF_DIR)
    from paper_2510_16172_b200 import datagen

    b = datagen.config2(3, 256)
    T, g, _ = _bfgs_kernel(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0,
                           SolveOptions(iterations=20, precision=Precision.SINGLE))
    r = O.bfgs(b.basis, b.anchor, b.start, b.end, b.T0, 20, 1, np.float32)
    assert np.array_equal(T, r["T"]) and np.array_equal(g, r["g"])

"""The reference's BFGS guard rails on the GPU, update by update.

solver.py:180-199 skips an inverse-Hessian update when the curvature test
s.y > 1e-12 |s| |y| fails or when H' is not finite; solver.py:100,110-111
keeps alpha on a zero direction. The kernels reproduce these with cheaper
tests (an ALU-pipe magnitude bound on H' that falls back to a per-entry
check, fp_path.cuh InvHess::step), so this file compares the FATE of every
update — `trace_fate` (FP_FATE_* bits) against the oracle's masks
(oracle/fermat_oracle.bfgs, pinned to the reference) — in the regimes that
exercise each branch:

- a stationary start (g = 0 exactly): every update is a zero-direction
  curvature skip, T never moves;
- long runs past convergence (s, y at the rounding floor): curvature skips
  on most updates;
- basis columns scaled to 1e-3 and scenes to 1e17 m: the inverse Hessian
  grows past 1e26 and t-space steps past 1e18; the reference's intermediates
  overflow on some updates, which it skips — the kernel flags them and checks
  every entry in the reference's order (FP_FATE_ENTRY_CHECK), skipping the
  same ones;
- NaN / Inf inputs: the affected rows go non-finite exactly where the
  oracle's do, and never disturb the other rows.

Fates are compared on DECISIVE updates — while the path is still far from
converged — because past convergence s and y are rounding noise and the
curvature test is a coin toss in any arithmetic.
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200 import _lib, datagen
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.geometry import PathSpec, make_edge, make_plane
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve
from oracle import fermat_oracle as O

from parity import converged_mask, points_ok

pytestmark = pytest.mark.gpu

FATE = _lib.FATE_CURVATURE_SKIP | _lib.FATE_NONFINITE_SKIP | _lib.FATE_ZERO_DIRECTION


def _run(b, iters, dtype, scale=1.0):
    sc = BatchScene(b.basis, b.anchor * scale, b.start * scale, b.end * scale)
    prec = Precision.SINGLE if dtype == np.float32 else Precision.DOUBLE
    res = solve(sc, b.T0, SolveOptions(iterations=iters, precision=prec, record_trace=True),
                return_state=True)
    with np.errstate(all="ignore"):
        ref = O.bfgs(b.basis, b.anchor * scale, b.start * scale, b.end * scale, b.T0, iters, 1, dtype,
                     trace=True, return_H=True)
    return res, ref


def _agreement(res, ref):
    f = res.trace_fate.cpu().numpy()
    return (f & FATE) == ref["trace_fate"], f


def test_stationary_start_skips_every_update():
    """T0 at the exact optimum of symmetric V paths (g = 0 exactly): zero
    direction and curvature skip on every update, T bitwise unchanged, H = I."""
    specs = []
    for h in (0.5, 1.0, 3.0):
        for kind in ("plane", "edge"):
            s = make_plane([0, 0, 0], [1, 0, 0], [0, 1, 0]) if kind == "plane" else \
                make_edge([0, 0, 0], [0, 1, 0])
            specs.append(PathSpec(start=[-2.0, 0.0, h], end=[2.0, 0.0, h], surfaces=(s,)))
    sc = BatchScene.from_specs(specs)
    T0 = np.zeros((len(specs), 1, 2))
    for prec, dt in ((Precision.SINGLE, np.float32), (Precision.DOUBLE, np.float64)):
        res = solve(sc, T0, SolveOptions(iterations=7, precision=prec, record_trace=True),
                    return_state=True)
        f = res.trace_fate.cpu().numpy()
        want = _lib.FATE_CURVATURE_SKIP | _lib.FATE_ZERO_DIRECTION
        assert (f == want).all(), f
        assert (res.T.cpu().numpy() == 0).all()
        assert np.array_equal(res.H.cpu().numpy(), np.broadcast_to(np.eye(2), (len(specs), 2, 2)))
        assert ((res.status.cpu().numpy() & _lib.STATUS_ZERO_DIRECTION) != 0).all()
        b = sc.astype(dt)
        ref = O.bfgs(b.basis.cpu().numpy(), b.anchor.cpu().numpy(), b.start.cpu().numpy(),
                     b.end.cpu().numpy(), T0, 7, 1, dt, trace=True)
        assert (ref["trace_fate"] == want).all()


def _decisive(ref):
    """Updates whose fate is decided by the path's curvature, not by rounding:
    the oracle's gradient after the update is still within a factor 1000 of
    its value after the first update (scale-free: the scaled scenes below
    have gradients of 1e-7). Once a path has converged, s and y are rounding
    noise and the curvature test is a coin toss in any arithmetic (the
    reference's fp32 self-agreement under a 1-ulp input change is 90-94%,
    SURVEY.md key fact 5)."""
    g = ref["trace_gnorm"]
    return g > 1e-3 * g[:1]


def _self_agreement(b, iters, dt, scale=1.0):
    """The reference's own fate agreement under a 1-ulp change of the inputs
    (start nudged to the next representable value): the floor any other
    arithmetic can be held to (90-94% for unconverged
    fp32 paths)."""
    start = np.nextafter(b.start.astype(dt) * dt(scale), np.asarray(np.inf, dt))
    with np.errstate(all="ignore"):
        ref = O.bfgs(b.basis, b.anchor * scale, b.start * scale, b.end * scale, b.T0, iters, 1, dt,
                     trace=True)
        pert = O.bfgs(b.basis, b.anchor * scale, start, b.end * scale, b.T0, iters, 1, dt, trace=True)
    dec = _decisive(ref)
    return float((ref["trace_fate"] == pert["trace_fate"])[dec].mean())


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("K,iters", [(1, 60), (2, 100), (3, 100)])
def test_update_fates_match_oracle(K, iters, prec):
    """Long runs: on every decisive update (_decisive) the fate — curvature
    skip, zero direction, or taken — agrees with the oracle's about as often
    as the reference agrees with itself under a 1-ulp input change: within
    0.2 percentage points in fp64, 1.5 in fp32 (the fp32 kernels differ from
    numpy by a few ulps per operation — paired summation order, refined
    MUFU reciprocals — a larger perturbation than one input ulp). The runs
    go far past convergence, so curvature skips are frequent overall."""
    dt = np.float32 if prec == "f32" else np.float64
    b = datagen.gen_batch(300 + K, datagen.all_orderings(K), 512 // 2 ** K)
    res, ref = _run(b, iters, dt)
    agree, f = _agreement(res, ref)
    dec = _decisive(ref)
    floor = _self_agreement(b, iters, dt)
    print(f"K={K} {prec}: decisive {dec.mean():.3f}, agreement {agree[dec].mean():.5f} "
          f"(reference self-agreement {floor:.5f}; all updates {agree.mean():.4f})")
    assert dec.sum() > 1000
    margin = 0.015 if dt == np.float32 else 0.002
    assert agree[dec].mean() >= floor - margin, (agree[dec].mean(), floor)
    assert ((f & _lib.FATE_CURVATURE_SKIP) != 0).mean() > 0.1
    T_ref = ref["T"]
    conv = converged_mask(b.basis, b.anchor, b.start, b.end, T_ref)
    pts = res.points.double().cpu().numpy()
    ref_pts = O.path_points(b.basis.astype(np.float64), b.anchor.astype(np.float64),
                            b.start.astype(np.float64), b.end.astype(np.float64),
                            T_ref.astype(np.float64))[:, 1:-1]
    assert points_ok(pts, ref_pts)[conv].all()


def test_huge_inverse_hessians_entry_check_and_overflow_skips():
    """Basis columns scaled by 1e-3..1e-4 and scenes by 1e16..1e17 m (segment
    norms stay below the fp32 range; no subnormal intermediates): the inverse
    Hessian approximation grows past 1e26 and the steps in t-space past
    1e18, so the reference's intermediates (s s^T, s (Hy)^T) overflow fp32 on
    some updates and it skips them (solver.py:196-199). The kernel's magnitude
    test flags those updates, evaluates the reference's expression entry by
    entry (FP_FATE_ENTRY_CHECK) and skips the same updates
    (FP_FATE_NONFINITE_SKIP). Decisive fates agree with the oracle at least
    as often as the reference with itself under a 1-ulp input change (less
    2 percentage points); T stays finite; H stays finite wherever the
    oracle's does."""
    checked = skips_dev = skips_ref = 0
    agree_n = agree_d = 0
    floors = []
    for K in (2, 3):
        for F, S in ((1e-3, 1e17), (1e-4, 1e16)):
            b = datagen.gen_batch(500 + K, datagen.all_orderings(K), 512 // 2 ** K)
            b.basis *= np.float32(F)
            res, ref = _run(b, 40, np.float32, scale=S)
            agree, f = _agreement(res, ref)
            dec = _decisive(ref)
            agree_n += int(agree[dec].sum())
            agree_d += int(dec.sum())
            floors.append(_self_agreement(b, 40, np.float32, scale=S))
            checked += int(((f & _lib.FATE_ENTRY_CHECK) != 0).sum())
            skips_dev += int(((f & _lib.FATE_NONFINITE_SKIP) != 0).sum())
            skips_ref += int(((ref["trace_fate"] & _lib.FATE_NONFINITE_SKIP) != 0).sum())
            assert np.isfinite(res.T.cpu().numpy()).all()
            H_fin_ref = np.isfinite(ref["H"]).all(axis=(1, 2))
            assert np.isfinite(res.H.cpu().numpy()).all(axis=(1, 2))[H_fin_ref].all()
    floor = float(np.mean(floors))
    print(f"entry checks {checked}, non-finite skips device {skips_dev} oracle {skips_ref}, "
          f"decisive agreement {agree_n / max(agree_d, 1):.4f} of {agree_d} "
          f"(reference self-agreement {floor:.4f})")
    assert checked >= 1 and skips_dev >= 1 and skips_ref >= 1
    assert agree_n >= (floor - 0.02) * agree_d


def test_long_paths_overflow_check_and_skips():
    """The long-path solver (orders 9..64, csrc/fp_wide.cu) in the same
    huge-H regime: its update runs the all-entries finite check only when a
    magnitude bound cannot exclude an overflow (FP_FATE_ENTRY_CHECK) and then
    skips exactly the updates whose H' has a non-finite entry. Decisive fates
    agree with the oracle at least as often as the reference with itself
    (less 2 points); T stays finite; H stays finite where the oracle's does."""
    checked = skips_dev = skips_ref = 0
    agree_n = agree_d = 0
    floors = []
    for K, orders in ((9, ["RDRRDRDDR", "RRRRRRRRR"]), (12, ["RRDRRDRRDRRD"])):
        for F, S in ((1e-3, 1e17), (1e-4, 1e16)):
            b = datagen.gen_batch(700 + K, orders, 96 // len(orders))
            b.basis *= np.float32(F)
            res, ref = _run(b, 40, np.float32, scale=S)
            agree, f = _agreement(res, ref)
            dec = _decisive(ref)
            agree_n += int(agree[dec].sum())
            agree_d += int(dec.sum())
            floors.append(_self_agreement(b, 40, np.float32, scale=S))
            checked += int(((f & _lib.FATE_ENTRY_CHECK) != 0).sum())
            skips_dev += int(((f & _lib.FATE_NONFINITE_SKIP) != 0).sum())
            skips_ref += int(((ref["trace_fate"] & _lib.FATE_NONFINITE_SKIP) != 0).sum())
            assert np.isfinite(res.T.cpu().numpy()).all()
            H_fin_ref = np.isfinite(ref["H"]).all(axis=(1, 2))
            assert np.isfinite(res.H.cpu().numpy()).all(axis=(1, 2))[H_fin_ref].all()
    floor = float(np.mean(floors))
    print(f"long paths: entry checks {checked}, non-finite skips device {skips_dev} oracle {skips_ref}, "
          f"decisive agreement {agree_n / max(agree_d, 1):.4f} of {agree_d} (self-agreement {floor:.4f})")
    assert checked >= 1 and skips_dev >= 1 and skips_ref >= 1
    assert agree_n >= (floor - 0.02) * agree_d


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_nonfinite_inputs_stay_in_their_rows(prec):
    """NaN / Inf in the basis, anchor, start or end of some rows: those rows
    end non-finite exactly where the oracle's do (FP_STATUS_NONFINITE set),
    and every other row is bitwise the result of the clean batch."""
    dt = np.float32 if prec == "f32" else np.float64
    K = 3
    b = datagen.gen_batch(77, datagen.all_orderings(K), 16)
    bad = {3: ("basis", np.nan), 17: ("anchor", np.inf), 40: ("start", -np.inf), 77: ("end", np.nan),
           90: ("basis", np.inf), 101: ("anchor", np.nan)}
    arrs = {k: getattr(b, k).astype(dt).copy() for k in ("basis", "anchor", "start", "end")}
    for row, (field, v) in bad.items():
        arrs[field][row].flat[1] = v
    prec_e = Precision.SINGLE if dt == np.float32 else Precision.DOUBLE
    opts = SolveOptions(iterations=20, precision=prec_e)
    clean = solve(BatchScene(*(getattr(b, k).astype(dt) for k in ("basis", "anchor", "start", "end"))),
                  b.T0, opts)
    dirty = solve(BatchScene(arrs["basis"], arrs["anchor"], arrs["start"], arrs["end"]), b.T0, opts)
    # the reference raises DegenerateSegment for a whole batch holding a
    # degenerate entry row (solver.py:166): run the oracle row by row, and
    # expect FP_STATUS_DEGENERATE_ENTRY (the batch-level raise) where it raises
    T_ref = np.empty((b.size, K, 2), dt)
    degen = np.zeros(b.size, bool)
    with np.errstate(all="ignore"):
        for r in range(b.size):
            try:
                T_ref[r] = O.bfgs(arrs["basis"][r:r + 1], arrs["anchor"][r:r + 1], arrs["start"][r:r + 1],
                                  arrs["end"][r:r + 1], b.T0[r:r + 1], 20, 1, dt)["T"][0]
            except O.OracleDegenerate:
                T_ref[r] = np.nan
                degen[r] = True
    rows = np.array(sorted(bad))
    keep = np.setdiff1d(np.arange(b.size), rows)
    T, Tc = dirty.T.cpu().numpy(), clean.T.cpu().numpy()
    assert np.array_equal(T[keep], Tc[keep])
    assert np.array_equal(dirty.status.cpu().numpy()[keep], clean.status.cpu().numpy()[keep])
    st_all = dirty.status.cpu().numpy()
    dev_degen = (st_all & _lib.STATUS_DEGENERATE_ENTRY) != 0
    assert np.array_equal(dev_degen, degen), [(int(r), int(st_all[r]), bool(degen[r]))
                                              for r in np.nonzero(dev_degen != degen)[0]]
    fin_dev = np.isfinite(T).all(axis=(1, 2))
    fin_ref = np.isfinite(T_ref).all(axis=(1, 2))
    assert np.array_equal(fin_dev[~degen], fin_ref[~degen])
    assert not fin_dev[rows].any()
    assert ((st_all[rows] & (_lib.STATUS_NONFINITE | _lib.STATUS_DEGENERATE_ENTRY)) != 0).all()
    assert not (st_all[keep] & _lib.STATUS_DEGENERATE_ENTRY).any()

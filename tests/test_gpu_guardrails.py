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
- scenes scaled to 1e17 m: the magnitude bound on H' passes 1e36 and the
  per-entry check runs (FP_FATE_ENTRY_CHECK);
- scenes scaled to 3e18 m: H' overflows fp32 and the update is skipped;
- NaN / Inf inputs: the affected rows go non-finite exactly where the
  oracle's do, and never disturb the other rows.

fp64 kernels round like the oracle's fp64 arithmetic to a few ulps, so their
fates must agree on (almost) every update; fp32 kernels use refined
MUFU reciprocals (<= 1 ulp), so trajectories that sit on a test threshold can
flip — agreement is measured and bounded per regime.
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


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("K,iters", [(1, 60), (2, 100), (3, 100)])
def test_update_fates_match_oracle(K, iters, prec):
    """Long runs: the fate of each update (curvature skip / zero direction)
    agrees with the oracle. fp64: >= 99.5% of all updates and >= 99.9% in
    the first 20. fp32: >= 97% and >= 99% (threshold-sitting paths can flip
    by one ulp); the counts of each kind agree within 3%."""
    dt = np.float32 if prec == "f32" else np.float64
    b = datagen.gen_batch(300 + K, datagen.all_orderings(K), 512 // 2 ** K)
    res, ref = _run(b, iters, dt)
    agree, f = _agreement(res, ref)
    lo_all, lo_early = (0.97, 0.99) if dt == np.float32 else (0.995, 0.999)
    assert agree.mean() >= lo_all, agree.mean()
    assert agree[:20].mean() >= lo_early, agree[:20].mean()
    for bit in (_lib.FATE_CURVATURE_SKIP, _lib.FATE_ZERO_DIRECTION):
        n_dev, n_ref = int(((f & bit) != 0).sum()), int(((ref["trace_fate"] & bit) != 0).sum())
        assert abs(n_dev - n_ref) <= 0.03 * max(n_ref, 100), (bit, n_dev, n_ref)
    # skips happen (the runs go far past convergence) and converged paths agree
    assert ((f & _lib.FATE_CURVATURE_SKIP) != 0).mean() > 0.2
    T_ref = ref["T"]
    conv = converged_mask(b.basis, b.anchor, b.start, b.end, T_ref)
    pts = res.points.double().cpu().numpy()
    ref_pts = O.path_points(b.basis.astype(np.float64), b.anchor.astype(np.float64),
                            b.start.astype(np.float64), b.end.astype(np.float64),
                            T_ref.astype(np.float64))[:, 1:-1]
    assert points_ok(pts, ref_pts)[conv].all()


def test_large_scene_exercises_the_entry_check():
    """A scene scaled by 1e17 m: the inverse Hessian grows past 1e27, the
    magnitude bound on H' crosses 1e36 and the kernel checks every entry
    (FP_FATE_ENTRY_CHECK); those updates are still taken exactly when the
    oracle takes them (the entries are finite), in both precisions."""
    K = 3
    b = datagen.gen_batch(303, datagen.all_orderings(K), 32)
    for dt in (np.float32, np.float64):
        res, ref = _run(b, 100, dt, scale=1e17)
        agree, f = _agreement(res, ref)
        checked = (f & _lib.FATE_ENTRY_CHECK) != 0
        if dt == np.float32:
            assert checked.sum() >= 10, int(checked.sum())
        assert agree[:20].mean() >= 0.99, agree[:20].mean()
        assert agree[checked].mean() >= 0.95 if checked.any() else True
        assert np.isfinite(res.T.cpu().numpy()).all() and np.isfinite(ref["T"]).all()


def test_overflowing_updates_are_skipped():
    """A scene scaled by 3e18 m (segment norms near the fp32 range): some
    fp32 updates produce a non-finite H' and are skipped, on the device as in
    the oracle; the inverse Hessian stays finite wherever the oracle's does,
    and T stays finite."""
    hits_dev = hits_ref = 0
    for K in (3, 4, 5):
        b = datagen.gen_batch(400 + K, datagen.all_orderings(K), 2048 // 2 ** K)
        res, ref = _run(b, 300, np.float32, scale=3e18)
        f = res.trace_fate.cpu().numpy()
        hits_dev += int(((f & _lib.FATE_NONFINITE_SKIP) != 0).sum())
        hits_ref += int(((ref["trace_fate"] & _lib.FATE_NONFINITE_SKIP) != 0).sum())
        H_fin_ref = np.isfinite(ref["H"]).all(axis=(1, 2))
        H_fin_dev = np.isfinite(res.H.cpu().numpy()).all(axis=(1, 2))
        assert H_fin_dev[H_fin_ref].all()
        agree, _ = _agreement(res, ref)
        assert agree[:20].mean() >= 0.99
    assert hits_ref >= 1 and hits_dev >= 1, (hits_dev, hits_ref)


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
    with np.errstate(all="ignore"):
        ref = O.bfgs(arrs["basis"], arrs["anchor"], arrs["start"], arrs["end"], b.T0, 20, 1, dt)
    rows = np.array(sorted(bad))
    keep = np.setdiff1d(np.arange(b.size), rows)
    T, Tc = dirty.T.cpu().numpy(), clean.T.cpu().numpy()
    assert np.array_equal(T[keep], Tc[keep])
    assert np.array_equal(dirty.status.cpu().numpy()[keep], clean.status.cpu().numpy()[keep])
    fin_dev = np.isfinite(T).all(axis=(1, 2))
    fin_ref = np.isfinite(ref["T"]).all(axis=(1, 2))
    assert np.array_equal(fin_dev, fin_ref)
    assert not fin_dev[rows].any()
    st = dirty.status.cpu().numpy()[rows]
    assert ((st & _lib.STATUS_NONFINITE) != 0).all()

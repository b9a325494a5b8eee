"""Config 3 on the REAL scene (BASELINE config 3: 16 buildings, 64 wall
reflectors, 32x32 RX grid, TX at 30 m) against the CPU oracle.

- orders 1 and 2, exhaustively (65,536 + 4,128,768 candidates): the traced
  valid set (converged and inside every wall, compacted by the fused
  enumeration kernel) against the oracle's valid set (the numpy BFGS of every
  candidate, fp64 gate recompute at its T, the same bounds rule);
- order 3, a 65,536-candidate random subsample of the 260M: the device
  solve + mask of the sampled candidates against the oracle.

Enumeration and the mask given T are integer / comparison work and bit-exact
(tests/test_gpu_enum.py). Valid-set disagreements come only from fp32
rounding moving a candidate across the stationarity gate or a wall boundary
(|t| = 1): the MASK FLIP RATE (symmetric difference / candidates) is
reported and bounded, and on the paths both sides call valid the interaction
points agree within the contract tolerance.
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200 import _lib
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.scene import make_urban_scene, pattern_count, trace
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve
from oracle import enumerate_oracle as E
from oracle import fermat_oracle as O
from oracle.cpu_baseline import bfgs_parallel

from parity import points_ok

pytestmark = pytest.mark.gpu

FLIP_MAX = 2e-4


@pytest.fixture(scope="module")
def city():
    return make_urban_scene(seed=0, alphabet="walls")


def _oracle_valid(basis, anchor, start, end, T, is_plane):
    """The device's validity rule restated: finite, |grad| < 1e-5 (1 + L)
    (fp64 recompute at T, implicit_diff.py:25,30-36), no segment <= eps
    (FP_STATUS_DEGENERATE_*), and |t| <= 1 on every active coordinate."""
    f = np.float64
    b, a, x0, x1, t = (np.asarray(z, f) for z in (basis, anchor, start, end, T))
    eps = O.seg_floor(x0, x1, f)
    with np.errstate(all="ignore"):
        s, n = O.seg_and_norm(O.path_points(b, a, x0, x1, t))
        u = s / np.maximum(n, eps[:, None])[..., None]
        g = np.einsum("bnij,bni->bnj", b, u[:, :-1] - u[:, 1:])
        gn = np.sqrt(np.einsum("bnj,bnj->b", g, g))
        L = n.sum(axis=1)
    fin = np.isfinite(t).all(axis=(1, 2)) & np.isfinite(L)
    conv = fin & (gn < 1e-5 * (1.0 + L)) & (n.min(axis=1) > eps)
    return conv & E.inside_bounds(T, is_plane)


def _candidates(city, order, pattern, rows=None):
    seqs = E.pattern_sequences(city.plane_ids, city.edge_ids, order, pattern)
    n_rx = city.rx.shape[0]
    c = np.arange(len(seqs) * n_rx) if rows is None else rows
    rx, seq = (c // len(seqs)).astype(np.int32), seqs[c % len(seqs)]
    basis = city.obj_basis[seq].astype(np.float32)
    anchor = city.obj_anchor[seq].astype(np.float32)
    start = np.broadcast_to(city.tx.astype(np.float32), (len(rx), 3)).copy()
    end = city.rx.astype(np.float32)[rx]
    return rx, seq, basis, anchor, start, end


def _keys(rx, seq):
    return {(int(r), *map(int, s)) for r, s in zip(rx, seq)}


@pytest.mark.parametrize("order", [1, 2])
def test_exhaustive_orders_against_oracle(city, order):
    res = trace(city, max_order=order, iterations=20)
    o = res.orders[order - 1]
    dev = _keys(o.rx.cpu().numpy(), o.seq.cpu().numpy())
    ref, total = set(), 0
    T_ref_by_key = {}
    for p in range(1 << order):
        if pattern_count(city, order, p) <= 0:
            continue
        rx, seq, basis, anchor, start, end = _candidates(city, order, p)
        total += len(rx)
        T = bfgs_parallel(basis, anchor, start, end, np.zeros((len(rx), order, 2), np.float32), 20)
        ok = _oracle_valid(basis, anchor, start, end, T, city.obj_plane[seq])
        idx = np.nonzero(ok)[0]
        ref |= _keys(rx[idx], seq[idx])
        T_ref_by_key.update({(int(rx[i]), *map(int, seq[i])): (T[i], basis[i], anchor[i], end[i])
                             for i in idx})
    assert total == o.candidates
    flips = len(ref ^ dev)
    rate = flips / total
    print(f"order {order}: {total} candidates, oracle valid {len(ref)}, device valid {len(dev)}, "
          f"flips {flips} (rate {rate:.2e})")
    assert ref, "no valid paths"
    assert rate <= FLIP_MAX, rate
    # interaction points of the paths both sides call valid
    key = {(int(r), *map(int, s)): i for i, (r, s) in enumerate(zip(o.rx.cpu().numpy(), o.seq.cpu().numpy()))}
    both = sorted(ref & dev)
    Tdev = o.T.cpu().numpy()
    rows = np.array([key[k] for k in both])
    Tr = np.stack([T_ref_by_key[k][0] for k in both]).astype(np.float64)
    Bs = np.stack([T_ref_by_key[k][1] for k in both]).astype(np.float64)
    As = np.stack([T_ref_by_key[k][2] for k in both]).astype(np.float64)
    Es = np.stack([T_ref_by_key[k][3] for k in both]).astype(np.float64)
    Ss = np.broadcast_to(city.tx.astype(np.float32).astype(np.float64), Es.shape)
    p_ref = O.path_points(Bs, As, Ss, Es, Tr)[:, 1:-1]
    p_dev = O.path_points(Bs, As, Ss, Es, Tdev[rows].astype(np.float64))[:, 1:-1]
    assert points_ok(p_dev, p_ref).all()


def test_order3_random_subsample_against_oracle(city):
    order = 3
    p = (1 << order) - 1  # the walls alphabet holds reflectors only
    n_all = pattern_count(city, order, p) * city.rx.shape[0]
    assert n_all > 2.5e8
    rows = np.sort(np.random.default_rng(33).choice(n_all, 1 << 16, replace=False))
    rx, seq, basis, anchor, start, end = _candidates(city, order, p, rows)
    sol = solve(BatchScene(basis, anchor, start, end), None,
                SolveOptions(iterations=20, precision=Precision.SINGLE))
    T_dev = sol.T.cpu().numpy()
    st = sol.status.cpu().numpy()
    dev = ((st & _lib.STATUS_UNCONVERGED_MASK) == 0) & E.inside_bounds(T_dev, city.obj_plane[seq])
    T_ref = bfgs_parallel(basis, anchor, start, end, np.zeros((len(rx), order, 2), np.float32), 20)
    ref = _oracle_valid(basis, anchor, start, end, T_ref, city.obj_plane[seq])
    rate = float((dev ^ ref).mean())
    print(f"order 3 subsample: {len(rows)} candidates, oracle valid {int(ref.sum())}, device valid "
          f"{int(dev.sum())}, flips {int((dev ^ ref).sum())} (rate {rate:.2e})")
    assert rate <= FLIP_MAX * 10, rate
    both = dev & ref
    f = np.float64
    args = (basis[both].astype(f), anchor[both].astype(f), start[both].astype(f), end[both].astype(f))
    assert points_ok(O.path_points(*args, T_dev[both].astype(f))[:, 1:-1],
                     O.path_points(*args, T_ref[both].astype(f))[:, 1:-1]).all()


def test_config4_gradient_on_the_real_scene(city):
    """Config 4 (the inverse-design step) on the real walls scene: loss =
    sum over valid paths of 1/L^2 and its gradient w.r.t. every wall object
    (full implicit VJP, cotangent -2/L^3, accumulated on the device), TX and
    the wall vertices, against the fp64 oracle gradient of every traced
    valid path (implicit_diff.py:74-106 restated) summed on the host. Within
    1e-3 relative (the north-star gradient tolerance), norm-wise."""
    from oracle.cpu_baseline import full_gradient_parallel

    res = trace(city, max_order=3, iterations=20, with_grad=True)
    N = city.n_objects
    obj_ref = np.zeros((N, 9))
    tx_ref = np.zeros(3)
    loss_ref = 0.0
    n_paths = 0
    for o in res.orders:
        if o.valid == 0:
            continue
        seq = o.seq.cpu().numpy()
        rxi = o.rx.cpu().numpy()
        T = o.T.cpu().numpy().astype(np.float64)
        L = o.length.cpu().numpy().astype(np.float64)
        basis = city.obj_basis[seq].astype(np.float32).astype(np.float64)
        anchor = city.obj_anchor[seq].astype(np.float32).astype(np.float64)
        start = np.broadcast_to(city.tx.astype(np.float32).astype(np.float64), (len(seq), 3)).copy()
        end = city.rx.astype(np.float32).astype(np.float64)[rxi]
        db, da, d0, d1, ok = full_gradient_parallel(basis, anchor, start, end, T, -2.0 / L ** 3)
        n_paths += int(ok.sum())
        loss_ref += float(np.sum(1.0 / L[ok] ** 2))
        # walls alphabet: reflectors only, every basis element is active
        np.add.at(obj_ref, seq[ok].ravel(), np.concatenate(
            [db[ok].reshape(-1, o.order, 6), da[ok]], axis=2).reshape(-1, 9))
        tx_ref += d0[ok].sum(axis=0)
    obj = res.obj_grad.cpu().numpy()
    rel = np.linalg.norm(obj - obj_ref) / np.linalg.norm(obj_ref)
    print(f"config 4 real scene: {n_paths} valid paths, loss {res.loss:.6e} (oracle {loss_ref:.6e}), "
          f"object-gradient rel err {rel:.2e}")
    assert n_paths > 10_000
    assert res.loss == pytest.approx(loss_ref, rel=1e-4)
    assert rel <= 1e-3
    assert np.linalg.norm(res.tx_grad.cpu().numpy() - tx_ref) <= 1e-3 * np.linalg.norm(tx_ref)

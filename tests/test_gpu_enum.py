"""GPU candidate enumeration / tracing (configs 3 and 4) against the CPU oracle.

Enumeration is integer work: bit-exact. The bounds mask is a pure function of
T: bit-exact given the same T (checked by solving the decoded candidates with
the batched solver, which computes bit-identical T). End-to-end validity and
gradients are compared with the numpy oracle within the stated tolerances.
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200 import _lib
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.scene import (candidate_count, decode_candidates, make_urban_scene,
                                         pattern_count, trace)
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve
from oracle import enumerate_oracle as E
from oracle import fermat_oracle as O

pytestmark = pytest.mark.gpu


def _small(alphabet="all", rx_grid=3, n_buildings=2, seed=3):
    return make_urban_scene(seed=seed, n_buildings=n_buildings, rx_grid=rx_grid, alphabet=alphabet,
                            side=80.0)


@pytest.mark.parametrize("order", [1, 2, 3])
def test_decode_bit_exact(order):
    sc = _small()
    all_seqs = set()
    for p in range(1 << order):
        rx, seq = decode_candidates(sc, order, p)
        rx_ref, seq_ref = E.pattern_candidates(sc.plane_ids, sc.edge_ids, sc.rx.shape[0], order, p)
        assert np.array_equal(rx.cpu().numpy(), rx_ref)
        assert np.array_equal(seq.cpu().numpy(), seq_ref)
        all_seqs |= {tuple(s) for s in seq_ref[: len(seq_ref) // sc.rx.shape[0]]}
    # union over kind patterns == every sequence without an immediate repeat
    assert all_seqs == E.brute_force_sequences(sc.obj_plane, order)


def test_candidate_counts():
    sc = make_urban_scene(seed=0)  # config 3: 16 buildings, 64 walls + 128 edges, 32x32 RX
    N, R = sc.n_objects, sc.rx.shape[0]
    assert N == 192 and R == 1024
    assert candidate_count(sc, 3) == R * (N + N * (N - 1) + N * (N - 1) ** 2)
    walls = make_urban_scene(seed=0, alphabet="walls")
    # the 64-object alphabet gives BASELINE's "~2.6e8 candidate paths"
    assert candidate_count(walls, 3) == 1024 * (64 + 64 * 63 + 64 * 63 * 63) == 264_306_688


def _candidates_all(sc, order):
    rows = []
    for p in range(1 << order):
        rx, seq = E.pattern_candidates(sc.plane_ids, sc.edge_ids, sc.rx.shape[0], order, p)
        rows.append((rx, seq))
    rx = np.concatenate([r for r, _ in rows])
    seq = np.concatenate([s for _, s in rows])
    basis = sc.obj_basis[seq]
    anchor = sc.obj_anchor[seq]
    start = np.broadcast_to(sc.tx.astype(np.float32), (len(rx), 3)).copy()
    end = sc.rx.astype(np.float32)[rx]
    return rx, seq, basis, anchor, start, end


@pytest.mark.parametrize("order", [1, 2, 3])
def test_trace_counts_and_mask_bit_exact(order):
    sc = _small()
    res = trace(sc, max_order=order, iterations=20)
    o = res.orders[order - 1]
    rx, seq, basis, anchor, start, end = _candidates_all(sc, order)
    assert o.candidates == len(rx)
    # same candidates through the batched solver: bit-identical T and status
    bs = BatchScene(basis, anchor, start, end)
    sol = solve(bs, None, SolveOptions(iterations=20, precision=Precision.SINGLE))
    st = sol.status.cpu().numpy()
    T = sol.T.cpu().numpy()
    conv = (st & _lib.STATUS_UNCONVERGED_MASK) == 0
    inb = E.inside_bounds(T, sc.obj_plane[seq])
    assert o.converged == int(conv.sum())
    assert o.in_bounds == int(inb.sum())
    assert o.valid == int((conv & inb).sum())
    # the compacted records are exactly the valid candidates, with their T and L
    key_dev = {(int(r), *map(int, s)): i for i, (r, s) in
               enumerate(zip(o.rx.cpu().numpy(), o.seq.cpu().numpy()))}
    valid_rows = np.nonzero(conv & inb)[0]
    assert {(int(rx[i]), *map(int, seq[i])) for i in valid_rows} == set(key_dev)
    Tdev, Ldev = o.T.cpu().numpy(), o.length.cpu().numpy()
    L = sol.length.cpu().numpy()
    for i in valid_rows[:500]:
        j = key_dev[(int(rx[i]), *map(int, seq[i]))]
        Ti = T[i].copy()
        Ti[~sc.obj_plane[seq[i]], 1] = 0.0
        assert np.array_equal(Tdev[j], Ti)
        assert Ldev[j] == L[i]


def test_trace_matches_oracle_solve():
    """End to end vs the numpy oracle: valid-set agreement and T on common paths."""
    sc = _small(rx_grid=2)
    order = 2
    res = trace(sc, max_order=order, iterations=20)
    o = res.orders[order - 1]
    rx, seq, basis, anchor, start, end = _candidates_all(sc, order)
    r = O.bfgs(basis, anchor, start, end, np.zeros((len(rx), order, 2), np.float32), 20, 1, np.float32)
    Tr = r["T"]
    from parity import converged_mask
    conv = converged_mask(basis, anchor, start, end, Tr)
    inb = E.inside_bounds(Tr, sc.obj_plane[seq])
    ref = {(int(rx[i]), *map(int, seq[i])) for i in np.nonzero(conv & inb)[0]}
    dev = {(int(a), *map(int, s)) for a, s in zip(o.rx.cpu().numpy(), o.seq.cpu().numpy())}
    assert ref, "no valid paths in the test scene"
    sym = len(ref ^ dev)
    assert sym <= max(2, 0.02 * len(ref)), (len(ref), len(dev), sym)


def test_scene_gradient_matches_oracle():
    """Config 4: loss = sum 1/L^2 over valid paths; full implicit VJP; vertex chain rule."""
    sc = _small(rx_grid=2)
    res = trace(sc, max_order=2, iterations=20, with_grad=True)
    N = sc.n_objects
    obj_ref = np.zeros((N, 9))
    tx_ref = np.zeros(3)
    loss_ref = 0.0
    for o in res.orders:
        if o.valid == 0:
            continue
        seq = o.seq.cpu().numpy()
        rxi = o.rx.cpu().numpy()
        T = o.T.cpu().numpy().astype(np.float64)
        L = o.length.cpu().numpy().astype(np.float64)
        basis = sc.obj_basis[seq].astype(np.float64)
        anchor = sc.obj_anchor[seq].astype(np.float64)
        start = np.broadcast_to(sc.tx.astype(np.float32).astype(np.float64), (len(seq), 3))
        end = sc.rx.astype(np.float32).astype(np.float64)[rxi]
        w = -2.0 / L ** 3
        db, da, d0, d1, ok = O.full_gradient_rows(basis, anchor, start, end, T, np.arange(len(seq)), w)
        loss_ref += float(np.sum(1.0 / L[ok] ** 2))
        for j in np.nonzero(ok)[0]:
            for i, obj in enumerate(seq[j]):
                obj_ref[obj, :6] += db[j, i].ravel() * ([1, 1] * 3 if sc.obj_plane[obj] else [1, 0] * 3)
                obj_ref[obj, 6:] += da[j, i]
            tx_ref += d0[j]
    obj = res.obj_grad.cpu().numpy()
    assert res.loss == pytest.approx(loss_ref, rel=1e-4)
    assert np.linalg.norm(obj - obj_ref) <= 1e-3 * np.linalg.norm(obj_ref)
    assert np.linalg.norm(res.tx_grad.cpu().numpy() - tx_ref) <= 1e-3 * np.linalg.norm(tx_ref)
    # vertex chain rule = coef^T applied to the object gradients
    vref = np.zeros((sc.walls.shape[0] * 4, 3))
    for n in range(N):
        dp = np.stack([obj_ref[n, 6:9], obj_ref[n, 0:6:2], obj_ref[n, 1:6:2]])  # anchor, col0, col1
        for v in range(4):
            vref[sc.vert_ids[n, v]] += sc.coef[n][:, v] @ dp
    vg = res.vertex_grad.cpu().numpy()
    assert np.linalg.norm(vg - vref) <= 1e-3 * np.linalg.norm(vref)


def test_rank_sharding_partitions_every_group():
    """Shards of a 3-rank job cover every candidate exactly once (counts add up)."""
    sc = _small(rx_grid=2)
    full = trace(sc, max_order=2, iterations=20, capacity=0)
    parts = [trace(sc, max_order=2, iterations=20, capacity=0, rank=r, world=3, allreduce=False)
             for r in range(3)]
    for k in range(2):
        for field in ("candidates", "converged", "in_bounds", "valid"):
            assert sum(getattr(p.orders[k], field) for p in parts) == getattr(full.orders[k], field)


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("exclude", [True, False])
def test_enumerate_candidates_bit_exact(order, exclude):
    """enumerate_candidates vs itertools: lexicographic, with and
    without the no-immediate-repeat predicate, whole list and a sub-range."""
    import itertools

    from paper_2510_16172_b200 import enumerate_candidates

    n = 7
    ref = np.array([s for s in itertools.product(range(n), repeat=order)
                    if not exclude or all(a != b for a, b in zip(s, s[1:]))], dtype=np.int32)
    got = enumerate_candidates(n, order, exclude_repeats=exclude).cpu().numpy()
    assert np.array_equal(got, ref.reshape(len(ref), order))
    lo, hi = len(ref) // 3, min(len(ref), len(ref) // 3 + 11)
    part = enumerate_candidates(n, order, exclude_repeats=exclude, begin=lo, end=hi).cpu().numpy()
    assert np.array_equal(part, ref[lo:hi].reshape(hi - lo, order))

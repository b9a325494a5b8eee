"""Full-size (BASELINE config 2, K=3, 2^22 paths) properties on the GPU.

The oracle cannot run 4M paths in seconds, so the full batch is checked
through size-independent properties plus an oracle subsample:
  * fused step == solve-then-VJP, bit for bit, on every path;
  * a random subset solved alone gives bit-identical results (per-path
    independence at full size);
  * translation invariance of the optimal length: for every converged path
    dL*/dstart + dL*/dend + sum_i dL*/danchor_i = 0 (test_implicit.py:95-101);
  * a 2048-path random subsample agrees with the numpy oracle (parity.py);
  * converged fraction in the range the survey measured (0.33 at K=3).
"""

import numpy as np
import pytest
import torch

from paper_2510_16172_b200 import _lib, datagen
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.implicit_diff import vjp_batch
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients
from oracle import fermat_oracle as O

from parity import GRAD_REL, agreement_floor, converged_mask, flat_grad, grad_rel_err, lengths_ok, points_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full():
    b = datagen.config2(3)  # 2^22 paths, 8 orderings
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    opts = SolveOptions(iterations=20, precision=Precision.SINGLE)
    res, grads = solve_with_gradients(sc, b.T0, opts, weight=1.0, mode="full")
    torch.cuda.synchronize()
    return b, sc, opts, res, grads


def test_fused_equals_separate_full_size(full):
    b, sc, opts, res, grads = full
    sep = solve(sc, b.T0, opts)
    assert torch.equal(res.T, sep.T) and torch.equal(res.length, sep.length)
    g2, st2, _ = vjp_batch(sc, sep.T, w_L=1.0, mode="full")
    # the fused status carries the solve bits and the VJP's (singular / non-finite)
    assert torch.equal(res.status, sep.status | st2)
    for x, y in ((grads.basis, g2.basis), (grads.anchor, g2.anchor), (grads.start, g2.start),
                 (grads.end, g2.end)):
        assert torch.equal(x, y)


def test_subset_bitwise_independent(full):
    b, sc, opts, _, _ = full
    whole = solve(sc, b.T0, opts)
    idx = np.sort(np.random.default_rng(5).choice(b.size, 100_000, replace=False))
    sub = solve(BatchScene(b.basis[idx], b.anchor[idx], b.start[idx], b.end[idx]), b.T0[idx], opts)
    it = torch.as_tensor(idx, device=whole.T.device)
    assert torch.equal(sub.T, whole.T[it]) and torch.equal(sub.status, whole.status[it])
    assert torch.equal(sub.points, whole.points[it]) and torch.equal(sub.g, whole.g[it])


def test_translation_invariance_full_size(full):
    _, _, _, res, grads = full
    conv = res.converged
    total = grads.start + grads.end + grads.anchor.sum(dim=1)
    scale = 1.0 + grads.start.norm(dim=1)
    err = (total.norm(dim=1) / scale)[conv]
    assert float(err.max()) < 1e-4
    frac = float(conv.float().mean())
    assert 0.30 < frac < 0.37


def test_oracle_subsample_full_size(full):
    b, _, _, res, grads = full
    idx = np.sort(np.random.default_rng(9).choice(b.size, 2048, replace=False))
    args = (b.basis[idx], b.anchor[idx], b.start[idx], b.end[idx])
    ref = O.solve_outputs(*args, b.T0[idx], 20, 1, np.float32)
    it = torch.as_tensor(idx, device=res.T.device)
    pts = res.points[it].double().cpu().numpy()
    L = res.length[it].cpu().numpy()
    conv = converged_mask(*args, ref["T"])
    ok = points_ok(pts, ref["points"]) & lengths_ok(L, ref["L"])
    assert ok[conv].all()
    floor = agreement_floor(*args, b.T0[idx], 20, 1, np.float32)
    assert ok[~conv].mean() >= floor, (ok[~conv].mean(), floor)
    rows = np.nonzero(conv)[0][:256]
    db, da, d0, d1, okg = O.full_gradient_rows(*args, ref["T"], rows)
    got = flat_grad(*(t[it].double().cpu().numpy()[rows] for t in
                      (grads.basis, grads.anchor, grads.start, grads.end)))
    err = grad_rel_err(got, flat_grad(db, da, d0, d1))
    assert np.all(err[okg] <= GRAD_REL)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_converged_gate_confusion_full_size(K):
    """Config 2 at full size (2^22 paths) for every order: on a 2048-path
    subsample, the device's fp32 convergence gate (the count behind bench
    `value`) against the oracle's fp64 classification at the reference T
    (parity.converged_mask), both ways. False positives (device converged,
    oracle not) and false negatives each stay below 1% of the sample, and
    every oracle-converged path is in tolerance."""
    b = datagen.config2(K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    res, _ = solve_with_gradients(sc, b.T0, SolveOptions(iterations=20, precision=Precision.SINGLE))
    idx = np.sort(np.random.default_rng(100 + K).choice(b.size, 2048, replace=False))
    it = torch.as_tensor(idx, device=res.T.device)
    dev = res.converged[it].cpu().numpy()
    args = (b.basis[idx], b.anchor[idx], b.start[idx], b.end[idx])
    ref = O.solve_outputs(*args, b.T0[idx], 20, 1, np.float32)
    conv = converged_mask(*args, ref["T"])
    fp = float((dev & ~conv).mean())
    fn = float((~dev & conv).mean())
    print(f"K={K}: device {dev.mean():.4f} oracle {conv.mean():.4f} FP {fp:.5f} FN {fn:.5f}")
    assert fp <= 0.01 and fn <= 0.01, (fp, fn)
    pts = res.points[it].double().cpu().numpy()
    L = res.length[it].cpu().numpy()
    ok = points_ok(pts, ref["points"]) & lengths_ok(L, ref["L"])
    assert ok[conv].all()
    del res
    torch.cuda.empty_cache()

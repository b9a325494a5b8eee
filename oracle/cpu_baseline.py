"""CPU baseline runner — TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).

Times the reference hot path on the host cores, one worker process per core
with single-threaded BLAS, the way the reference runs (pure numpy):
each worker runs the batched forward BFGS (`_bfgs_kernel`, solver.py:146-215)
on its contiguous shard and then, per path like the reference
(implicit_diff.py is per-path), the full implicit gradient
`length_param_gradient + vjp_solution(gradient)` where the stationarity gate
passes (NotStationary paths are skipped, as the reference would raise for
them).

Two implementations of that work:
- kind "reference": the genuine reference package installed into oracle/_ref
  by oracle/build_ref.py (its own `_bfgs_kernel`, `gradient`,
  `length_param_gradient`, `vjp_solution` on PathSpec objects built from the
  arrays before the clock starts);
- kind "port": the numpy restatement oracle/fermat_oracle.py (bit-exact to
  the reference, tests/test_oracle_pin.py), used when oracle/_ref is absent
  and as the cross-check.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np


REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "fermatpath", "solver.py"))


def _ref_worker(args):
    """The genuine reference (oracle/_ref) on one shard."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import sys

    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from fermatpath.batching import BatchScene
    from fermatpath.errors import FermatPathError
    from fermatpath.geometry import PathSpec, Surface, SurfaceKind
    from fermatpath.implicit_diff import vjp_solution
    from fermatpath.objective import gradient, length_param_gradient
    from fermatpath.solver import Precision, SolveOptions, _bfgs_kernel

    basis, anchor, start, end, T0, iters, fp_iters, do_vjp = args
    specs = []
    if do_vjp:  # the reference's per-path API takes PathSpec objects (its input format)
        for b in range(basis.shape[0]):
            surfs = tuple(Surface(basis=np.asarray(basis[b, i], np.float64),
                                  anchor=np.asarray(anchor[b, i], np.float64),
                                  kind=SurfaceKind.EDGE if not basis[b, i, :, 1].any() else SurfaceKind.PLANE)
                          for i in range(basis.shape[1]))
            specs.append(PathSpec(start=np.asarray(start[b], np.float64),
                                  end=np.asarray(end[b], np.float64), surfaces=surfs))
    t0 = time.perf_counter()
    opts = SolveOptions(iterations=iters, fixed_point_iters=fp_iters, precision=Precision.SINGLE)
    T, g, _ = _bfgs_kernel(BatchScene(basis, anchor, start, end), T0, opts)
    t_fwd = time.perf_counter() - t0
    conv = 0
    if do_vjp:
        for spec, t in zip(specs, T):
            t = np.asarray(t, np.float64)
            try:
                part = length_param_gradient(spec, t)
                corr = vjp_solution(spec, t, gradient(spec, t))
            except FermatPathError:
                continue
            _ = part.flat() + corr.flat()
            conv += 1
    else:
        from fermatpath.batching import path_length_batch

        L = path_length_batch(BatchScene(basis, anchor, start, end).astype(np.float32), T)
        gn = np.linalg.norm(g.reshape(len(L), -1), axis=1)
        conv = int(np.sum(gn < 1e-5 * (1.0 + L)))
    return conv, t_fwd, time.perf_counter() - t0


def _worker(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import fermat_oracle as O

    basis, anchor, start, end, T0, iters, fp_iters, do_vjp = args
    t0 = time.perf_counter()
    r = O.bfgs(basis, anchor, start, end, T0, iters, fp_iters, np.float32)
    t_fwd = time.perf_counter() - t0
    conv = 0
    if do_vjp:
        f64 = np.float64
        for j in range(basis.shape[0]):
            a = (basis[j].astype(f64), anchor[j].astype(f64), start[j].astype(f64),
                 end[j].astype(f64), r["T"][j].astype(f64))
            try:
                O.full_gradient(*a)
            except (O.OracleNotStationary, O.OracleDegenerate, O.OracleSingular):
                continue
            conv += 1
    else:
        L = O.length_batch(basis.astype(np.float32), anchor.astype(np.float32),
                           start.astype(np.float32), end.astype(np.float32), r["T"])
        gn = np.linalg.norm(r["g"].reshape(len(L), -1), axis=1)
        conv = int(np.sum(gn < 1e-5 * (1.0 + L)))
    return conv, t_fwd, time.perf_counter() - t0


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class CpuPool:
    """Persistent spawn-context worker pool (workers never touch CUDA).

    kind: "reference" (oracle/_ref, when installed), "port", or "auto"
    (reference when available, else port)."""

    def __init__(self, cores: int | None = None, kind: str = "port"):
        if kind == "auto":
            kind = "reference" if reference_available() else "port"
        if kind == "reference" and not reference_available():
            raise RuntimeError("oracle/_ref is not installed (python oracle/build_ref.py)")
        self.kind = kind
        self._fn = _ref_worker if kind == "reference" else _worker
        self.cores = cores or host_cores()
        env_threads = os.environ.get("OMP_NUM_THREADS")
        os.environ["OMP_NUM_THREADS"] = "1"
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.cores)
        if env_threads is None:
            os.environ.pop("OMP_NUM_THREADS", None)
        else:
            os.environ["OMP_NUM_THREADS"] = env_threads

    def run(self, basis, anchor, start, end, T0, iters, fp_iters=1, do_vjp=True):
        """One step over the sample; returns (converged paths, wall seconds)."""
        B = basis.shape[0]
        bounds = np.linspace(0, B, self.cores + 1).astype(int)
        jobs = [(basis[lo:hi], anchor[lo:hi], start[lo:hi], end[lo:hi], T0[lo:hi], iters,
                 fp_iters, do_vjp) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
        t0 = time.perf_counter()
        out = self.pool.map(self._fn, jobs)
        wall = time.perf_counter() - t0
        return sum(o[0] for o in out), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def _bfgs_T(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import fermat_oracle as O

    basis, anchor, start, end, T0, iters, dtype = args
    with np.errstate(all="ignore"):
        return O.bfgs(basis, anchor, start, end, T0, iters, 1, dtype)["T"]


def bfgs_parallel(basis, anchor, start, end, T0, iters, dtype=np.float32, chunk=1 << 16,
                  cores: int | None = None):
    """The oracle's batched BFGS (T only) over host cores, in row chunks —
    for parity checks on millions of candidates (per-path results do not
    depend on the batch composition)."""
    B = basis.shape[0]
    jobs = [(basis[lo:lo + chunk], anchor[lo:lo + chunk], start[lo:lo + chunk], end[lo:lo + chunk],
             T0[lo:lo + chunk], iters, dtype) for lo in range(0, B, chunk)]
    if not jobs:
        return np.zeros((0,) + tuple(T0.shape[1:]), dtype)
    env_threads = os.environ.get("OMP_NUM_THREADS")
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        with mp.get_context("spawn").Pool(min(cores or host_cores(), len(jobs))) as pool:
            out = pool.map(_bfgs_T, jobs)
    finally:
        if env_threads is None:
            os.environ.pop("OMP_NUM_THREADS", None)
        else:
            os.environ["OMP_NUM_THREADS"] = env_threads
    return np.concatenate(out)


def _full_grad_rows(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import fermat_oracle as O

    basis, anchor, start, end, T, weights = args
    return O.full_gradient_rows(basis, anchor, start, end, T, np.arange(len(T)), weights)


def full_gradient_parallel(basis, anchor, start, end, T, weights=None, chunk=4096,
                           cores: int | None = None):
    """oracle.full_gradient_rows over every row, in chunks on the host cores."""
    n = len(T)
    jobs = [(basis[lo:lo + chunk], anchor[lo:lo + chunk], start[lo:lo + chunk], end[lo:lo + chunk],
             T[lo:lo + chunk], None if weights is None else weights[lo:lo + chunk])
            for lo in range(0, n, chunk)]
    env_threads = os.environ.get("OMP_NUM_THREADS")
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        with mp.get_context("spawn").Pool(max(1, min(cores or host_cores(), len(jobs)))) as pool:
            out = pool.map(_full_grad_rows, jobs)
    finally:
        if env_threads is None:
            os.environ.pop("OMP_NUM_THREADS", None)
        else:
            os.environ["OMP_NUM_THREADS"] = env_threads
    return tuple(np.concatenate([o[i] for o in out]) for i in range(5))

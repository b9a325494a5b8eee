"""CPU baseline runner — TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).

Times the numpy restatement of the reference hot path (oracle/fermat_oracle.py)
on the host cores, one worker process per core with single-threaded BLAS, the
way the reference runs (pure numpy): each worker runs the batched
forward BFGS (`_bfgs_kernel`, solver.py:146-215) on its contiguous shard and
then, per path like the reference (implicit_diff.py is per-path), the full
implicit gradient `length_param_gradient + vjp_solution(gradient)` where the
stationarity gate passes (NotStationary paths are skipped, as the reference
would raise for them).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np


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
    """Persistent spawn-context worker pool (workers never touch CUDA)."""

    def __init__(self, cores: int | None = None):
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
        out = self.pool.map(_worker, jobs)
        wall = time.perf_counter() - t0
        return sum(o[0] for o in out), wall

    def close(self):
        self.pool.close()
        self.pool.join()

"""Seeded synthetic path batches for the BASELINE.json configurations.

The reference ships no generator for these workloads (its own
``bench.gen_scenes``, /root/reference/pkg/src/fermatpath/bench.py:292-306,
builds well-conditioned specular waypoints instead), so this module is the
spec SURVEY.md §8(d) recommends:

* numpy ``default_rng`` (PCG64) on the host, float64 draws, cast once to the
  working dtype; the very same arrays go to the GPU and to the CPU oracle;
* draw order: TX (B,3) U[-10,10]; RX (B,3) U[-10,10]; origins (B,K,3)
  U[-5,5]; then for each interaction position in order, a reflector draws
  normal ~ N(0,I3) (normalised) and r ~ N(0,I3), e1 = normalise(r - (r.n)n),
  e2 = n x e1; a diffraction edge draws a direction ~ N(0,I3) (normalised)
  and stores an exactly-zero second basis column
  (/root/reference/pkg/src/fermatpath/geometry.py:86-90);
* zero initial parameters.

Arrays follow the reference batch layout (batching.py:20-25): basis
(B,K,3,2), anchor (B,K,3), start (B,3), end (B,3), T0 (B,K,2).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

BOX_ENDPOINTS = 10.0
BOX_ORIGINS = 5.0


@dataclass
class PathBatch:
    """Host-side stacked batch in the reference layout."""

    basis: np.ndarray  # (B, K, 3, 2)
    anchor: np.ndarray  # (B, K, 3)
    start: np.ndarray  # (B, 3)
    end: np.ndarray  # (B, 3)
    T0: np.ndarray  # (B, K, 2)
    orderings: list  # list of (kinds string, first row, row count)

    @property
    def size(self) -> int:
        return int(self.start.shape[0])

    @property
    def order(self) -> int:
        return int(self.basis.shape[1])

    def astype(self, dtype) -> "PathBatch":
        return PathBatch(
            self.basis.astype(dtype),
            self.anchor.astype(dtype),
            self.start.astype(dtype),
            self.end.astype(dtype),
            self.T0.astype(dtype),
            list(self.orderings),
        )

    def slice(self, lo: int, hi: int) -> "PathBatch":
        return PathBatch(
            self.basis[lo:hi], self.anchor[lo:hi], self.start[lo:hi],
            self.end[lo:hi], self.T0[lo:hi], [],
        )

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.basis, self.anchor, self.start, self.end, self.T0))


def all_orderings(K: int) -> list[str]:
    """Every R/D ordering of order K, in lexicographic order R < D."""
    return ["".join(p) for p in itertools.product("RD", repeat=K)]


def _normalise(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _draw(rng: np.random.Generator, B: int, kinds: str):
    K = len(kinds)
    start = rng.uniform(-BOX_ENDPOINTS, BOX_ENDPOINTS, size=(B, 3))
    end = rng.uniform(-BOX_ENDPOINTS, BOX_ENDPOINTS, size=(B, 3))
    anchor = rng.uniform(-BOX_ORIGINS, BOX_ORIGINS, size=(B, K, 3))
    basis = np.zeros((B, K, 3, 2))
    for i, kind in enumerate(kinds):
        if kind == "R":
            nrm = _normalise(rng.normal(size=(B, 3)))
            r = rng.normal(size=(B, 3))
            e1 = _normalise(r - np.sum(r * nrm, axis=1, keepdims=True) * nrm)
            e2 = np.cross(nrm, e1)
            basis[:, i, :, 0] = e1
            basis[:, i, :, 1] = e2
        elif kind == "D":
            basis[:, i, :, 0] = _normalise(rng.normal(size=(B, 3)))
        else:
            raise ValueError(f"unknown interaction kind {kind!r}")
    return basis, anchor, start, end


def gen_batch(seed: int, orderings, per_ordering: int, dtype=np.float32) -> PathBatch:
    """Ordering-major batch: `per_ordering` paths for each kinds string."""
    orderings = list(orderings)
    if not orderings:
        raise ValueError("need at least one ordering")
    K = len(orderings[0])
    if any(len(o) != K for o in orderings):
        raise ValueError("orderings must share the same order K")
    parts = []
    rows = []
    for j, kinds in enumerate(orderings):
        rng = np.random.default_rng([int(seed), K, j])
        parts.append(_draw(rng, per_ordering, kinds))
        rows.append((kinds, j * per_ordering, per_ordering))
    basis = np.concatenate([p[0] for p in parts]).astype(dtype)
    anchor = np.concatenate([p[1] for p in parts]).astype(dtype)
    start = np.concatenate([p[2] for p in parts]).astype(dtype)
    end = np.concatenate([p[3] for p in parts]).astype(dtype)
    T0 = np.zeros((basis.shape[0], K, 2), dtype=dtype)
    return PathBatch(basis, anchor, start, end, T0, rows)


def config0(B: int = 4096, seed: int = 0, dtype=np.float32) -> PathBatch:
    """BASELINE config 0: order-2 'RD', 4096 paths, zero init (10 iterations)."""
    return gen_batch(seed, ["RD"], B, dtype)


def config1(K: int, B: int = 1 << 20, dtype=np.float32) -> PathBatch:
    """BASELINE config 1: diffraction-only order K (seed 1..3 by K)."""
    return gen_batch(K, ["D" * K], B, dtype)


def config2(K: int, B: int = 1 << 22, dtype=np.float32) -> PathBatch:
    """BASELINE config 2: every R/D ordering of order K, B paths split evenly."""
    ords = all_orderings(K)
    if B % len(ords):
        raise ValueError("B must divide evenly over the 2^K orderings")
    return gen_batch(100 + K, ords, B // len(ords), dtype)


def interleave(batch: PathBatch, seed: int = 0) -> PathBatch:
    """Random permutation of the path axis (tests batch-order invariance)."""
    perm = np.random.default_rng(seed).permutation(batch.size)
    return PathBatch(
        batch.basis[perm], batch.anchor[perm], batch.start[perm], batch.end[perm],
        batch.T0[perm], [],
    )

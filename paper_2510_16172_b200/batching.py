"""Device-resident stacked batches (the reference's BatchScene, on HBM).

Mirrors /root/reference/pkg/src/fermatpath/batching.py:20-126. The layout is
the reference's C-contiguous one — basis (B,K,3,2), anchor (B,K,3),
start/end (B,3), parameters (B,K,2) — held as CUDA tensors so that the C-ABI
kernels read them in place. Host numpy arrays are accepted everywhere and
uploaded once.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import NonUniformBatch, ShapeMismatch
from .geometry import PathSpec

_TORCH_DTYPES = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.ExtensionMissing("no CUDA device: the solver runs on the GPU only")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None) -> torch.Tensor:
    """Contiguous CUDA tensor view/copy of a numpy array or tensor."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass(frozen=True)
class BatchScene:
    """Stacked scene of B paths with K interactions each, on the GPU."""

    basis: torch.Tensor   # (B, K, 3, 2)
    anchor: torch.Tensor  # (B, K, 3)
    start: torch.Tensor   # (B, 3)
    end: torch.Tensor     # (B, 3)

    def __post_init__(self):
        basis = to_device(self.basis)
        dt = basis.dtype if basis.dtype in (torch.float32, torch.float64) else torch.float64
        basis = basis.to(dt)
        anchor, start, end = (to_device(x, dt) for x in (self.anchor, self.start, self.end))
        if basis.dim() != 4 or basis.shape[2:] != (3, 2):
            raise ShapeMismatch(f"basis must be (B, K, 3, 2), got {tuple(basis.shape)}")
        B, K = basis.shape[0], basis.shape[1]
        if tuple(anchor.shape) != (B, K, 3) or tuple(start.shape) != (B, 3) or tuple(end.shape) != (B, 3):
            raise ShapeMismatch("anchor/start/end shapes do not match basis")
        object.__setattr__(self, "basis", basis)
        object.__setattr__(self, "anchor", anchor)
        object.__setattr__(self, "start", start)
        object.__setattr__(self, "end", end)

    @classmethod
    def from_specs(cls, specs: Sequence[PathSpec]) -> "BatchScene":
        """Stack specs sharing one interaction count (batching.py:28-39)."""
        if not specs:
            raise NonUniformBatch("empty batch")
        n = specs[0].n
        if any(s.n != n for s in specs):
            raise NonUniformBatch("batch members have differing interaction counts")
        return cls(np.stack([s.basis_tensor for s in specs]),
                   np.stack([s.anchor_tensor for s in specs]),
                   np.stack([s.start for s in specs]),
                   np.stack([s.end for s in specs]))

    @classmethod
    def from_arrays(cls, basis, anchor, start, end, dtype=None) -> "BatchScene":
        sc = cls(basis, anchor, start, end)
        return sc if dtype is None else sc.astype(dtype)

    @property
    def size(self) -> int:
        return int(self.start.shape[0])

    @property
    def n(self) -> int:
        return int(self.basis.shape[1])

    @property
    def dtype(self):
        return np.float32 if self.basis.dtype == torch.float32 else np.float64

    def astype(self, dtype) -> "BatchScene":
        tdt = _TORCH_DTYPES[np.dtype(dtype)]
        if self.basis.dtype == tdt:
            return self
        return BatchScene(self.basis.to(tdt), self.anchor.to(tdt), self.start.to(tdt), self.end.to(tdt))

    def active_mask(self) -> torch.Tensor:
        """(B, K, 2) mask of coordinates whose basis column is nonzero (batching.py:63-65)."""
        return (self.basis != 0).any(dim=2)

    def seg_epsilon(self) -> torch.Tensor:
        """Per-path segment floor, fp64 then cast (batching.py:67-72)."""
        d = self.end.double() - self.start.double()
        return (1e-12 * (1.0 + torch.linalg.vector_norm(d, dim=1))).to(self.basis.dtype)

    def slice(self, lo: int, hi: int) -> "BatchScene":
        return BatchScene(self.basis[lo:hi], self.anchor[lo:hi], self.start[lo:hi], self.end[lo:hi])


def stack_params(specs: Sequence[PathSpec], T0s) -> np.ndarray:
    """Stack per-path (n, 2) parameters into (B, n, 2) (batching.py:75-80)."""
    T = np.stack([np.asarray(t, dtype=float) for t in T0s])
    if T.shape != (len(specs), specs[0].n, 2):
        raise ShapeMismatch(f"bad stacked parameter shape {T.shape}")
    return T


def params_tensor(sc: BatchScene, T) -> torch.Tensor:
    t = to_device(T, sc.basis.dtype)
    if tuple(t.shape) != (sc.size, sc.n, 2):
        raise ShapeMismatch(f"parameters must be ({sc.size}, {sc.n}, 2), got {tuple(t.shape)}")
    return t


def objective_batch(sc: BatchScene, T, hessian: bool = False):
    """Unclamped length, gradient and (optionally) dense Hessian per path, fp64.

    The batched form of objective.path_length / gradient / hessian
    (objective.py:34-64). Returns (L (B,), g (B,K,2), H (B,2K,2K) or None,
    status (B,) uint8 with FP_STATUS_DEGENERATE_FINAL where the reference
    would raise DegenerateSegment).
    """
    lib = _lib.load()
    sc64 = sc.astype(np.float64)
    T = params_tensor(sc64, T)
    B, K = sc.size, sc.n
    dev = sc64.basis.device
    L = torch.empty(B, dtype=torch.float64, device=dev)
    g = torch.empty(B, K, 2, dtype=torch.float64, device=dev)
    H = torch.empty(B, 2 * K, 2 * K, dtype=torch.float64, device=dev) if hessian else None
    st = torch.empty(B, dtype=torch.uint8, device=dev)
    rc = lib.fp_objective_f64(ptr(sc64.basis), ptr(sc64.anchor), ptr(sc64.start), ptr(sc64.end),
                              ptr(T), B, K, ptr(L), ptr(g), ptr(H), ptr(st), stream_ptr())
    _lib.check(rc, "fp_objective_f64")
    return L, g, H, st


def embed_batch(sc: BatchScene, T) -> torch.Tensor:
    """(B, K+2, 3) path points (batching.py:83-86)."""
    T = params_tensor(sc, T)
    mid = torch.einsum("bnij,bnj->bni", sc.basis, T) + sc.anchor
    return torch.cat([sc.start[:, None], mid, sc.end[:, None]], dim=1)


def path_length_batch(sc: BatchScene, T) -> torch.Tensor:
    """(B,) unclamped path lengths (batching.py:123-126), via the objective kernel."""
    return objective_batch(sc, T)[0]

"""fp64 throughput (the reference's default precision) at config-2 sizes: forward
solve and fused solve + VJP, ordering-major and scattered (interleaved) layouts,
AUTO policy vs the dense kernel; fp32 AUTO for scale."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients  # noqa: E402


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for K in (1, 2, 3, 4, 5):
    b0 = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 20) // 2 ** K)
    for layout in ("ordered", "interleaved"):
        b = b0 if layout == "ordered" else datagen.interleave(b0, seed=K)
        for prec, pol in ((Precision.DOUBLE, "auto"), (Precision.DOUBLE, "dense"), (Precision.SINGLE, "auto")):
            sc = BatchScene(b.basis, b.anchor, b.start, b.end).astype(prec.dtype)
            T0 = torch.zeros(b.size, K, 2, dtype=torch.float64 if prec is Precision.DOUBLE else torch.float32,
                             device="cuda")
            opts = SolveOptions(iterations=20, precision=prec)
            _lib.set_kernel_policy(pol)
            try:
                f = timed(lambda: solve(sc, T0, opts, want_grad=False, want_points=False))
                g = timed(lambda: solve_with_gradients(sc, T0, opts))
            finally:
                _lib.set_kernel_policy("auto")
            print(f"K={K} {layout:11s} {prec.name:6s} {pol:5s} {b.size} paths: fwd {f:7.3f} ms  "
                  f"fused {g:7.3f} ms  ({b.size / g * 1e3:.3g} paths/s fused)", flush=True)

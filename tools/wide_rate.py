"""Throughput of the warp-per-path solver (orders 9..64), fp32 and fp64, fused solve + VJP."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve_with_gradients  # noqa: E402

for K in (9, 16, 33, 64):
    n = (1 << 20) // K
    order = "".join("RD"[(i * 7 + K) % 3 == 0] for i in range(K))
    b = datagen.gen_batch(200 + K, [order], n)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    for prec in (Precision.SINGLE, Precision.DOUBLE):
        opts = SolveOptions(iterations=20, precision=prec)
        solve_with_gradients(sc, b.T0, opts)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            res, _ = solve_with_gradients(sc, b.T0, opts)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"K={K:2d} {prec.name:6s} {b.size} paths, 20 it: {ms:8.3f} ms  {b.size / ms * 1e3:.3g} paths/s "
              f"converged {float(res.converged.float().mean()):.2f}", flush=True)

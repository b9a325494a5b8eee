"""fp64 forward solve throughput (the reference's default precision) at config-2 sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve  # noqa: E402

for K in (1, 2, 3, 4, 5):
    b = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 20) // 2 ** K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end).astype(np.float64)
    T0 = torch.zeros(b.size, K, 2, dtype=torch.float64, device="cuda")
    for prec, scc in ((Precision.DOUBLE, sc), (Precision.SINGLE, sc.astype(np.float32))):
        opts = SolveOptions(iterations=20, precision=prec)
        t0_ = T0 if prec is Precision.DOUBLE else T0.float()
        for _ in range(2):
            solve(scc, t0_, opts)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            solve(scc, t0_, opts)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"K={K} {prec.name:6s} {b.size} paths: {ms:.3f} ms  {b.size / ms * 1e3:.3g} paths/s", flush=True)

"""fp64 tile kernels, ordering-major 2^20-path batches: fused and forward ms for the orders given."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients  # noqa: E402


def timed(fn, n=10):
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


for K in [int(k) for k in sys.argv[1:]] or [2, 3]:
    b = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 20) // 2 ** K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end).astype("float64")
    T0 = torch.zeros(b.size, K, 2, dtype=torch.float64, device="cuda")
    opts = SolveOptions(iterations=20, precision=Precision.DOUBLE)
    f = timed(lambda: solve(sc, T0, opts, want_grad=False))
    g = timed(lambda: solve_with_gradients(sc, T0, opts))
    print(f"K={K} fp64: fwd {f:.3f} ms, fused {g:.3f} ms", flush=True)

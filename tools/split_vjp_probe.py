"""Is the fused solve + VJP kernel faster than solve followed by the VJP-only kernel? (per order)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.implicit_diff import vjp_batch  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients  # noqa: E402


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


opts = SolveOptions(iterations=20, precision=Precision.SINGLE)
for K in (3, 4, 5):
    b = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 22) // 2 ** K)
    sc = BatchScene(b.basis, b.anchor, b.start, b.end)
    T0 = torch.zeros(b.size, K, 2, device="cuda")
    fused = timed(lambda: solve_with_gradients(sc, T0, opts))
    fwd = timed(lambda: solve(sc, T0, opts, want_grad=False))
    T = solve(sc, T0, opts).T
    vjp = timed(lambda: vjp_batch(sc, T, w_L=1.0, mode="full"))
    print(f"K={K}: fused {fused:.3f} ms, fwd {fwd:.3f} + vjp-only {vjp:.3f} = {fwd + vjp:.3f} ms", flush=True)

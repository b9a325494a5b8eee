"""Per-call wall times (synchronised) of the forward solve and the fused step on a
scattered (interleaved) or ordering-major layout under the AUTO / TILE / BUCKET /
DENSE policies: first-call costs and the steady state of each route.
    python tools/f64_probe.py K [f64|f32] [interleaved|ordered]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = Precision.DOUBLE if (len(sys.argv) < 3 or sys.argv[2] == "f64") else Precision.SINGLE
b0 = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 20) // 2 ** K)
layout = sys.argv[3] if len(sys.argv) > 3 else "interleaved"
b = datagen.interleave(b0, seed=K) if layout == "interleaved" else b0
sc = BatchScene(b.basis, b.anchor, b.start, b.end).astype(prec.dtype)
dt = torch.float64 if prec is Precision.DOUBLE else torch.float32
T0 = torch.zeros(b.size, K, 2, dtype=dt, device="cuda")
opts = SolveOptions(iterations=20, precision=prec)
for pol in ("auto", "tile", "bucket", "dense", "auto"):
    _lib.set_kernel_policy(pol)
    for name, fn in (("fwd", lambda: solve(sc, T0, opts, want_grad=False, want_points=False)),
                     ("fwd+g", lambda: solve(sc, T0, opts)),
                     ("fused", lambda: solve_with_gradients(sc, T0, opts))):
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"K={K} {prec.name} {layout[:5]} {pol:6s} {name:6s} per call ms: " + " ".join(f"{x:.3f}" for x in ts), flush=True)
_lib.set_kernel_policy("auto")

import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen
from paper_2510_16172_b200.batching import BatchScene
from paper_2510_16172_b200.solver import Precision, SolveOptions, solve, solve_with_gradients
K = 2
b0 = datagen.gen_batch(102, datagen.all_orderings(K), (1 << 20) // 4)
for layout in ("ordered", "interleaved", "ordered", "interleaved"):
    b = b0 if layout == "ordered" else datagen.interleave(b0, seed=K)
    for prec in (Precision.SINGLE, Precision.DOUBLE):
        sc = BatchScene(b.basis, b.anchor, b.start, b.end).astype(prec.dtype)
        T0 = torch.zeros(b.size, K, 2, dtype=torch.float64 if prec is Precision.DOUBLE else torch.float32, device="cuda")
        opts = SolveOptions(iterations=20, precision=prec)
        ts = []
        for i in range(8):
            n0 = _lib.launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            solve(sc, T0, opts, want_grad=False, want_points=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(f"{e0.elapsed_time(e1):.2f}/{_lib.launch_count()-n0}")
        print(layout, prec.name, " ".join(ts), flush=True)

"""Bitwise comparison and timing of two libraries on the long-path solver (orders 9..64).

    python tools/ab_wide.py libA.so libB.so [iterations] [orders, e.g. 9,12,16]

Both libraries are loaded side by side with ctypes; the same device inputs
(the tools/wide_rate.py batches: 2^20 / K paths of one mixed ordering) go
through fp_solve_vjp_f32 / _f64 of each; every output is compared bit for bit
and each library's fused step is timed with CUDA events (3 alternating rounds).
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402


def load(path):
    lib = C.CDLL(path)
    fns = {}
    for name, ft in (("fp_solve_vjp_f32", C.c_float), ("fp_solve_vjp_f64", C.c_double)):
        fn = getattr(lib, name)
        fn.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, ft, C.c_int] + \
            [C.c_void_p] * 8 + [C.c_void_p]
        fn.restype = C.c_int
        fns[name] = fn
    return fns


libs = [load(sys.argv[1]), load(sys.argv[2])]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
orders = [int(k) for k in sys.argv[4].split(",")] if len(sys.argv) > 4 else [9, 16, 33, 64]
dev = torch.device("cuda")
for K in orders:
    n = (1 << 20) // K
    order = "".join("RD"[(i * 7 + K) % 3 == 0] for i in range(K))
    b = datagen.gen_batch(200 + K, [order], n)
    for dt, name in ((torch.float32, "fp_solve_vjp_f32"), (torch.float64, "fp_solve_vjp_f64")):
        ins = [torch.from_numpy(a).to(dev, dt) for a in (b.basis, b.anchor, b.start, b.end, b.T0)]
        B = b.size
        outs = []
        for L in libs:
            o = [torch.empty(B, K, 2, device=dev, dtype=dt), torch.empty(B, K, 3, device=dev, dtype=dt),
                 torch.empty(B, device=dev, dtype=dt), torch.empty(B, K, 3, 2, device=dev, dtype=dt),
                 torch.empty(B, K, 3, device=dev, dtype=dt), torch.empty(B, 3, device=dev, dtype=dt),
                 torch.empty(B, 3, device=dev, dtype=dt), torch.empty(B, dtype=torch.uint8, device=dev)]
            outs.append(o)

        def run(i):
            rc = libs[i][name](*(t.data_ptr() for t in ins), B, K, iters, 1, None, 1.0, 0,
                               *(t.data_ptr() for t in outs[i]), None)
            assert rc == 0, rc

        ms = [0.0, 0.0]
        for i in (0, 1):
            run(i)
        torch.cuda.synchronize()
        for _ in range(3):
            for i in (0, 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(i)
                e1.record()
                torch.cuda.synchronize()
                ms[i] += e0.elapsed_time(e1) / 3
        names = ("T", "points", "length", "d_basis", "d_anchor", "d_start", "d_end", "status")
        diff = []
        for nm, x, y in zip(names, *outs):
            same = (x.view(torch.uint8) == y.view(torch.uint8)).reshape(B, -1).all(dim=1)
            diff.append(f"{nm}:{int((~same).sum())}")
        print(f"K={K:2d} {str(dt)[6:]:7s} {B} paths {iters} it: A {ms[0]:8.3f} ms ({B / ms[0] * 1e3:.3g} paths/s)"
              f"  B {ms[1]:8.3f} ms ({B / ms[1] * 1e3:.3g} paths/s)  differing paths " + " ".join(diff),
              flush=True)

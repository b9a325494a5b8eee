"""Bitwise comparison of two libraries on the fused step (config 2 data):
    python tools/ab_bits.py libA.so libB.so [orders]
Both libraries are loaded side by side with ctypes; the same device inputs go
through fp_solve_vjp_f32 of each; every output is compared bit for bit."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import datagen  # noqa: E402


def load(path):
    lib = C.CDLL(path)
    fn = lib.fp_solve_vjp_f32
    fn.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_float, C.c_int] + \
        [C.c_void_p] * 8 + [C.c_void_p]
    fn.restype = C.c_int
    return fn


fa, fb = load(sys.argv[1]), load(sys.argv[2])
orders = [int(k) for k in (sys.argv[3] if len(sys.argv) > 3 else "1,3").split(",")]
dev = torch.device("cuda")
for K in orders:
    b = datagen.config2(K, 1 << 20)
    ins = [torch.from_numpy(a).to(dev) for a in (b.basis, b.anchor, b.start, b.end, b.T0)]
    B = b.size
    outs = []
    for fn in (fa, fb):
        o = [torch.empty(B, K, 2, device=dev), torch.empty(B, K, 3, device=dev), torch.empty(B, device=dev),
             torch.empty(B, K, 3, 2, device=dev), torch.empty(B, K, 3, device=dev), torch.empty(B, 3, device=dev),
             torch.empty(B, 3, device=dev), torch.empty(B, dtype=torch.uint8, device=dev)]
        rc = fn(*(t.data_ptr() for t in ins), B, K, 20, 1, None, 1.0, 0, *(t.data_ptr() for t in o), None)
        assert rc == 0, rc
        torch.cuda.synchronize()
        outs.append(o)
    names = ("T", "points", "length", "d_basis", "d_anchor", "d_start", "d_end", "status")
    for n, x, y in zip(names, *outs):
        same = (x.view(torch.uint8) == y.view(torch.uint8)).reshape(B, -1).all(dim=1)
        per = [int((~same[lo:lo + cnt]).sum()) for _, lo, cnt in b.orderings]
        print(f"K={K} {n}: {int((~same).sum())} of {B} paths differ; per ordering "
              + " ".join(f"{o}:{d}" for (o, _, _), d in zip(b.orderings, per)))
        if n == "T" and int((~same).sum()):
            i = int(torch.nonzero(~same)[0])
            print("   first differing path", i, x[i].tolist(), y[i].tolist())

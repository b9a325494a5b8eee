"""Does the fused kernel run directly on pinned host buffers (zero-copy over PCIe)?

Runs fp_solve_vjp_f32 with host-pinned input/output pointers (UVA-mapped) and
compares against the device-buffer run; then times both at 2^22 paths.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402

lib = _lib.load()
K = 3
for B_exp in (10, 22):
    host = datagen.gen_batch(103, datagen.all_orderings(K), (1 << B_exp) // 8)
    B = host.size
    pin = lambda shape, dt=torch.float32: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
    hin = [pin(tuple(host.basis.shape)), pin(tuple(host.anchor.shape)), pin((B, 3)), pin((B, 3)), pin((B, K, 2))]
    for t, a in zip(hin, (host.basis, host.anchor, host.start, host.end, host.T0)):
        t.numpy()[...] = a
    shapes = [(B, K, 2), (B, K, 3), (B,), (B, K, 3, 2), (B, K, 3), (B, 3), (B, 3)]
    hout = [pin(s) for s in shapes] + [pin((B,), torch.uint8)]
    din = [t.cuda() for t in hin]
    dout = [torch.empty(s, device="cuda") for s in shapes] + [torch.empty(B, dtype=torch.uint8, device="cuda")]
    P = lambda t: t.data_ptr()  # noqa: E731
    s = torch.cuda.current_stream().cuda_stream

    def run(i, o):
        rc = lib.fp_solve_vjp_f32(*(P(t) for t in i), B, K, 20, 1, None, 1.0, _lib.VJP_FULL,
                                  *(P(t) for t in o), s)
        assert rc == 0, rc

    run(din, dout)
    run(hin, hout)
    torch.cuda.synchronize()
    same = all(torch.equal(a.cpu(), b) for a, b in zip(dout, hout))
    print(f"B={B}: zero-copy results equal device results: {same}", flush=True)
    if B_exp == 22:
        for name, i, o in (("device", din, dout), ("zero-copy", hin, hout)):
            run(i, o)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                run(i, o)
            torch.cuda.synchronize()
            print(f"{name}: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms/step", flush=True)

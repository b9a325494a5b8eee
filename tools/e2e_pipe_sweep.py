"""Host-buffer step streamed through submit / wait: ms per step over (chunk, depth)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402

lib = _lib.load()
K = 3
host = datagen.config2(K)
B = host.size
pin = lambda shape, dt=torch.float32: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
# bench.py's e2e copies: scene in (T0 = NULL: zero init on the device), points not copied out
hin = [pin(tuple(host.basis.shape)), pin(tuple(host.anchor.shape)), pin((B, 3)), pin((B, 3))]
for t, a in zip(hin, (host.basis, host.anchor, host.start, host.end)):
    t.numpy()[...] = a
mk = lambda: [pin((B, K, 2)), None, pin((B,)), pin((B, K, 3, 2)), pin((B, K, 3)), pin((B, 3)),  # noqa: E731
              pin((B, 3)), pin((B,), torch.uint8)]
outs = [mk(), mk()]
P = lambda t: None if t is None else t.data_ptr()  # noqa: E731


def submit(i, chunk, depth):
    tk = ctypes.c_uint64(0)
    rc = lib.fp_solve_vjp_host_submit_f32(*(P(t) for t in hin), None, B, K, 20, 1, 1.0, 0,
                                          *(P(t) for t in outs[i % 2]), chunk, depth, ctypes.addressof(tk))
    assert rc == 0, rc
    return tk.value


for chunk in (1 << 19, 1 << 20, 1 << 21, 1 << 22):
    for depth in (2, 3, 4):
        lib.fp_host_wait(submit(0, chunk, depth))
        n = 8
        t0 = time.perf_counter()
        prev = None
        for i in range(n):
            tk = submit(i, chunk, depth)
            if prev is not None:
                lib.fp_host_wait(prev)
            prev = tk
        lib.fp_host_wait(prev)
        print(chunk, depth, round((time.perf_counter() - t0) / n * 1e3, 3), "ms/step", flush=True)

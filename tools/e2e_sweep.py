import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2510_16172_b200 import _lib, datagen
lib = _lib.load()
K = 3
host = datagen.config2(K)
B = host.size
pin = lambda shape, dt=torch.float32: torch.empty(shape, dtype=dt, pin_memory=True)
hin = [pin(tuple(host.basis.shape)), pin(tuple(host.anchor.shape)), pin((B, 3)), pin((B, 3)), pin((B, K, 2))]
for t, a in zip(hin, (host.basis, host.anchor, host.start, host.end, host.T0)):
    t.numpy()[...] = a
hout = [pin((B, K, 2)), pin((B, K, 3)), pin((B,)), pin((B, K, 3, 2)), pin((B, K, 3)), pin((B, 3)), pin((B, 3)), pin((B,), torch.uint8)]
P = lambda t: t.data_ptr()
for chunk in (1 << 17, 1 << 18, 1 << 19, 1 << 20):
    for ns in (2, 3, 4, 6):
        f = lambda: lib.fp_solve_vjp_host_f32(*(P(t) for t in hin), B, K, 20, 1, 1.0, 0, *(P(t) for t in hout), chunk, ns)
        f()
        t0 = time.perf_counter()
        for _ in range(5):
            assert f() == 0
        print(chunk, ns, round((time.perf_counter() - t0) / 5 * 1e3, 2), 'ms', flush=True)
# raw copy bandwidths
d = torch.empty(B * 39, device='cuda')
h = pin((B * 39,))
for name, fn in (('h2d', lambda: d.copy_(h, non_blocking=True)), ('d2h', lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    print(name, round(B * 39 * 4 * 5 / (time.perf_counter() - t0) / 1e9, 1), 'GB/s')
# simultaneous copies in both directions (is the link full duplex at full rate?)
d2 = torch.empty(B * 39, device='cuda')
h2 = pin((B * 39,))
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(sa):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(sb):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print('bidirectional', round(2 * B * 39 * 4 / dt / 1e9, 1), 'GB/s total,', round(dt * 1e3, 2), 'ms per pair of', round(B * 39 * 4 / 1e6), 'MB copies')

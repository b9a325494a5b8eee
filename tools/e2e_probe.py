"""Where does the host-buffer pipeline's time go? Copy pattern alone (no kernel,
no dependencies), with the same per-chunk copies as fp_solve_vjp_host_f32."""
import sys, time, torch
sys.path.insert(0, '.')
K, B = 3, 1 << 22
w_in = [6 * K, 3 * K, 3, 3, 2 * K]
w_out = [2 * K, 3 * K, 1, 6 * K, 3 * K, 3, 3]
pin = lambda n, dt=torch.float32: torch.empty(n, dtype=dt, pin_memory=True)
hin = [pin(B * w) for w in w_in]
hout = [pin(B * w) for w in w_out] + [pin(B, torch.uint8)]
din = [torch.empty(B * w, device='cuda') for w in w_in]
dout = [torch.empty(B * w, device='cuda') for w in w_out] + [torch.empty(B, dtype=torch.uint8, device='cuda')]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
wo = w_out + [1]

def run(chunk, do_in=True, do_out=True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for lo in range(0, B, chunk):
        n = min(chunk, B - lo)
        if do_in:
            with torch.cuda.stream(s_in):
                for h, d, w in zip(hin, din, w_in):
                    d[lo * w:(lo + n) * w].copy_(h[lo * w:(lo + n) * w], non_blocking=True)
        if do_out:
            with torch.cuda.stream(s_out):
                for h, d, w in zip(hout, dout, wo):
                    h[lo * w:(lo + n) * w].copy_(d[lo * w:(lo + n) * w], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3

for chunk in (1 << 16, 1 << 18, 1 << 19, 1 << 20, 1 << 22):
    run(chunk)
    r = [min(run(chunk, *f) for _ in range(3)) for f in ((True, True), (True, False), (False, True))]
    print(f"chunk {chunk}: both {r[0]:.2f} ms, in only {r[1]:.2f}, out only {r[2]:.2f}", flush=True)

# The same copies with the pipeline's dependencies: copy-out of chunk c waits
# for copy-in of chunk c (optionally with the fused kernel in between).
from paper_2510_16172_b200 import _lib, datagen
lib = _lib.load()
host = datagen.config2(K)
for h, a in zip(hin, (host.basis, host.anchor, host.start, host.end, host.T0)):
    h.numpy()[...] = a.reshape(-1)
s_k = torch.cuda.Stream()
P = lambda t: t.data_ptr()

def run_dep(chunk, kernel):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for lo in range(0, B, chunk):
        n = min(chunk, B - lo)
        with torch.cuda.stream(s_in):
            for h, d, w in zip(hin, din, w_in):
                d[lo * w:(lo + n) * w].copy_(h[lo * w:(lo + n) * w], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        if kernel:
            s_k.wait_event(ev)
            sl = lambda t, w: P(t) + lo * w * t.element_size()
            rc = lib.fp_solve_vjp_f32(*(sl(d, w) for d, w in zip(din, w_in)), n, K, 20, 1, None, 1.0, 0,
                                      *(sl(d, w) for d, w in zip(dout[:7], w_out)), sl(dout[7], 1),
                                      s_k.cuda_stream)
            assert rc == 0
            ev = torch.cuda.Event()
            ev.record(s_k)
        s_out.wait_event(ev)
        with torch.cuda.stream(s_out):
            for h, d, w in zip(hout, dout, wo):
                h[lo * w:(lo + n) * w].copy_(d[lo * w:(lo + n) * w], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3

for chunk in (1 << 18, 1 << 19, 1 << 20):
    run_dep(chunk, True)
    r = [min(run_dep(chunk, k) for _ in range(3)) for k in (False, True)]
    print(f"chunk {chunk}: deps only {r[0]:.2f} ms, deps + kernel {r[1]:.2f}", flush=True)

"""Per-step timing distribution of the K=3 fused step (CUDA events per step).

Looks for bimodal / drifting step times behind bench-to-bench noise.
    python tools/step_jitter.py [steps] [K]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_16172_b200 import _lib, datagen  # noqa: E402
from paper_2510_16172_b200.batching import BatchScene  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
with_sampler = len(sys.argv) > 3 and sys.argv[3] == "nvml"
lib = _lib.load()
dev = torch.device("cuda", 0)
host = datagen.gen_batch(100 + K, datagen.all_orderings(K), (1 << 22) // 2 ** K)
B = host.size
sc = BatchScene(host.basis, host.anchor, host.start, host.end)
T0 = torch.from_numpy(host.T0).to(dev)
f = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)  # noqa: E731
outs = [f(B, K, 2), f(B, K, 3), f(B), f(B, K, 3, 2), f(B, K, 3), f(B, 3), f(B, 3)]
st = torch.empty(B, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream().cuda_stream
P = lambda t: t.data_ptr()  # noqa: E731


def step():
    rc = lib.fp_solve_vjp_f32(P(sc.basis), P(sc.anchor), P(sc.start), P(sc.end), P(T0), B, K, 20, 1,
                              None, 1.0, _lib.VJP_FULL, *(P(t) for t in outs), P(st), stream)
    assert rc == 0


for _ in range(5):
    step()
torch.cuda.synchronize()
if with_sampler:
    import bench as bench_mod

    sampler = bench_mod.ClockSampler(0)
    sampler.__enter__()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
t0 = time.perf_counter()
for a, b in evs:
    a.record()
    step()
    b.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
if with_sampler:
    sampler.__exit__(None, None, None)
    print("nvml samples", len(sampler.samples))
ms = np.array([a.elapsed_time(b) for a, b in evs])
gaps = np.array([evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(steps - 1)])
print(f"K={K} steps={steps} wall/step {wall / steps * 1e3:.4f} ms; step ms: min {ms.min():.4f} "
      f"p10 {np.percentile(ms, 10):.4f} med {np.median(ms):.4f} p90 {np.percentile(ms, 90):.4f} "
      f"max {ms.max():.4f} mean {ms.mean():.4f}; gap ms: mean {gaps.mean():.4f} max {gaps.max():.4f}")
chunks = ms[: steps // 40 * 40].reshape(40, -1).mean(axis=1)
print("mean per 1/40th:", " ".join(f"{c:.3f}" for c in chunks))

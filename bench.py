"""Benchmark: converged Fermat paths/s for the fused forward + implicit-VJP step.

Workload (BASELINE.json config 2 at the headline order K=3): every R/D
ordering of order 3, 2^22 paths per GPU split evenly over the 8 orderings,
fp32, zero init, 20 BFGS iterations with one fixed-point step-size
iteration, then the implicit-differentiation VJP of the summed path length
w.r.t. TX, RX and every object origin/basis vector. A step is one pass of
that fused kernel over the batch; inputs (654 MB/step) exceed the 126 MB L2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU. Under torchrun (WORLD_SIZE set) each process
is one rank; `--gpus N` without torchrun relaunches itself through
torch.distributed.run with N ranks (127.0.0.1). Each rank owns its own 2^22
paths (weak scaling, no data-path collective); time = max over ranks.
`--backend gloo` lets several ranks share one GPU (a functional check of
the multi-rank path; NCCL needs one device per rank).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "converged paths/sec (fwd+implicit VJP) at order K"
UNIT = "paths/s"


def flops_per_path(K: int, I: int, F: int = 1) -> tuple[int, int]:
    """Algorithmic FLOP per path: (forward, VJP).

    add/sub/mul/div/sqrt = 1, FMA = 2; dense uniform 2K formulation.
    """
    S = K + 1
    per_it = 32 * K * K + 90 * K + 29 + (F - 1) * (16 * K + 15)
    fwd = I * per_it + (25 * K + 12 * S) + (S - 1)
    vjp = 219 * K + 22 * S - 32
    return fwd, vjp


def bytes_per_path(K: int) -> tuple[int, int]:
    """HBM bytes per path of the fused step: (read, write)."""
    read = (6 * K + 3 * K + 3 + 3 + 2 * K) * 4
    write = (2 * K + 3 * K + 1 + 6 * K + 3 * K + 3 + 3) * 4 + 1
    return read, write


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                bits = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _init_dist(args):
    """Bind this process to its GPU and (N > 1) join the process group.

    NCCL: one device per rank (LOCAL_RANK). gloo: ranks may share devices
    (LOCAL_RANK modulo the device count) — reductions then stage through
    host memory."""
    import torch

    ws, rank, local = _dist()
    ndev = torch.cuda.device_count()
    if ws > 1 and args.backend == "nccl" and local >= ndev:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {ndev} GPU(s); NCCL needs one "
                         "device per rank (use --backend gloo to share devices)")
    torch.cuda.set_device(local % max(1, ndev) if ws > 1 else 0)
    dev = torch.device("cuda", torch.cuda.current_device())
    if ws > 1:
        import torch.distributed as dist

        if args.backend == "nccl":
            # the communicator's init line (stderr) reports nranks = N
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    return ws, rank, local, dev


def _reduce_dev(dev):
    import torch.distributed as dist

    return "cpu" if dist.get_backend() == "gloo" else dev


def _max_over_ranks(x: float, ws: int, dev) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_reduce_dev(dev))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x: float, ws: int, dev) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_reduce_dev(dev))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _devices_in_use(ws: int, dev) -> int:
    """Distinct GPUs across the ranks (ranks may share one under gloo)."""
    if ws == 1:
        return 1
    import torch.distributed as dist

    ids = [None] * ws
    dist.all_gather_object(ids, (os.uname().nodename, dev.index))
    return len(set(ids))


def _self_launch(args, argv) -> int:
    """`--gpus N` (N > 1) without torchrun: relaunch this script through
    torch.distributed.run with N ranks on this node, as the driver does."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    # the communicator's init line reports nranks = N (stderr)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *argv]
    return subprocess.run(cmd, env=env).returncode


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def _ncu_entry(K: int):
    """The committed `ncu --set full` capture of the fused kernel of order K
    (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as fh:
            return json.load(fh).get(f"fused_k{K}")
    except (OSError, ValueError):
        return None


def _load_ncu_traffic(K: int, paths: int):
    """DRAM bytes (read + write) per launch of the fused kernel, scaled per path."""
    ent = _ncu_entry(K)
    try:
        return None if ent is None else float(ent["dram_bytes_per_path"]) * paths
    except (KeyError, ValueError):
        return None


def gate_check(lib, sc, T, status, n=2048, seed=0):
    """The device's fp32 convergence gate (status bits, the count behind
    `value`) against the reference's gate recomputed in fp64 at the same T:
    objective.gradient / path_length (unclamped norms) through the library's
    fp64 objective kernel, |g| < 1e-5 (1 + L) (implicit_diff.py:25,30-36), on
    a random n-path subsample. Returns the two-way confusion counts."""
    import torch

    from paper_2510_16172_b200 import _lib

    B, K = T.shape[0], T.shape[1]
    idx = torch.as_tensor(np.sort(np.random.default_rng(seed).choice(B, min(n, B), replace=False)),
                          device=T.device)
    f8 = torch.float64
    args = [sc.basis[idx].to(f8).contiguous(), sc.anchor[idx].to(f8).contiguous(),
            sc.start[idx].to(f8).contiguous(), sc.end[idx].to(f8).contiguous(), T[idx].to(f8).contiguous()]
    m = len(idx)
    L = torch.empty(m, dtype=f8, device=T.device)
    g = torch.empty(m, K, 2, dtype=f8, device=T.device)
    st = torch.empty(m, dtype=torch.uint8, device=T.device)
    P = lambda t: t.data_ptr()  # noqa: E731
    _lib.check(lib.fp_objective_f64(*(P(a) for a in args), m, K, P(L), P(g), None, P(st),
                                    torch.cuda.current_stream().cuda_stream), "fp_objective_f64")
    gn = g.reshape(m, -1).norm(dim=1)
    ref = (torch.isfinite(gn) & torch.isfinite(L) & (gn < 1e-5 * (1 + L))
           & ((st & _lib.STATUS_DEGENERATE_FINAL) == 0))
    dev = (status[idx] & _lib.STATUS_UNCONVERGED_MASK) == 0
    return {"sample": m, "device_converged": int(dev.sum()), "fp64_converged": int(ref.sum()),
            "device_only": int((dev & ~ref).sum()), "fp64_only": int((~dev & ref).sum()),
            "what": "device fp32 gate vs the reference gate recomputed in fp64 at the device T "
                    "(fp_objective_f64); the oracle comparison at the reference T is "
                    "tests/test_gpu_fullsize.py::test_converged_gate_confusion_full_size"}


def measure_ffma_peak(lib, stream, dev, register_operands=False):
    """FP32 FFMA peak in TFLOP/s (best of 5, CUDA events). register_operands:
    every operand in a distinct register pair (fp_peak_ffma_reg), the operand
    form of the path kernels' arithmetic."""
    import torch

    props = torch.cuda.get_device_properties(dev)
    blocks = props.multi_processor_count * 8
    iters = 4096
    out = torch.zeros(1, device=dev)
    best = 0.0
    fn = lib.fp_peak_ffma_reg if register_operands else lib.fp_peak_ffma
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = fn(blocks, iters, out.data_ptr(), stream)
        e1.record()
        torch.cuda.synchronize()
        if rc != 0:
            return None
        ms = e0.elapsed_time(e1)
        flops = blocks * 256 * iters * 128 * 2
        best = max(best, flops / (ms * 1e-3) / 1e12)
    return best


def pcie_link(h2d: int, d2h: int, dev, e2e_s: float, reps: int = 3) -> dict:
    """The end-to-end step's bound: the same byte counts moved between pinned
    host memory and the device by plain copies, each direction alone and both
    at once on two streams (copy engines only, no kernel). `frac` = that
    duplex copy time / the e2e step time."""
    import torch

    hi = torch.empty(h2d, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(d2h, dtype=torch.uint8, pin_memory=True)
    di = torch.empty(h2d, dtype=torch.uint8, device=dev)
    do = torch.empty(d2h, dtype=torch.uint8, device=dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(parts):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            evs = []
            for st, fn in parts:
                with torch.cuda.stream(st):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    fn()
                    b.record(st)
                    evs.append((a, b))
            torch.cuda.synchronize(dev)
            # concurrent parts start together: the span is max(end) - min(start)
            t = max(max(a.elapsed_time(b2) for b2 in (b for _, b in evs)) for a, _ in evs)
            best = min(best, t)
        return best

    cin = (s_in, lambda: di.copy_(hi, non_blocking=True))
    cout = (s_out, lambda: ho.copy_(do, non_blocking=True))
    t_in, t_out, t_both = timed([cin]), timed([cout]), timed([cin, cout])
    return {"h2d_gbs": h2d / t_in / 1e6, "d2h_gbs": d2h / t_out / 1e6, "h2d_ms": t_in, "d2h_ms": t_out,
            "duplex_ms": t_both, "frac": t_both / (e2e_s * 1e3),
            "what": "pinned host <-> device copies of the step's h2d / d2h bytes, alone and concurrent "
                    "(two streams, best of 3); frac = duplex_ms / e2e ms_per_step"}


def cpu_sample(batch, n: int):
    """A bounded, ordering-balanced sample of the workload (every ordering equally)."""
    K = batch.order
    nord = max(1, len(batch.orderings))
    per = max(1, n // nord)
    rows = np.concatenate([np.arange(lo, lo + min(per, cnt)) for _, lo, cnt in batch.orderings]) \
        if batch.orderings else np.arange(min(n, batch.size))
    return (batch.basis[rows], batch.anchor[rows], batch.start[rows], batch.end[rows],
            batch.T0[rows]), len(rows), K


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path on all
    host cores — the genuine package installed into oracle/_ref by
    oracle/build_ref.py (kind "reference"), else the bit-exact numpy port
    (kind "port"). With the reference available, the port runs the last
    step's sample once more as a cross-check (same converged count)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    ws = max(ws, args.gpus)
    from paper_2510_16172_b200 import datagen
    from oracle.cpu_baseline import CpuPool

    K, I = args.order, args.iterations
    batch = datagen.config2(K, 1 << 12 if args.quick else args.sample)
    pool = CpuPool(kind="auto")
    # Warm-up steps on a small slice also calibrate the per-step sample: the
    # timed steps together stay within ~150 s of CPU work whatever --steps is.
    (b, a, s0, s1, T0), n_cal, _ = cpu_sample(batch, min(batch.size, 8192))
    rate = None
    for _ in range(max(1, args.warmup)):
        c, w = pool.run(b, a, s0, s1, T0, I)
        rate = n_cal / w
    n_step = int(min(batch.size, max(4096, rate * 150.0 / max(1, args.steps))))
    (b, a, s0, s1, T0), n, _ = cpu_sample(batch, n_step)
    conv_total, wall_total = 0, 0.0
    for _ in range(args.steps):
        c, w = pool.run(b, a, s0, s1, T0, I)
        conv_total += c
        wall_total += w
    pool.close()
    value = conv_total / wall_total
    cross = None
    if pool.kind == "reference":
        port = CpuPool(kind="port")
        pc, pw = port.run(b, a, s0, s1, T0, I)
        port.close()
        cross = {"kind": "port", "value": pc / pw, "converged": pc,
                 "reference_converged": c, "equal": pc == c,
                 "note": "oracle/fermat_oracle.py on the last step's sample"}
    what = ("the reference package itself (oracle/_ref, pip-installed from /root/reference by "
            "oracle/build_ref.py): _bfgs_kernel batched, then per path length_param_gradient + "
            "vjp_solution(gradient)" if pool.kind == "reference" else
            "oracle/fermat_oracle.py numpy restatement, batched forward + per-path implicit "
            "gradient like the reference")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy PCG64, SURVEY.md §8(d) generator)",
        "config": _config(K, I, args.paths, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": pool.cores, "kind": pool.kind,
                         "sample": f"{n} paths per step (all {2 ** K} orderings equally) of config 2 "
                                   f"K={K}; {what}", "cross_check": cross},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "converged_fraction": conv_total / (n * args.steps),
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(K, I, paths, ws):
    return {"workload": f"config2: every R/D ordering of order K={K}, fwd + full implicit VJP of sum L",
            "K": K, "orderings": 2 ** K, "paths_per_gpu": paths, "iterations": I, "fp_iters": 1,
            "init": "zero", "l2": "inputs larger than L2 (no flush needed)",
            "parallelism": f"dp{ws} (independent path shards)"}


def run_ours(args):
    import torch

    from paper_2510_16172_b200 import _lib, datagen
    from paper_2510_16172_b200.batching import BatchScene

    ws, rank, local, dev = _init_dist(args)
    lib = _lib.load()
    _lib.set_kernel_policy(args.policy)
    K, I, F = args.order, args.iterations, 1
    B = args.paths
    host = datagen.gen_batch(100 + K + 1000 * rank, datagen.all_orderings(K), B // 2 ** K)
    B = host.size
    sc = BatchScene(host.basis, host.anchor, host.start, host.end)
    T0 = torch.from_numpy(host.T0).to(dev)
    f32 = torch.float32
    outT = torch.empty(B, K, 2, dtype=f32, device=dev)
    outP = torch.empty(B, K, 3, dtype=f32, device=dev)
    outL = torch.empty(B, dtype=f32, device=dev)
    gB = torch.empty(B, K, 3, 2, dtype=f32, device=dev)
    gA = torch.empty(B, K, 3, dtype=f32, device=dev)
    g0 = torch.empty(B, 3, dtype=f32, device=dev)
    g1 = torch.empty(B, 3, dtype=f32, device=dev)
    st = torch.empty(B, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    P = lambda t: t.data_ptr()  # noqa: E731

    def step():
        rc = lib.fp_solve_vjp_f32(P(sc.basis), P(sc.anchor), P(sc.start), P(sc.end), P(T0), B, K,
                                  I, F, None, 1.0, _lib.VJP_FULL, P(outT), P(outP), P(outL),
                                  P(gB), P(gA), P(g0), P(g1), P(st), stream)
        if rc:
            _lib.check(rc, "fp_solve_vjp_f32")

    def fwd_step():
        rc = lib.fp_solve_f32(P(sc.basis), P(sc.anchor), P(sc.start), P(sc.end), P(T0), B, K, I, F,
                              P(outT), None, P(outP), P(outL), P(st), None, None, None, None, stream)
        if rc:
            _lib.check(rc, "fp_solve_f32")

    gate = torch.zeros(1, dtype=torch.int32).pin_memory()
    # (never with ranks sharing a device: their gates would wait on other contexts' time slices)
    use_gate = (K <= _lib.TILE_MAX_ORDER and args.policy in ("auto", "tile") and not args.no_gate
                and not (ws > 1 and args.backend == "gloo"))

    def timed(fn, steps, warmup, sampler=None):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        _barrier(ws)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        n0 = _lib.launch_count()
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            # Hold the stream until every timed step is enqueued (fp_gate_wait),
            # so host-side jitter cannot idle the device inside a timed step.
            # (Only when the dispatch has no host round trip: the bucketed path
            # synchronises on the stream to read its classification.)
            gate[0] = 0
            if use_gate:
                _lib.check(lib.fp_gate_wait(gate.data_ptr(), 10.0, stream), "fp_gate_wait")
            for e0, e1 in evs:
                e0.record()
                fn()
                e1.record()
            gate[0] = 1
            torch.cuda.synchronize()
        launches = _lib.launch_count() - n0
        _barrier(ws)
        ms = [e0.elapsed_time(e1) for e0, e1 in evs]
        return float(np.sum(ms)), ms, launches

    # FP32 roofline probe first: it also brings the SM clock up from idle
    # before the warm-up steps, so the first timed steps are not ramping.
    peak = measure_ffma_peak(lib, stream, dev) if rank == 0 else None
    peak_reg = (measure_ffma_peak(lib, stream, dev, register_operands=True)
                if rank == 0 and hasattr(lib, "fp_peak_ffma_reg") else None)

    # ---- fused forward + VJP step (the headline) ------------------------------
    sampler = ClockSampler(torch.cuda.current_device())
    tot_ms, ms_list, launches = timed(step, args.steps, args.warmup, sampler)
    conv = int(((st & _lib.STATUS_UNCONVERGED_MASK) == 0).sum().item())
    gates = gate_check(lib, sc, outT, st) if rank == 0 else None
    tot_ms_max = _max_over_ranks(tot_ms, ws, dev)
    conv_all = _sum_over_ranks(conv, ws, dev)
    paths_all = _sum_over_ranks(B, ws, dev)
    step_s = tot_ms_max * 1e-3 / args.steps
    value = conv_all / step_s
    raw = paths_all / step_s

    # ---- forward only ------------------------------------------------------------
    f_ms, f_list, _ = timed(fwd_step, args.steps, args.warmup)
    f_conv = int(((st & _lib.STATUS_UNCONVERGED_MASK) == 0).sum().item())
    f_step_s = _max_over_ranks(f_ms, ws, dev) * 1e-3 / args.steps
    f_conv_all = _sum_over_ranks(f_conv, ws, dev)

    # ---- roofline ------------------------------------------------------------------
    fl_fwd, fl_vjp = flops_per_path(K, I, F)
    avg_launch_s = float(np.mean(ms_list)) * 1e-3
    achieved = (fl_fwd + fl_vjp) * B / avg_launch_s / 1e12
    rd, wr = bytes_per_path(K)
    hbm_gbs = (rd + wr) * B / avg_launch_s / 1e9
    peaks = {}
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic = _load_ncu_traffic(K, B)
    ncu = _ncu_entry(K) or {}
    exec_flop = ncu.get("executed_flop_per_path")

    # ---- end to end through the host-buffer C-ABI entry ---------------------------------
    e2e = None
    if not args.no_e2e:
        pin = lambda shape, dt=torch.float32: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
        # Inputs: the scene (basis, anchor, TX, RX); the zero T0 is set on the
        # device (T0 = NULL). Outputs: T*, L*, the scene gradient and status;
        # the interaction points are not copied back (they follow from T*,
        # as the reference derives them on the host, bench.py:313-314).
        assert not host.T0.any()
        hin = [pin(tuple(host.basis.shape)), pin(tuple(host.anchor.shape)), pin((B, 3)), pin((B, 3))]
        for t, a in zip(hin, (host.basis, host.anchor, host.start, host.end)):
            t.numpy()[...] = a
        hout = [pin((B, K, 2)), None, pin((B,)), pin((B, K, 3, 2)), pin((B, K, 3)),
                pin((B, 3)), pin((B, 3)), pin((B,), torch.uint8)]
        h2d = sum(t.numel() * t.element_size() for t in hin)
        d2h = sum(t.numel() * t.element_size() for t in hout if t is not None)
        Pn = lambda t: None if t is None else t.data_ptr()  # noqa: E731

        def e2e_step():
            rc = lib.fp_solve_vjp_host_f32(*(P(t) for t in hin), None, B, K, I, F, 1.0, _lib.VJP_FULL,
                                           *(Pn(t) for t in hout), args.chunk, 3)
            if rc:
                _lib.check(rc, "fp_solve_vjp_host_f32")

        # Streaming through the public submit / wait API: step i is waited
        # for only after step i + lag was submitted, so later steps' host-to-
        # device copies and kernels are already queued while step i's results
        # stream out (lag + 1 output sets in flight). Every step still copies
        # its inputs in and its results out.
        lag = max(1, args.e2e_lag)
        hout2 = [hout] + [[None if t is None else pin(tuple(t.shape), t.dtype) for t in hout]
                          for _ in range(lag)]
        nsets = len(hout2)
        import ctypes

        def e2e_submit(i):
            tk = ctypes.c_uint64(0)
            rc = lib.fp_solve_vjp_host_submit_f32(*(P(t) for t in hin), None, B, K, I, F, 1.0,
                                                  _lib.VJP_FULL, *(Pn(t) for t in hout2[i % nsets]),
                                                  args.stream_chunk, args.stream_slots,
                                                  ctypes.addressof(tk))
            if rc:
                _lib.check(rc, "fp_solve_vjp_host_submit_f32")
            return tk.value

        def e2e_wait(tk):
            _lib.check(lib.fp_host_wait(tk), "fp_host_wait")

        e2e_step()
        _barrier(ws)
        e_steps = max(3, args.steps // 4)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        e_blocking_s = _max_over_ranks((time.perf_counter() - t0) / e_steps, ws, dev)
        e2e_wait(e2e_submit(0))
        _barrier(ws)
        t0 = time.perf_counter()
        pending = []
        for i in range(e_steps):
            pending.append(e2e_submit(i))
            if len(pending) > lag:
                e2e_wait(pending.pop(0))
        for tk in pending:
            e2e_wait(tk)
        e_s = _max_over_ranks((time.perf_counter() - t0) / e_steps, ws, dev)
        e_conv = int(((hout2[(e_steps - 1) % nsets][7] & _lib.STATUS_UNCONVERGED_MASK) == 0).sum().item())
        e2e = {"value": _sum_over_ranks(e_conv, ws, dev) / e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_s * 1e3, "raw_paths_per_s": paths_all / e_s,
               "path": ("fp_solve_vjp_host_submit_f32 + fp_host_wait (pinned host buffers; steps "
                        f"submitted back to back, each waited {lag} step(s) later; copy-in, compute and "
                        f"copy-out streams over {args.stream_slots} device chunk slots of up to {args.stream_chunk} "
                        "paths)"),
               "copies": ("in: basis, anchor, start, end (T0 = NULL: zero init on the device); "
                          "out: T, length, d_basis, d_anchor, d_start, d_end, status (points "
                          "skipped: derivable from T)"),
               "blocking": {"ms_per_step": e_blocking_s * 1e3,
                            "value": _sum_over_ranks(e_conv, ws, dev) / e_blocking_s,
                            "path": ("fp_solve_vjp_host_f32 (one blocking call per step; chunks of "
                                     f"{args.chunk} paths over 3 slots)")},
               "link": pcie_link(h2d, d2h, dev, e_s)}

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle.cpu_baseline import CpuPool

        (b, a, s0, s1, T0h), n, _ = cpu_sample(host, 1 << 12 if args.quick else args.sample)
        pool = CpuPool(kind="auto")
        pool.run(b[:pool.cores * 8], a[:pool.cores * 8], s0[:pool.cores * 8], s1[:pool.cores * 8],
                 T0h[:pool.cores * 8], I)  # warm the workers
        c, w = pool.run(b, a, s0, s1, T0h, I)
        pool.close()
        what = ("the reference package (oracle/_ref): _bfgs_kernel batched + per-path "
                "length_param_gradient + vjp_solution(gradient)" if pool.kind == "reference" else
                "numpy restatement (oracle/fermat_oracle.py): batched forward + per-path "
                "implicit gradient like the reference")
        cpu = {"value": c / w, "unit": UNIT, "cores": pool.cores, "kind": pool.kind,
               "sample": f"{n} paths (all {2 ** K} orderings equally) of this workload; {what}",
               "wall_s": w, "converged_fraction": c / n}

    n_devices = _devices_in_use(ws, dev)
    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "devices": n_devices,
            "backend": args.backend if ws > 1 else None, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy PCG64, SURVEY.md §8(d) generator)",
            "config": _config(K, I, B, ws),
            "raw_paths_per_s": raw, "converged_fraction": conv_all / paths_all,
            "fwd": {"value": f_conv_all / f_step_s, "raw_paths_per_s": paths_all / f_step_s,
                    "ms_per_step": f_step_s * 1e3, "unit": UNIT},
            "roofline": {
                "bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if peak else None, "traffic": traffic,
                "flop_per_path": fl_fwd + fl_vjp, "paths_per_launch": B,
                "peak_source": "FFMA microbenchmark (fp_peak_ffma) measured in this run; "
                               "MEASURED_PEAKS.json has no FP32 SIMT figure",
                # what the kernel really executes (ncu: FADD+FMUL+2 FFMA, paired
                # ops x2, of the committed capture) and the register-operand
                # FFMA2 ceiling measured in this run (fp_peak_ffma_reg)
                "executed_flop_per_path": exec_flop,
                "executed_achieved": (exec_flop * B / avg_launch_s / 1e12) if exec_flop else None,
                "peak_register_operands": peak_reg,
                "executed_frac_of_register_peak": (exec_flop * B / avg_launch_s / 1e12 / peak_reg)
                if (exec_flop and peak_reg) else None,
                "hbm": {"achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                        "frac": hbm_gbs / hbm_peak, "bytes_per_path": rd + wr},
            },
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "converged_gate": gates,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_scene(args):
    """--workload config3 / config4: exhaustive tracing in the synthetic city.

    config3: one step = enumerate + solve + bounds-mask + compact every
    candidate of order <= 3 (value: candidate paths/s, whole job).
    config4: one step = the config-3 trace plus the implicit VJP of sum 1/L^2
    over valid paths, gradient scatter, vertex chain rule and the NCCL
    all-reduce of the scene gradient (value: steps/s; ms_per_step reported).
    """
    import torch

    from paper_2510_16172_b200 import _lib
    from paper_2510_16172_b200.scene import (DeviceScene, blockers, candidate_count, make_urban_scene,
                                             trace, visibility)

    ws, rank, local, dev = _init_dist(args)
    _lib.set_kernel_policy(args.policy)
    grad = args.workload == "config4"
    sc = make_urban_scene(seed=0, alphabet=args.alphabet)
    ds = DeviceScene(sc)
    total = candidate_count(sc, 3)
    cap = 0 if args.no_records else None

    vis = args.visibility and not args.no_records
    blk = blockers(sc) if vis else None

    def step():
        r = trace(sc, max_order=3, iterations=args.iterations, capacity=cap, with_grad=grad,
                  device_scene=ds, points=vis, gather=args.gather)
        if vis:
            r.vis = [visibility(sc, o, device_scene=ds, blocker_array=blk)[0] for o in r.orders]
        return r

    peak = measure_ffma_peak(_lib.load(), torch.cuda.current_stream().cuda_stream, dev) if rank == 0 else None
    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    _barrier(ws)
    n0 = _lib.launch_count()
    sampler = ClockSampler(torch.cuda.current_device())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    _barrier(ws)
    ms = _max_over_ranks(e0.elapsed_time(e1), ws, dev) / args.steps
    n_devices = _devices_in_use(ws, dev)
    if rank == 0:
        per_order = [{"order": o.order, "candidates": o.candidates, "converged": o.converged,
                      "in_bounds": o.in_bounds, "valid": o.valid} for o in res.orders]
        line = {
            "metric": ("candidate paths/sec (exhaustive order<=3 tracing, enumerate+solve+mask+compact)"
                       if not grad else "inverse-design gradient steps/sec (trace + implicit VJP + allreduce)"),
            "value": (total / (ms * 1e-3)) if not grad else 1e3 / ms,
            "unit": "paths/s" if not grad else "steps/s",
            "n_gpus": ws, "devices": n_devices, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic city (paper_2510_16172_b200.scene.make_urban_scene, seed 0)",
            "config": {"workload": args.workload, "buildings": 16, "walls": int(sc.walls.shape[0]),
                       "objects": sc.n_objects, "alphabet": args.alphabet, "rx": int(sc.rx.shape[0]),
                       "candidates": total, "max_order": 3, "iterations": args.iterations,
                       "parallelism": f"dp{ws} (contiguous candidate shares)",
                       "records": ("none" if args.no_records else
                                   "all-gathered to every rank" if args.gather and ws > 1 else
                                   "sharded (kept on the rank that traced them)")},
            "orders": per_order, "valid_paths": res.valid, "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        # FP32 roofline of the whole step by the SURVEY §8(d) convention: every
        # candidate of order K costs the dense forward count at I iterations
        # (config 4 adds the VJP count for each valid path); this rank's share.
        flop = sum(o.candidates * flops_per_path(o.order, args.iterations)[0] for o in res.orders) / ws
        if grad:
            flop += sum(o.valid * flops_per_path(o.order, args.iterations)[1] for o in res.orders) / ws
        achieved = flop / (ms * 1e-3) / 1e12
        line["roofline"] = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                            "frac": achieved / peak if peak else None, "traffic": None,
                            "flop_per_step": flop,
                            "peak_source": "FFMA microbenchmark (fp_peak_ffma) measured in this run"}
        if grad:
            line["loss"] = res.loss
            line["grad_norm"] = float(torch.linalg.vector_norm(res.vertex_grad).item())
        if vis:
            # visibility stage alone (csrc/fp_visibility.cu), on the last step's records
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v0.record()
            for o in res.orders:
                visibility(sc, o, device_scene=ds, blocker_array=blk)
            v1.record()
            torch.cuda.synchronize()
            for d, o, f in zip(per_order, res.orders, res.vis):
                d["records"] = int(f.numel())
                d["visible"] = int((f == 0).sum().item())
                d["blocked"] = int(((f & _lib.VIS_BLOCKED) != 0).sum().item())
                d["wrong_side"] = int(((f & _lib.VIS_WRONG_SIDE) != 0).sum().item())
            nrec = sum(int(f.numel()) for f in res.vis)
            line["visibility"] = {"blockers": int(blk.shape[0]), "records": nrec,
                                  "ms": v0.elapsed_time(v1),
                                  "paths_per_s": nrec / max(v0.elapsed_time(v1) * 1e-3, 1e-12),
                                  "note": "included in ms_per_step (trace with points + visibility)"}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_config1(args):
    """--workload config1: diffraction-only K=1,2,3, 2^20 paths each; residual
    gradient norm vs iteration for the BFGS solver and the damped-Newton
    comparator (GPU; plus the reference's Newton restated on the CPU for a
    4096-path sample), iterations 5/10/20. value: BFGS paths/s at K=3, I=20."""
    import torch

    from paper_2510_16172_b200 import _lib, datagen
    from paper_2510_16172_b200.baselines import newton_batch
    from paper_2510_16172_b200.batching import BatchScene
    from paper_2510_16172_b200.solver import Precision, SolveOptions, solve
    from oracle import fermat_oracle as O

    torch.cuda.set_device(0)
    _lib.set_kernel_policy(args.policy)
    rows, value = [], None
    for K in (1, 2, 3):
        b = datagen.config1(K, args.paths if args.paths != 1 << 22 else 1 << 20)
        sc = BatchScene(b.basis, b.anchor, b.start, b.end)
        T0 = torch.zeros(b.size, K, 2, device="cuda")
        sub = slice(0, 4096)
        for I in (5, 10, 20):
            opts = SolveOptions(iterations=I, precision=Precision.SINGLE)
            tr = solve(sc, T0, SolveOptions(iterations=I, precision=Precision.SINGLE, record_trace=True))
            med_bfgs = torch.median(tr.trace_gnorm, dim=1).values.tolist()
            conv_b = float(tr.converged.float().mean().item())
            _, gN, tgN = newton_batch(sc, T0, opts, trace=True)
            med_newt = torch.median(tgN, dim=1).values.tolist()
            for _ in range(args.warmup):
                solve(sc, T0, opts, want_grad=False, want_points=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                solve(sc, T0, opts, want_grad=False, want_points=False)
            e1.record()
            torch.cuda.synchronize()
            bfgs_s = e0.elapsed_time(e1) * 1e-3 / args.steps
            e0.record()
            for _ in range(max(1, args.steps // 3)):
                newton_batch(sc, T0, opts)
            e1.record()
            torch.cuda.synchronize()
            newt_s = e0.elapsed_time(e1) * 1e-3 / max(1, args.steps // 3)
            ref = O.newton(b.basis[sub], b.anchor[sub], b.start[sub], b.end[sub], b.T0[sub], I,
                           np.float32, trace=True)
            med_ref = np.median(ref["trace_gnorm"], axis=1).tolist()
            rows.append({"K": K, "iterations": I, "paths": b.size,
                         "bfgs_median_grad_norm": med_bfgs, "newton_median_grad_norm": med_newt,
                         "reference_newton_cpu_median_grad_norm_4096": med_ref,
                         "bfgs_converged_fraction": conv_b,
                         "bfgs_paths_per_s": b.size / bfgs_s, "newton_paths_per_s": b.size / newt_s})
            if K == 3 and I == 20:
                value = b.size / bfgs_s
    line = {"metric": "paths/sec (diffraction-only BFGS, K=3, 20 it) + residual-gradient curves",
            "value": value, "unit": "paths/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (SURVEY §8(d) generator, D-only)",
            "config": {"workload": "config1: D-only K=1,2,3, 2^20 paths, I=5/10/20"}, "rows": rows}
    print(json.dumps(line), flush=True)
    return 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--iterations", type=int, default=20)
    ap.add_argument("--paths", type=int, default=1 << 22, help="paths per GPU")
    ap.add_argument("--sample", type=int, default=1 << 17, help="CPU baseline sample size")
    ap.add_argument("--chunk", type=int, default=1 << 19, help="e2e blocking call: pipeline chunk (paths)")
    ap.add_argument("--stream-chunk", type=int, default=1 << 22,
                    help="e2e submitted steps: pipeline chunk (paths; tools/e2e_pipe_sweep.py)")
    ap.add_argument("--stream-slots", type=int, default=2, help="e2e submitted steps: device chunk slots")
    ap.add_argument("--e2e-lag", type=int, default=1,
                    help="e2e submitted steps: step i is waited for after step i + lag was submitted")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="tiny CPU samples (debugging)")
    ap.add_argument("--policy", choices=("auto", "dense", "serial", "bucket", "tile"), default="auto",
                    help="kernel selection (fp_set_kernel_policy)")
    ap.add_argument("--workload", choices=("config1", "config2", "config3", "config4"),
                    default="config2")
    ap.add_argument("--alphabet", choices=("all", "walls"), default="all",
                    help="config3/4 objects: walls + edges (192) or the 64 walls only")
    ap.add_argument("--no-records", action="store_true", help="config3: counts only")
    ap.add_argument("--gather", action="store_true",
                    help="config3/4 under torchrun: all-gather every rank's path records (NCCL) "
                         "inside the timed step; default keeps them sharded")
    ap.add_argument("--visibility", action="store_true",
                    help="config3/4: also flag occluded / wrong-side paths (fp_visibility_f64)")
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl",
                    help="process group for N > 1 (gloo: ranks may share one GPU)")
    ap.add_argument("--no-gate", action="store_true",
                    help="do not hold the stream behind fp_gate_wait (for runs under ncu)")
    raw = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return _self_launch(args, raw)
    if args.workload in ("config3", "config4") and args.impl == "ours":
        return run_scene(args)
    if args.workload == "config1" and args.impl == "ours":
        return run_config1(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""Multi-rank runs of the real sharded code on one GPU (gloo process group).

The GPU pool gives one device, and NCCL refuses two ranks per device, so two
ranks share cuda:0 over gloo (collectives staged through host memory). The
ranks' kernels never wait on one another (paths are independent,
SPEC.md:253): this checks the sharding and the collectives, not scaling.

- scene tracing (configs 3/4): `trace(..., with_grad=True, gather=True)` on
  2 ranks returns the 1-rank valid set (same records, rank-major) and the
  all-reduced scene gradient within 1e-8 relative of the 1-rank sum;
- the config-2 fused step on a contiguous path shard per rank
  (`scene._share`, as bench.py assigns rows): the union of the shards is
  bitwise the 1-rank result;
- `bench.py --gpus 2 --backend gloo` (self-launched through
  torch.distributed.run) prints one JSON line with n_gpus 2 from two ranks.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from paper_2510_16172_b200.scene import make_urban_scene

    return make_urban_scene(seed=5, n_buildings=3, rx_grid=3, alphabet="all", side=80.0)


def _step_batch():
    from paper_2510_16172_b200 import datagen

    return datagen.gen_batch(77, datagen.all_orderings(3), 1000)  # 8000 paths


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2510_16172_b200.batching import BatchScene
    from paper_2510_16172_b200.scene import _share, gather_rows, trace
    from paper_2510_16172_b200.solver import Precision, SolveOptions, solve_with_gradients

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = trace(_scene(), max_order=3, iterations=20, with_grad=True, gather=True)
        recs = [(o.order, o.candidates, o.valid, o.rx.cpu().numpy(), o.seq.cpu().numpy(),
                 o.T.cpu().numpy(), o.length.cpu().numpy()) for o in res.orders]
        grad = (res.loss, res.tx_grad.cpu().numpy(), res.obj_grad.cpu().numpy(),
                res.vertex_grad.cpu().numpy())
        # config-2 step: rank r takes rows [lo, hi) of the batch
        b = _step_batch()
        lo, hi = _share(b.size, rank, world)
        sc = BatchScene(b.basis[lo:hi], b.anchor[lo:hi], b.start[lo:hi], b.end[lo:hi])
        r, g = solve_with_gradients(sc, b.T0[lo:hi], SolveOptions(iterations=20, precision=Precision.SINGLE))
        step = [t.cpu() for t in gather_rows([r.T, r.length, r.status, g.basis, g.anchor, g.start,
                                              g.end], world)]
        q.put((rank, recs, grad, [t.numpy() for t in step]))
    finally:
        dist.destroy_process_group()


def _one_rank():
    from paper_2510_16172_b200.batching import BatchScene
    from paper_2510_16172_b200.scene import trace
    from paper_2510_16172_b200.solver import Precision, SolveOptions, solve_with_gradients

    res = trace(_scene(), max_order=3, iterations=20, with_grad=True, rank=0, world=1)
    b = _step_batch()
    r, g = solve_with_gradients(BatchScene(b.basis, b.anchor, b.start, b.end), b.T0,
                                SolveOptions(iterations=20, precision=Precision.SINGLE))
    step = [t.cpu().numpy() for t in (r.T, r.length, r.status, g.basis, g.anchor, g.start, g.end)]
    return res, step


def test_two_ranks_shard_trace_and_step():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=600) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, ref_step = _one_rank()
    for rank, recs, (loss, tx, obj, vert), step in outs:
        for o, (k, cand, valid, rx, seq, T, L) in zip(ref.orders, recs):
            assert (k, cand, valid) == (o.order, o.candidates, o.valid)
            # the same valid paths (the kernel compacts in its own order: compare as sets of rows)
            key = lambda rx_, seq_: np.lexsort(np.column_stack([rx_, seq_]).T[::-1])  # noqa: E731
            a, b2 = key(rx, seq), key(o.rx.cpu().numpy(), o.seq.cpu().numpy())
            assert np.array_equal(rx[a], o.rx.cpu().numpy()[b2])
            assert np.array_equal(seq[a], o.seq.cpu().numpy()[b2])
            assert np.array_equal(T[a], o.T.cpu().numpy()[b2])  # per-path results are bitwise
            assert np.array_equal(L[a], o.length.cpu().numpy()[b2])
        # fp64 sums of fp32 per-path terms in a different order (two ranks,
        # atomics): equal to ~1e-9 relative (measured 2.4e-9 on the object
        # gradient, whose entries cancel)
        rel = lambda x, y: np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)  # noqa: E731
        assert abs(loss - ref.loss) <= 1e-9 * abs(ref.loss)
        assert rel(tx, ref.tx_grad.cpu().numpy()) <= 1e-8
        assert rel(obj, ref.obj_grad.cpu().numpy()) <= 1e-8
        assert rel(vert, ref.vertex_grad.cpu().numpy()) <= 1e-8
        for got, want in zip(step, ref_step):
            assert np.array_equal(got, want)


def test_bench_self_launch_two_ranks():
    """`bench.py --gpus 2` without torchrun relaunches itself with two ranks;
    rank 0 prints the one JSON line (gloo: both ranks on this GPU)."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--backend",
                          "gloo", "--steps", "3", "--warmup", "3", "--paths", str(1 << 16),
                          "--no-e2e"], capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["backend"] == "gloo" and line["devices"] == 1
    assert line["value"] > 0 and line["config"]["parallelism"] == "dp2 (independent path shards)"

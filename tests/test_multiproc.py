"""World-size-2 gloo tests of the multi-rank host logic (CPU, no GPU).

The data path has no collective: ranks own contiguous shares of every
candidate group (scene._share) or of the path axis (bench.py). The only
collectives are the sums of counters and of the config-4 scene gradient
(scene.reduce_sum / reduce_sum_many) and the optional gather of traced path
records (scene.gather_rows) — NCCL on the GPU box, gloo here.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_16172_b200.scene import _share, gather_rows, reduce_sum, reduce_sum_many


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # counters: each rank contributes its share of a 1000-candidate group
        lo, hi = _share(1000, rank, world)
        c = torch.tensor([hi - lo, rank + 1, 2 * rank, 7], dtype=torch.int64)
        tot = reduce_sum(c, world)
        # scene gradient: vertex (256,3), tx (3), loss (1), objects (192,9)
        g = [torch.full((256, 3), float(rank + 1)), torch.full((3,), 0.5 * rank),
             torch.tensor([1.0]), torch.arange(192 * 9, dtype=torch.float32).reshape(192, 9)]
        red = reduce_sum_many(g, world)
        # path records of different lengths per rank (rank 0: 3 rows, rank 1: 5 rows)
        n = 3 + 2 * rank
        rx = torch.arange(n, dtype=torch.int32) + 100 * rank
        seq = torch.stack([rx, rx + 1], dim=1)
        L = rx.to(torch.float32) * 0.5
        g_rx, g_seq, g_L = gather_rows([rx, seq, L], world)
        q.put((rank, tot.tolist(), [t.shape for t in red], float(red[0][0, 0]), float(red[1][0]),
               float(red[2][0]), float(red[3][1, 2]), g_rx.tolist(), g_seq.shape, g_L.tolist()))
    finally:
        dist.destroy_process_group()


def test_share_partitions_exactly():
    for total in (0, 1, 7, 1000, 2 ** 31 + 5):
        for world in (1, 2, 3, 8):
            spans = [_share(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_gloo_world2_reductions():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_rx = [0, 1, 2, 100, 101, 102, 103, 104]
    for rank, tot, shapes, v, t, l, o, g_rx, g_seq_shape, g_L in out:
        assert g_rx == want_rx and g_seq_shape == torch.Size([8, 2])
        assert g_L == [0.5 * x for x in want_rx]
        assert tot == [1000, 3, 2, 14]
        assert shapes == [torch.Size([256, 3]), torch.Size([3]), torch.Size([1]), torch.Size([192, 9])]
        assert v == 3.0 and t == 0.5 and l == 2.0 and o == 2 * 11.0

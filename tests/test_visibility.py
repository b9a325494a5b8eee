"""Visibility post-processing (occluding walls / roofs, reflection side test).

CPU tests pin the oracle (oracle/visibility_oracle.py) with known answers and
check the blocker construction; GPU tests compare the kernel
(csrc/fp_visibility.cu through fp_visibility_f64) with the oracle bit for bit
on traced paths of a small city and on constructed edge cases.
"""

import numpy as np
import pytest

from paper_2510_16172_b200.scene import blockers, make_urban_scene
from oracle import visibility_oracle as V

UNIT_WALL = np.array([[[0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [0.0, 0.0, 2.0]]])  # O, U, V: y = 0, x,z in [0,2]


def _flags(P, Q, blk=UNIT_WALL, e=1e-9):
    P, Q = np.atleast_2d(P).astype(np.float64), np.atleast_2d(Q).astype(np.float64)
    return V.crosses(P, Q - P, blk, e)[:, 0]


def test_segment_through_wall_is_blocked():
    assert _flags([1.0, -1.0, 1.0], [1.0, 1.0, 1.0])[0]


def test_segment_missing_or_parallel_or_touching_is_not_blocked():
    assert not _flags([3.0, -1.0, 1.0], [3.0, 1.0, 1.0])[0]    # passes beside the quad
    assert not _flags([1.0, -1.0, 2.5], [1.0, 1.0, 2.5])[0]    # passes above it
    assert not _flags([0.5, 0.0, 1.0], [1.5, 0.0, 1.0])[0]     # in its plane (det == 0)
    assert not _flags([1.0, -1.0, 1.0], [1.0, 0.0, 1.0])[0]    # ends on it (s = 1)
    assert not _flags([1.0, 0.0, 1.0], [1.0, 1.0, 1.0])[0]     # starts on it (s = 0)
    assert not _flags([1.0, 1.0, 1.0], [1.0, 2.0, 1.0])[0]     # stops short of it


def test_boundary_of_quad_counts_as_inside():
    # a = 0 exactly (through the O-V edge) and b = 1 exactly (through the top edge)
    assert _flags([0.0, -1.0, 1.0], [0.0, 1.0, 1.0])[0]
    assert _flags([1.0, -1.0, 2.0], [1.0, 1.0, 2.0])[0]


def test_wrong_side_reflection():
    # reflector = the unit wall (normal along y); TX and RX on the same side: fine
    basis = np.array([[[1.0, 0.0], [0.0, 0.0], [0.0, 1.0]]], np.float32)  # columns x, z
    plane = np.array([1], np.uint8)
    tx = np.array([0.0, -3.0, 1.0])
    rx = np.array([[2.0, -3.0, 1.0], [2.0, 3.0, 1.0]])
    pts = np.array([[[1.0, 0.0, 1.0]], [[1.0, 0.0, 1.0]]], np.float32)
    f, first = V.visibility(np.zeros((0, 3, 3)), tx, rx, np.array([0, 1]), pts,
                            rec_seq=np.array([[0], [0]]), obj_basis=basis, obj_plane=plane)
    assert f[0] == 0 and f[1] == V.WRONG_SIDE
    assert (first == -1).all()


def test_fp32_rounded_interaction_point_does_not_block_itself():
    # an interaction point on a wall 100 m away, rounded to fp32, sits ~1e-6 m off
    # the plane: the distance tolerance keeps the wall from blocking its own path
    blk = np.array([[[100.0, 30.0, 0.0], [0.0, 7.0, 0.0], [0.0, 0.0, 20.0]]])  # x = 100 plane
    tx = np.array([0.1, 0.3, 30.0])
    x = np.array([100.0, 33.3333333, 7.7777777])
    pts = np.array([[x]], np.float32)
    for rx in ([3.3, 61.7, 1.5], [3.3, 1.7, 1.5]):
        f, _ = V.visibility(blk, tx, np.array([rx]), np.array([0]), pts)
        assert f[0] == 0


def test_first_blocker_is_lowest_index_on_first_blocked_segment():
    blk = np.concatenate([UNIT_WALL, UNIT_WALL + [[0.0, -0.5, 0.0], [0, 0, 0], [0, 0, 0]]])
    tx = np.array([1.0, -1.0, 1.0])
    rx = np.array([[1.0, 1.0, 1.0]])
    pts = np.array([[[1.0, 0.5, 1.0]]], np.float32)  # segment 0 crosses both walls
    f, first = V.visibility(blk, tx, rx, np.array([0]), pts)
    assert f[0] == V.BLOCKED and first[0] == 0


def test_blockers_cover_walls_and_roofs():
    sc = make_urban_scene(seed=0)
    blk = blockers(sc)
    assert blk.shape == (64 + 16, 3, 3)
    # a wall parallelogram reproduces its quad corners
    w = sc.walls[5]
    assert np.allclose(blk[5, 0], w[0]) and np.allclose(blk[5, 0] + blk[5, 1], w[1])
    assert np.allclose(blk[5, 0] + blk[5, 2], w[3])
    assert np.allclose(blk[5, 0] + blk[5, 1] + blk[5, 2], w[2])
    # roofs are horizontal at each building's height and span its footprint
    roofs = blk[64:]
    assert np.allclose(roofs[:, 1:, :, ][:, :, 2], 0.0)
    for b in range(16):
        walls = sc.walls[4 * b:4 * b + 4]
        assert np.isclose(roofs[b, 0, 2], walls[0, 2, 2])
        corners = roofs[b, 0] + np.array([[0, 0], [1, 0], [1, 1], [0, 1]]) @ roofs[b, 1:]
        assert np.allclose(np.sort(corners[:, :2], axis=0), np.sort(walls[:, 2, :2], axis=0))


# ---------------------------------------------------------------- GPU ----
def _trace_small(order, seed=1):
    from paper_2510_16172_b200.scene import trace

    sc = make_urban_scene(seed=seed, n_buildings=6, rx_grid=6, side=120.0, alphabet="all")
    res = trace(sc, max_order=order, points=True)
    return sc, res


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2, 3])
def test_kernel_matches_oracle_on_traced_paths(order):
    from paper_2510_16172_b200.scene import visibility

    sc, res = _trace_small(order)
    r = res.orders[order - 1]
    assert r.valid > 0
    flags, first = visibility(sc, r)
    f_ref, first_ref = V.visibility(blockers(sc), sc.tx, sc.rx, r.rx.cpu().numpy(), r.points.cpu().numpy(),
                                    rec_seq=r.seq.cpu().numpy(), obj_basis=sc.obj_basis,
                                    obj_plane=sc.obj_plane)
    assert np.array_equal(flags.cpu().numpy(), f_ref)
    assert np.array_equal(first.cpu().numpy(), first_ref)
    if order >= 2:
        # the city occludes some paths and keeps others
        assert 0 < (f_ref & V.BLOCKED).astype(bool).sum() < len(f_ref)


@pytest.mark.gpu
def test_kernel_matches_oracle_on_edge_cases():
    """Segments aimed at quad edges, corners and the s = eps band, built directly as order-1 paths."""
    import torch

    from paper_2510_16172_b200 import _lib
    from paper_2510_16172_b200.batching import stream_ptr

    rng = np.random.default_rng(7)
    blk = np.concatenate([UNIT_WALL, [[[0.0, 0.0, 2.0], [2.0, 0.0, 0.0], [0.0, -2.0, 0.0]]]])  # wall + roof
    n = 4096
    a = rng.choice([0.0, 1.0, 0.5, 1e-17, 1 - 1e-16], size=n)
    b = rng.choice([0.0, 1.0, 0.25, 1 + 1e-16], size=n)
    hit = blk[0, 0] + a[:, None] * blk[0, 1] + b[:, None] * blk[0, 2]
    tx = np.array([1.0, -3.0, 1.0], np.float32)
    # point = interaction point of an order-1 path; RX beyond the wall on the line tx -> hit
    pts = (hit + rng.normal(size=(n, 3)) * [0.0, 1e-3, 0.0]).astype(np.float32)[:, None, :]
    rx = (2 * hit - tx + rng.normal(size=(n, 3))).astype(np.float32)
    rec_rx = np.arange(n, dtype=np.int32)
    f_ref, first_ref = V.visibility(blk, tx, rx, rec_rx, pts, eps=1e-4)
    dev = torch.device("cuda", 0)
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dt)).to(dev)  # noqa: E731
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    first = torch.empty(n, dtype=torch.int32, device=dev)
    lib = _lib.load()
    keep = [t(blk, np.float64), t(tx, np.float32), t(rx, np.float32), t(rec_rx, np.int32), t(pts, np.float32)]
    rc = lib.fp_visibility_f64(keep[0].data_ptr(), 2, keep[1].data_ptr(), keep[2].data_ptr(),
                               keep[3].data_ptr(), keep[4].data_ptr(), None, None, None, 0, n, 1, 1e-4,
                               flags.data_ptr(), first.data_ptr(), stream_ptr())
    assert rc == 0
    assert np.array_equal(flags.cpu().numpy(), f_ref)
    assert np.array_equal(first.cpu().numpy(), first_ref)
    assert 0 < f_ref.astype(bool).sum() < n

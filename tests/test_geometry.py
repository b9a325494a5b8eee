"""Host-side geometry types and their validation rules (no GPU).

The rules are the reference's (/root/reference/pkg/src/fermatpath/geometry.py:
43-165): plane columns nonzero and not parallel (cross-product test 1e-9),
edge second column exactly zero, 3-vector shapes, finite values, start and
end at least 1e-9 apart, at most MAX_INTERACTIONS (64) interactions, T of
shape (n, 2) and finite; embed is affine in T with the inert coordinate
dropping out exactly; params_from_points inverts embed on the active span.
"""

import numpy as np
import pytest

from paper_2510_16172_b200 import (DegenerateBasis, PathSpec, ShapeMismatch, Surface, SurfaceKind,
                                   embed, make_edge, make_plane, params_from_points)
from paper_2510_16172_b200.geometry import MAX_INTERACTIONS, check_params


def _two_hop():
    """TX -> plane (x-z span through the origin) -> edge -> RX."""
    return PathSpec(start=[-2.0, 3.0, 0.5], end=[2.5, 1.0, -0.5],
                    surfaces=(make_plane([0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]),
                              make_edge([1.0, 0.5, 0.0], [0.0, 2.0, 1.0])))


@pytest.mark.parametrize("build", [
    lambda: make_plane([0, 0, 0], [1, 0, 0], [3.0, 1e-11, 0.0]),          # parallel columns
    lambda: make_plane([0, 0, 0], [0, 1, 0], [0, -2.0, 0]),               # anti-parallel
    lambda: make_plane([0, 0, 0], [0, 0, 0], [1, 0, 0]),                  # zero first column
    lambda: make_plane([0, 0, 0], [1, 0, 0], [0, 0, 0]),                  # zero second column
    lambda: make_edge([1, 1, 1], [0, 0, 0]),                              # zero direction
    lambda: Surface(basis=np.array([[0.0, 1e-3], [1, 0], [0, 0]]), anchor=[0, 0, 0],
                    kind=SurfaceKind.EDGE),                               # edge column 2 not exactly 0
    lambda: Surface(basis=np.array([[np.nan, 0.0], [1, 0], [0, 0]]), anchor=[0, 0, 0],
                    kind=SurfaceKind.EDGE),                               # non-finite basis
])
def test_degenerate_bases_rejected(build):
    with pytest.raises(DegenerateBasis):
        build()


@pytest.mark.parametrize("build", [
    lambda: make_plane([0, 0], [1, 0, 0], [0, 1, 0]),                     # anchor not a 3-vector
    lambda: make_edge([0, 0, 0, 0], [1, 0, 0]),
    lambda: make_plane([0, np.inf, 0], [1, 0, 0], [0, 1, 0]),             # non-finite anchor
    lambda: Surface(basis=np.zeros((2, 2)), anchor=[0, 0, 0], kind=SurfaceKind.PLANE),
    lambda: PathSpec(start=[1, 2, 3], end=[1, 2, 3 + 1e-12], surfaces=()),  # coincident ends
    lambda: PathSpec(start=[0, 0, 0], end=[1, 0, 0],
                     surfaces=(make_edge([0, 1, 0], [1, 0, 0]),) * (MAX_INTERACTIONS + 1)),
])
def test_shape_and_range_violations_rejected(build):
    with pytest.raises(ShapeMismatch):
        build()


def test_valid_surfaces_and_masks():
    p = make_plane([0, 0, 0], [1, 0, 0], [0.0, 1.0, 1e-3])
    e = make_edge([4, 5, 6], [0, 0, 3])
    assert p.kind is SurfaceKind.PLANE and e.kind is SurfaceKind.EDGE
    assert p.active.tolist() == [True, True] and e.active.tolist() == [True, False]
    assert np.all(e.basis[:, 1] == 0.0)
    spec = PathSpec(start=[0, 0, 0], end=[1, 1, 1], surfaces=(make_edge([0, 0, 0], [1, 0, 0]),) * MAX_INTERACTIONS)
    assert spec.n == MAX_INTERACTIONS
    s = _two_hop()
    assert s.basis_tensor.shape == (2, 3, 2) and s.anchor_tensor.shape == (2, 3)
    assert s.active_mask.tolist() == [[True, True], [True, False]]
    assert s.scene_scale == pytest.approx(np.linalg.norm(np.subtract(s.end, s.start)))


def test_surfaces_are_read_only():
    p = make_plane([0, 0, 0], [1, 0, 0], [0, 1, 0])
    with pytest.raises(ValueError):
        p.basis[1, 1] = 5.0
    with pytest.raises(ValueError):
        p.anchor[0] = 1.0


def test_check_params():
    s = _two_hop()
    assert check_params(s, [[1, 2], [3, 4]]).dtype == np.float64
    for bad in (np.zeros((3, 2)), np.zeros((2, 3)), np.zeros(4)):
        with pytest.raises(ShapeMismatch):
            check_params(s, bad)
    for v in (np.nan, np.inf, -np.inf):
        T = np.zeros((2, 2))
        T[1, 0] = v
        with pytest.raises(ShapeMismatch):
            check_params(s, T)


def test_embed_is_affine_and_drops_inert_coordinates():
    s = _two_hop()
    rng = np.random.default_rng(0)
    for _ in range(25):
        T1, T2 = rng.uniform(-5, 5, (2, 2, 2))
        lam = rng.uniform()
        lhs = embed(s, lam * T1 + (1 - lam) * T2)
        rhs = lam * embed(s, T1) + (1 - lam) * embed(s, T2)
        assert np.allclose(lhs, rhs, atol=1e-12)
        P = embed(s, T1)
        assert np.array_equal(P[0], s.start) and np.array_equal(P[-1], s.end)
        for i, surf in enumerate(s.surfaces):
            assert np.allclose(P[i + 1], surf.basis @ T1[i] + surf.anchor, atol=1e-13)
        T3 = T1.copy()
        T3[1, 1] = rng.uniform(-1e8, 1e8)  # the edge's inert coordinate
        assert np.array_equal(embed(s, T3), P)


def test_params_from_points_inverts_embed():
    s = _two_hop()
    T = np.array([[0.25, -1.5], [0.75, 0.0]])
    back = params_from_points(s, embed(s, T)[1:-1])
    assert np.allclose(back, T, atol=1e-12)
    # off-surface points project onto the active span; inert coordinates stay 0
    back = params_from_points(s, embed(s, np.full((2, 2), 3.0))[1:-1] + 0.01)
    assert back[1, 1] == 0.0
    with pytest.raises(ShapeMismatch):
        params_from_points(s, np.zeros((2, 2)))

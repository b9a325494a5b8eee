"""CPU oracle for candidate enumeration and the bounds mask — TEST INFRASTRUCTURE ONLY.

The reference has no enumeration (SPEC.md:11 declares it out of scope; the
paper describes it in prose), so there are no golden vectors:
this restatement of the specification in csrc/fp_enum.cu / DESIGN.md is the
oracle ("parity unpinned" against the reference; pinned against itself by the
brute-force `itertools.product` + predicate cross-check in the tests).
"""

from __future__ import annotations

import itertools

import numpy as np


def patterns(order: int) -> list[int]:
    """Kind patterns of an order: bit j set = position j is a plane."""
    return list(range(1 << order))


def pattern_kinds(order: int, pattern: int) -> list[bool]:
    return [bool((pattern >> j) & 1) for j in range(order)]


def pattern_sequences(plane_ids, edge_ids, order: int, pattern: int) -> np.ndarray:
    """All object sequences of a pattern, no immediate repeat, lexicographic in list positions."""
    kinds = pattern_kinds(order, pattern)
    lists = [list(plane_ids) if k else list(edge_ids) for k in kinds]
    out = []
    for pos in itertools.product(*[range(len(l)) for l in lists]):
        if any(kinds[j] == kinds[j - 1] and pos[j] == pos[j - 1] for j in range(1, order)):
            continue
        out.append([lists[j][pos[j]] for j in range(order)])
    return np.array(out, dtype=np.int32).reshape(-1, order)


def brute_force_sequences(kinds_of_objects, order: int) -> set:
    """Independent check: every ordered sequence with no immediate repeat."""
    n = len(kinds_of_objects)
    return {seq for seq in itertools.product(range(n), repeat=order)
            if all(seq[j] != seq[j - 1] for j in range(1, order))}


def pattern_candidates(plane_ids, edge_ids, n_rx: int, order: int, pattern: int):
    """(rx, sequence) for every candidate of the group, RX-major."""
    seqs = pattern_sequences(plane_ids, edge_ids, order, pattern)
    rx = np.repeat(np.arange(n_rx, dtype=np.int32), len(seqs))
    return rx, np.tile(seqs, (n_rx, 1))


def inside_bounds(T, is_plane) -> np.ndarray:
    """|t_0| <= 1 and, for planes, |t_1| <= 1 for every interaction (B, K, 2) -> (B,)."""
    T = np.asarray(T)
    ok = np.abs(T[..., 0]) <= 1.0
    plane = np.asarray(is_plane, dtype=bool)
    ok &= ~plane | (np.abs(T[..., 1]) <= 1.0)
    return ok.all(axis=-1)

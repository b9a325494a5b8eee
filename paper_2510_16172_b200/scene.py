"""Exhaustive candidate tracing in a scene: enumeration, solve, bounds mask.

BASELINE configs 3 and 4 (no reference code: SPEC.md:11,90).
The scene is a set of objects — reflecting wall quads (centroid anchor,
half-extent basis, so a point is inside when |t| <= 1 per coordinate) and
diffraction edges (midpoint anchor, half-length direction) — plus one TX and a
grid of RX. Every ordered object sequence of order <= 3 with no immediate
repeat is a candidate for every RX; candidates are grouped by kind pattern and
each group runs one fused kernel (csrc/fp_enum.cu): decode -> solve -> bounds
mask -> compaction, optionally -> implicit VJP of sum 1/L^2 -> gradient
scatter. Ranks of a torch.distributed job take contiguous shares of every
group; NCCL (through torch.distributed) only sums the scene gradients and the
counters.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .batching import device, stream_ptr

WALL_COEF = np.array([  # (anchor, col0, col1) x (V0, V1, V2, V3)
    [0.25, 0.25, 0.25, 0.25],
    [-0.25, 0.25, 0.25, -0.25],
    [-0.25, -0.25, 0.25, 0.25]], dtype=np.float32)
VERT_EDGE_COEF = np.array([  # edge V0 -> V3: anchor, direction, (zero column)
    [0.5, 0.0, 0.0, 0.5],
    [-0.5, 0.0, 0.0, 0.5],
    [0.0, 0.0, 0.0, 0.0]], dtype=np.float32)
ROOF_EDGE_COEF = np.array([  # edge V3 -> V2
    [0.0, 0.0, 0.5, 0.5],
    [0.0, 0.0, 0.5, -0.5],
    [0.0, 0.0, 0.0, 0.0]], dtype=np.float32)


@dataclass
class UrbanScene:
    """Wall quads (W, 4, 3) + derived objects + TX + RX grid (host arrays)."""

    walls: np.ndarray
    tx: np.ndarray
    rx: np.ndarray
    alphabet: str = "all"
    obj_basis: np.ndarray = field(init=False)
    obj_anchor: np.ndarray = field(init=False)
    obj_plane: np.ndarray = field(init=False)
    vert_ids: np.ndarray = field(init=False)
    coef: np.ndarray = field(init=False)

    def __post_init__(self):
        self.walls = np.asarray(self.walls, np.float64)
        self.build_objects()

    def build_objects(self):
        """Objects as affine functions of the wall vertices (walls, vertical edges, roof edges)."""
        W = self.walls.shape[0]
        V = self.walls  # (W, 4, 3)
        kinds = [("wall", WALL_COEF)]
        if self.alphabet == "all":
            kinds += [("vedge", VERT_EDGE_COEF), ("redge", ROOF_EDGE_COEF)]
        elif self.alphabet != "walls":
            raise ValueError("alphabet must be 'all' or 'walls'")
        basis, anchor, plane, vids, coef = [], [], [], [], []
        for name, C in kinds:
            for w in range(W):
                a = C[0] @ V[w]
                b = np.stack([C[1] @ V[w], C[2] @ V[w]], axis=1)
                anchor.append(a)
                basis.append(b)
                plane.append(name == "wall")
                vids.append([4 * w + v for v in range(4)])
                coef.append(C)
        self.obj_basis = np.asarray(basis, np.float32)
        self.obj_anchor = np.asarray(anchor, np.float32)
        self.obj_plane = np.asarray(plane, bool)
        self.vert_ids = np.asarray(vids, np.int32)
        self.coef = np.asarray(coef, np.float32)

    @property
    def n_objects(self) -> int:
        return int(self.obj_plane.shape[0])

    @property
    def plane_ids(self) -> np.ndarray:
        return np.nonzero(self.obj_plane)[0].astype(np.int32)

    @property
    def edge_ids(self) -> np.ndarray:
        return np.nonzero(~self.obj_plane)[0].astype(np.int32)

    def with_vertices(self, walls, tx=None) -> "UrbanScene":
        return UrbanScene(walls, self.tx if tx is None else tx, self.rx, self.alphabet)


def make_urban_scene(seed: int = 0, n_buildings: int = 16, side: float = 200.0,
                     height=(10.0, 40.0), size=(10.0, 30.0), rx_grid: int = 32,
                     rx_height: float = 1.5, tx_height: float = 30.0, alphabet: str = "all",
                     gap: float = 4.0) -> UrbanScene:
    """Config 3's synthetic city: axis-aligned box buildings (4 wall quads each,
    random footprints in a side x side square, heights U[10, 40] m), one TX at
    30 m outside every footprint, a rx_grid x rx_grid RX grid at 1.5 m."""
    rng = np.random.default_rng([int(seed), 0xC17])
    half = side / 2.0
    boxes = []
    tries = 0
    while len(boxes) < n_buildings:
        tries += 1
        if tries > 100000:
            raise RuntimeError("could not place non-overlapping buildings")
        w, d = rng.uniform(*size, 2)
        cx = rng.uniform(-half + w / 2, half - w / 2)
        cy = rng.uniform(-half + d / 2, half - d / 2)
        box = (cx - w / 2, cy - d / 2, cx + w / 2, cy + d / 2)
        if any(box[0] < b[2] + gap and b[0] < box[2] + gap and box[1] < b[3] + gap and b[1] < box[3] + gap
               for b in boxes):
            continue
        boxes.append(box)
    heights = rng.uniform(*height, n_buildings)
    walls = []
    for (x0, y0, x1, y1), h in zip(boxes, heights):
        corners = [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]
        for k in range(4):
            (ax, ay), (bx, by) = corners[k], corners[(k + 1) % 4]
            walls.append([[ax, ay, 0.0], [bx, by, 0.0], [bx, by, h], [ax, ay, h]])
    while True:
        tx = np.array([*rng.uniform(-half, half, 2), tx_height])
        if not any(b[0] - gap <= tx[0] <= b[2] + gap and b[1] - gap <= tx[1] <= b[3] + gap
                   for b in boxes):
            break
    g = -half + (np.arange(rx_grid) + 0.5) * side / rx_grid
    gx, gy = np.meshgrid(g, g, indexing="ij")
    rx = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, rx_height)], axis=1)
    return UrbanScene(np.asarray(walls), tx, rx, alphabet)


def blockers(scene: UrbanScene) -> np.ndarray:
    """Occluders as parallelograms (Q, 3, 3) = (O, U, V), point = O + a U + b V, a, b in [0, 1].

    Every wall quad (O = V0, U = V1 - V0, V = V3 - V0) and, per building (four
    consecutive walls), its roof spanned by the first two walls' top edges.
    float64, from the scene's float64 vertices.
    """
    V = np.asarray(scene.walls, np.float64)
    out = [np.stack([V[:, 0], V[:, 1] - V[:, 0], V[:, 3] - V[:, 0]], axis=1)]
    nb = V.shape[0] // 4
    if nb:
        w0, w1 = V[0:4 * nb:4], V[1:4 * nb:4]
        out.append(np.stack([w0[:, 3], w0[:, 2] - w0[:, 3], w1[:, 2] - w1[:, 3]], axis=1))
    return np.ascontiguousarray(np.concatenate(out, axis=0))


def visibility(scene: UrbanScene, res: "OrderResult", eps: float = 1e-4, wrong_side: bool = True,
               device_scene: "DeviceScene | None" = None, blocker_array: np.ndarray | None = None):
    """Visibility flags of traced paths (csrc/fp_visibility.cu): (flags u8, first_blocker i32).

    flags bit 0 (VIS_BLOCKED): a segment crosses a wall or roof farther than
    `eps` metres from both its ends (the ends lie on the surfaces they interact
    with, up to the fp32 rounding of the points); bit 1 (VIS_WRONG_SIDE): a reflection whose neighbours are not on one
    side of the wall. `res` must carry points (trace(..., points=True)).
    """
    lib = _lib.load()
    if res.points is None:
        raise ValueError("visibility needs interaction points: trace(..., points=True)")
    ds = device_scene or DeviceScene(scene)
    dev = ds.basis.device
    blk = blockers(scene) if blocker_array is None else np.asarray(blocker_array, np.float64)
    blk_d = torch.from_numpy(np.ascontiguousarray(blk, np.float64)).to(dev)
    n = int(res.points.shape[0])
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    first = torch.empty(n, dtype=torch.int32, device=dev)
    if n:
        plane = torch.from_numpy(scene.obj_plane.astype(np.uint8)).to(dev)
        pts = res.points.contiguous()
        rc = lib.fp_visibility_f64(
            blk_d.data_ptr(), int(blk.shape[0]), ds.tx.data_ptr(), ds.rx.data_ptr(),
            res.rx.contiguous().data_ptr(), pts.data_ptr(),
            res.seq.contiguous().data_ptr() if wrong_side else None, ds.basis.data_ptr(),
            plane.data_ptr(), scene.n_objects, n, res.order, float(eps), flags.data_ptr(),
            first.data_ptr(), stream_ptr())
        _lib.check(rc, "fp_visibility_f64")
    return flags, first


def pattern_count(scene: UrbanScene, order: int, pattern: int) -> int:
    """Per-RX number of sequences of a kind pattern (fp_enum_pattern_count)."""
    lib = _lib.load()
    return int(lib.fp_enum_pattern_count(int(scene.obj_plane.sum()), int((~scene.obj_plane).sum()),
                                         order, pattern))


def candidate_count(scene: UrbanScene, max_order: int) -> int:
    return sum(pattern_count(scene, k, p) * scene.rx.shape[0]
               for k in range(1, max_order + 1) for p in range(1 << k))


@dataclass
class OrderResult:
    order: int
    candidates: int
    converged: int
    in_bounds: int
    valid: int
    rx: torch.Tensor | None = None       # (n,) int32
    seq: torch.Tensor | None = None      # (n, order) int32 object ids
    T: torch.Tensor | None = None        # (n, order, 2)
    length: torch.Tensor | None = None   # (n,)
    points: torch.Tensor | None = None   # (n, order, 3)


@dataclass
class TraceResult:
    orders: list
    loss: float | None = None
    obj_grad: torch.Tensor | None = None     # (N, 9): basis (3,2) row-major then anchor
    tx_grad: torch.Tensor | None = None      # (3,)
    vertex_grad: torch.Tensor | None = None  # (W*4, 3)

    @property
    def candidates(self) -> int:
        return sum(o.candidates for o in self.orders)

    @property
    def valid(self) -> int:
        return sum(o.valid for o in self.orders)


class DeviceScene:
    """Scene arrays resident on the GPU."""

    def __init__(self, scene: UrbanScene):
        dev = device()
        f = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)  # noqa: E731
        i = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev)  # noqa: E731
        self.scene = scene
        self.basis = f(scene.obj_basis)
        self.anchor = f(scene.obj_anchor)
        self.plane_ids = i(scene.plane_ids)
        self.edge_ids = i(scene.edge_ids)
        # non-empty placeholders keep the pointers valid when a kind is absent
        if self.plane_ids.numel() == 0:
            self.plane_ids = torch.zeros(1, dtype=torch.int32, device=dev)
        if self.edge_ids.numel() == 0:
            self.edge_ids = torch.zeros(1, dtype=torch.int32, device=dev)
        self.n_planes = int(scene.obj_plane.sum())
        self.n_edges = int((~scene.obj_plane).sum())
        self.tx = f(scene.tx)
        self.rx = f(scene.rx)
        self.vert_ids = i(scene.vert_ids)
        self.coef = f(scene.coef)


def _share(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous share [lo, hi) of `total` candidates for `rank` of `world`."""
    return total * rank // world, total * (rank + 1) // world


def _host_staged() -> bool:
    """gloo (the CPU tests, and ranks sharing one GPU) moves CPU tensors only:
    device tensors are staged through host memory for its collectives."""
    return torch.distributed.get_backend() == "gloo"


def reduce_sum(t: torch.Tensor, world: int) -> torch.Tensor:
    """Sum over ranks (NCCL on GPU tensors, gloo in the CPU tests); identity for one rank."""
    if world <= 1:
        return t
    out = t.detach().to("cpu", copy=True) if _host_staged() else t.clone()
    torch.distributed.all_reduce(out)
    return out.to(t.device)


def reduce_sum_many(ts, world: int):
    """One all-reduce over the concatenation of several tensors (the ~3 KB scene gradient)."""
    if world <= 1:
        return list(ts)
    flat = torch.cat([t.reshape(-1) for t in ts])
    dev = flat.device
    if _host_staged():
        flat = flat.cpu()
    torch.distributed.all_reduce(flat)
    flat = flat.to(dev)
    out, o = [], 0
    for t in ts:
        out.append(flat[o:o + t.numel()].reshape(t.shape))
        o += t.numel()
    return out


def gather_rows(ts, world: int):
    """All-gather per-rank row blocks of different lengths (the traced path
    records: rx, sequence, T, L, points), concatenated in rank order on every
    rank: the per-rank counts go first (one all_gather), then each field is
    padded to the longest block and all-gathered (NCCL on GPU tensors, gloo in
    the CPU tests). Identity for one rank."""
    if world <= 1:
        return list(ts)
    dist = torch.distributed
    dev = ts[0].device
    if _host_staged():
        return [t.to(dev) for t in gather_rows([t.cpu() for t in ts], world)] if dev.type != "cpu" \
            else _gather_rows(ts, world)
    return _gather_rows(ts, world)


def _gather_rows(ts, world: int):
    dist = torch.distributed
    dev = ts[0].device
    n = torch.tensor([ts[0].shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    out = []
    for t in ts:
        pad = t.new_zeros((m,) + tuple(t.shape[1:]))
        pad[:t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        out.append(torch.cat([b[:c] for b, c in zip(bufs, counts)]))
    return out


def decode_candidates(scene: UrbanScene, order: int, pattern: int, begin: int = 0, end: int | None = None):
    """(rx, sequence) of candidates [begin, end) of a (order, pattern) group, on the GPU."""
    lib = _lib.load()
    ds = DeviceScene(scene)
    total = pattern_count(scene, order, pattern) * scene.rx.shape[0]
    end = total if end is None else end
    n = max(0, end - begin)
    rx = torch.empty(n, dtype=torch.int32, device=ds.basis.device)
    seq = torch.empty(n, order, dtype=torch.int32, device=ds.basis.device)
    if n:
        rc = lib.fp_enum_decode(ds.plane_ids.data_ptr(), ds.n_planes, ds.edge_ids.data_ptr(),
                                ds.n_edges, scene.rx.shape[0], order, pattern, begin, end,
                                rx.data_ptr(), seq.data_ptr(), stream_ptr())
        _lib.check(rc, "fp_enum_decode")
    return rx, seq


def enumerate_candidates(num_objects: int, order: int, *, exclude_repeats: bool = True,
                         begin: int = 0, end: int | None = None, device=None) -> torch.Tensor:
    """Every object-index sequence (o_1 .. o_order), o_j in [0, num_objects),
    in lexicographic order, decoded on the GPU (SURVEY.md §8(b) "enumeration"):
    int32 (n, order) for the linear candidate range [begin, end).

    exclude_repeats: no immediate repeat (o_j != o_{j+1}; a path cannot
    interact with the same object twice in a row). The fused tracing kernel
    (`trace`) decodes the same indices on the fly and never materialises
    this list. Orders 1..3 (the tracing configs).
    """
    if not 1 <= order <= 3:
        raise ValueError("enumerate_candidates: order must be 1..3")
    if num_objects < 0:
        raise ValueError("num_objects must be >= 0")
    lib = _lib.load()
    n_obj = int(num_objects)
    total = n_obj * (n_obj - 1) ** (order - 1) if exclude_repeats else n_obj ** order
    end = total if end is None else int(end)
    if not 0 <= begin <= end <= total:
        raise ValueError(f"candidate range [{begin}, {end}) outside [0, {total})")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    seq = torch.empty(end - begin, order, dtype=torch.int32, device=dev)
    if end > begin:
        ids = torch.arange(n_obj, dtype=torch.int32, device=dev)
        # One kind everywhere: the decoder skips the previous object at every
        # position (no immediate repeat). Alternating kinds: consecutive
        # positions never share a kind, so nothing is skipped (plain product).
        pattern = (1 << order) - 1 if exclude_repeats else sum(1 << j for j in range(0, order, 2))
        rc = lib.fp_enum_decode(ids.data_ptr(), n_obj, ids.data_ptr(), n_obj, 1, order, pattern,
                                begin, end, None, seq.data_ptr(), stream_ptr())
        _lib.check(rc, "fp_enum_decode")
    return seq


def trace(scene: UrbanScene, max_order: int = 3, iterations: int = 20, fp_iters: int = 1,
          capacity: int | None = None, with_grad: bool = False, points: bool = False,
          rank: int | None = None, world: int | None = None, allreduce: bool = True,
          device_scene: DeviceScene | None = None, gather: bool = False) -> TraceResult:
    """Enumerate, solve and mask every candidate of order 1..max_order.

    capacity: records kept per order (default: all candidates of that order on
    this rank, capped at 2^26); 0 keeps counts only. with_grad: also the
    config-4 step (loss = sum 1/L^2 over valid paths and its gradient w.r.t.
    every object, TX and the wall vertices). Under torch.distributed, each
    rank takes a contiguous share of every group and (allreduce=True) the
    counters and gradients are summed over ranks with NCCL; gather=True also
    all-gathers every rank's path records (gather_rows), so each rank returns
    the whole job's valid paths (rank-major; within a rank the compaction
    order of the kernel). Otherwise records stay sharded.
    """
    lib = _lib.load()
    dist = torch.distributed
    if rank is None or world is None:
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(), dist.get_world_size()
        else:
            rank, world = 0, 1
    ds = device_scene or DeviceScene(scene)
    dev = ds.basis.device
    N, n_rx = scene.n_objects, scene.rx.shape[0]
    s = stream_ptr()
    grads = None
    if with_grad:
        # fp64 accumulators: per-path terms are fp32, their sums are not
        grads = dict(obj=torch.zeros(N, 9, dtype=torch.float64, device=dev),
                     tx=torch.zeros(3, dtype=torch.float64, device=dev),
                     loss=torch.zeros(1, dtype=torch.float64, device=dev))
    P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    counters = torch.zeros(max_order, 4, dtype=torch.int64, device=dev)
    recs = []
    for k in range(1, max_order + 1):
        groups = [(p, pattern_count(scene, k, p) * n_rx) for p in range(1 << k)]
        mine = sum(_share(tot, rank, world)[1] - _share(tot, rank, world)[0] for _, tot in groups)
        cap = min(mine, 1 << 26) if capacity is None else int(capacity)
        rec = dict(cap=cap, rx=torch.empty(cap, dtype=torch.int32, device=dev),
                   seq=torch.empty(cap, k, dtype=torch.int32, device=dev),
                   T=torch.empty(cap, k, 2, dtype=torch.float32, device=dev),
                   L=torch.empty(cap, dtype=torch.float32, device=dev),
                   pts=torch.empty(cap, k, 3, dtype=torch.float32, device=dev) if points else None)
        recs.append(rec)
        for p, tot in groups:
            lo, hi = _share(tot, rank, world)
            if hi <= lo:
                continue
            rc = lib.fp_enum_trace_f32(
                P(ds.basis), P(ds.anchor), P(ds.plane_ids), ds.n_planes, P(ds.edge_ids), ds.n_edges,
                P(ds.tx), P(ds.rx), n_rx, k, p, lo, hi, iterations, fp_iters, P(counters[k - 1]), cap,
                P(rec["rx"]) if cap else None, P(rec["seq"]) if cap else None,
                P(rec["T"]) if cap else None, P(rec["L"]) if cap else None,
                P(rec["pts"]) if cap else None,
                P(grads["obj"]) if grads else None, P(grads["tx"]) if grads else None, None,
                P(grads["loss"]) if grads else None, s)
            _lib.check(rc, "fp_enum_trace_f32")
    if with_grad:
        vg = torch.zeros(scene.walls.shape[0] * 4, 3, dtype=torch.float64, device=dev)
        rc = lib.fp_vertex_chain_f32(P(grads["obj"]), N, P(ds.vert_ids), P(ds.coef), P(vg), s)
        _lib.check(rc, "fp_vertex_chain_f32")
        if allreduce:
            # one NCCL all-reduce: wall vertices, TX, loss, object parameters (~10 KB)
            vg, grads["tx"], grads["loss"], grads["obj"] = reduce_sum_many(
                [vg, grads["tx"], grads["loss"], grads["obj"]], world)
    local = counters.cpu()
    total = (reduce_sum(counters, world) if allreduce else counters).cpu()
    orders = []
    for k, rec in zip(range(1, max_order + 1), recs):
        cand, conv, inb, valid = (int(x) for x in total[k - 1].tolist())
        n_keep = min(int(local[k - 1, 3]), rec["cap"])
        fields = [rec["rx"][:n_keep], rec["seq"][:n_keep], rec["T"][:n_keep], rec["L"][:n_keep]]
        if points:
            fields.append(rec["pts"][:n_keep])
        if gather and allreduce:
            fields = gather_rows(fields, world)
        orders.append(OrderResult(k, cand, conv, inb, valid, *fields[:4],
                                  fields[4] if points else None))
    res = TraceResult(orders)
    if with_grad:
        res.loss = float(grads["loss"].item())
        res.obj_grad, res.tx_grad, res.vertex_grad = grads["obj"], grads["tx"], vg
    return res

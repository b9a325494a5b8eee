"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only,
never copied) and records inputs and outputs of its public/internal entry
points on seeded inputs. The GPU box never runs this script; tests there only
read the committed .npz files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fermatpath import (  # noqa: E402  (reference package)
    Kinds,
    PathSpec,
    Precision,
    SolveOptions,
    bfgs_solve,
    gen_scenes,
    init_params,
    line_search_alpha,
    make_plane,
    reference_solve_batch,
)
from fermatpath.batching import BatchScene, embed_batch, path_length_batch  # noqa: E402
from fermatpath.implicit_diff import (  # noqa: E402
    grad_length_wrt_params,
    solve_stationary_system,
    vjp_solution,
)
from fermatpath.objective import gradient, hessian, length_param_gradient  # noqa: E402
from fermatpath.solver import _bfgs_kernel  # noqa: E402
from fermatpath.errors import FermatPathError  # noqa: E402
from fermatpath.baselines import _newton_kernel, image_points_batch  # noqa: E402

from paper_2510_16172_b200 import datagen  # noqa: E402

F32, F64 = Precision.SINGLE, Precision.DOUBLE


def _scene(batch):
    return BatchScene(batch.basis, batch.anchor, batch.start, batch.end)


def _spec_arrays(specs):
    sc = BatchScene.from_specs(specs)
    return sc.basis, sc.anchor, sc.start, sc.end


def _fwd(batch_arrays, T0, iters, fp, prec, trace=False):
    basis, anchor, start, end = batch_arrays
    sc = BatchScene(basis, anchor, start, end)
    opts = SolveOptions(iterations=iters, fixed_point_iters=fp, precision=prec,
                        record_trace=trace)
    T, g, traces, H = _bfgs_kernel(sc, T0, opts, return_state=True)
    L = path_length_batch(sc.astype(T.dtype), T)
    sc64 = sc.astype(np.float64)
    pts = embed_batch(sc64, np.asarray(T, np.float64))[:, 1:-1]
    out = dict(T=T, g=g, L=L, points=pts, H=H)
    if trace:
        out["trace_len"] = np.array([[t[1] for t in tr] for tr in traces]).T
        out["trace_gnorm"] = np.array([[t[2] for t in tr] for tr in traces]).T
    return out


def _specs_from_arrays(basis, anchor, start, end):
    from fermatpath import Surface, SurfaceKind

    specs = []
    for b in range(start.shape[0]):
        surfs = []
        for i in range(basis.shape[1]):
            A = np.asarray(basis[b, i], np.float64)
            kind = SurfaceKind.EDGE if np.all(A[:, 1] == 0.0) else SurfaceKind.PLANE
            surfs.append(Surface(basis=A, anchor=np.asarray(anchor[b, i], np.float64), kind=kind))
        specs.append(PathSpec(start=np.asarray(start[b], np.float64),
                              end=np.asarray(end[b], np.float64), surfaces=tuple(surfs)))
    return specs


def _grads_at(specs, Ts, rng):
    """Reference implicit-diff outputs per spec; NaN rows where it raises."""
    n = len(specs)
    K = specs[0].n
    res = {k: np.full(shape, np.nan) for k, shape in dict(
        full_basis=(n, K, 3, 2), full_anchor=(n, K, 3), full_start=(n, 3), full_end=(n, 3),
        env_basis=(n, K, 3, 2), env_anchor=(n, K, 3), env_start=(n, 3), env_end=(n, 3),
        vjp_basis=(n, K, 3, 2), vjp_anchor=(n, K, 3), vjp_start=(n, 3), vjp_end=(n, 3),
        u=(n, K, 2), v=(n, K, 2), hess=(n, 2 * K, 2 * K)).items()}
    res["stationary"] = np.zeros(n, dtype=bool)
    for j, (spec, T) in enumerate(zip(specs, Ts)):
        T = np.asarray(T, np.float64)
        v = rng.normal(size=(K, 2)) * spec.active_mask
        res["v"][j] = v
        try:
            env = grad_length_wrt_params(spec, T)
            g = gradient(spec, T)
            corr = vjp_solution(spec, T, g)
            part = length_param_gradient(spec, T)
            vj = vjp_solution(spec, T, v)
            u = solve_stationary_system(spec, T, v)
            H = hessian(spec, T)
        except FermatPathError:
            continue
        res["stationary"][j] = True
        res["full_basis"][j] = part.basis + corr.basis
        res["full_anchor"][j] = part.anchor + corr.anchor
        res["full_start"][j] = part.start + corr.start
        res["full_end"][j] = part.end + corr.end
        res["env_basis"][j], res["env_anchor"][j] = env.basis, env.anchor
        res["env_start"][j], res["env_end"][j] = env.start, env.end
        res["vjp_basis"][j], res["vjp_anchor"][j] = vj.basis, vj.anchor
        res["vjp_start"][j], res["vjp_end"][j] = vj.start, vj.end
        res["u"][j] = u
        res["hess"][j] = H
    return res


def main():
    meta = dict(numpy_version=np.__version__)
    out_files = {}

    # 1. config 0 (order-2 RD, 4096 paths, 10 iterations, fp32, zero init)
    c0 = datagen.config0()
    arrs = (c0.basis, c0.anchor, c0.start, c0.end)
    r = _fwd(arrs, c0.T0, 10, 1, F32)
    out_files["fwd_config0"] = dict(basis=c0.basis, anchor=c0.anchor, start=c0.start,
                                    end=c0.end, T0=c0.T0, iterations=10, fp_iters=1,
                                    T=r["T"], g=r["g"], L=r["L"], points=r["points"], H=r["H"])

    # 2. config-2 generator, every ordering K=1..5, 32 paths each, 20 it, fp32 + fp64
    for K in range(1, 6):
        b = datagen.gen_batch(100 + K, datagen.all_orderings(K), 32)
        arrs = (b.basis, b.anchor, b.start, b.end)
        r32 = _fwd(arrs, b.T0, 20, 1, F32)
        r64 = _fwd(arrs, b.T0, 20, 1, F64)
        d = dict(basis=b.basis, anchor=b.anchor, start=b.start, end=b.end, T0=b.T0,
                 iterations=20, fp_iters=1)
        for k in ("T", "g", "L", "points", "H"):
            d[k + "_f32"] = r32[k]
            d[k + "_f64"] = r64[k]
        # implicit gradients at the fp32 solution (fp64 arithmetic, the oracle contract)
        specs = _specs_from_arrays(*arrs)
        gr = _grads_at(specs, r32["T"], np.random.default_rng([7, K]))
        d.update({"grad_" + k: v for k, v in gr.items()})
        out_files[f"fwd_mixed_k{K}"] = d

    # 3. trace (record_trace), order 3, 8 orderings x 16 paths, 20 it fp32, F=2
    b = datagen.gen_batch(5, datagen.all_orderings(3), 16)
    r = _fwd((b.basis, b.anchor, b.start, b.end), b.T0, 20, 2, F32, trace=True)
    out_files["fwd_trace"] = dict(basis=b.basis, anchor=b.anchor, start=b.start, end=b.end,
                                  T0=b.T0, iterations=20, fp_iters=2, T=r["T"], g=r["g"],
                                  trace_len=r["trace_len"], trace_gnorm=r["trace_gnorm"])

    # 4. reference's own generator (well-conditioned), init_params start, F=4, 50 it
    for kinds in (Kinds.REFLECTIONS, Kinds.DIFFRACTIONS, Kinds.MIXED):
        for n in range(1, 6):
            specs = gen_scenes(41, n, kinds, 8)
            arrs = _spec_arrays(specs)
            T0 = np.stack([init_params(s) for s in specs])
            if kinds is Kinds.DIFFRACTIONS:
                # nonzero inert coordinates (criterion 3 scramble)
                T0[..., 1] = np.random.default_rng(n).normal(size=T0[..., 1].shape) * 10.0
            r64 = _fwd(arrs, T0, 50, 4, F64)
            r32 = _fwd(arrs, T0, 50, 4, F32)
            Tref, conv = reference_solve_batch(specs, list(T0))
            gr = _grads_at(specs, Tref, np.random.default_rng([9, n]))
            d = dict(basis=arrs[0], anchor=arrs[1], start=arrs[2], end=arrs[3], T0=T0,
                     iterations=50, fp_iters=4, Tref=Tref, ref_converged=conv)
            for k in ("T", "g", "L", "points"):
                d[k + "_f32"] = r32[k]
                d[k + "_f64"] = r64[k]
            d.update({"grad_" + k: v for k, v in gr.items()})
            if kinds is Kinds.REFLECTIONS:
                d["image_points"] = image_points_batch(BatchScene.from_specs(specs))
            Tn, gn = _newton_kernel(BatchScene.from_specs(specs), T0,
                                    SolveOptions(iterations=10, precision=F64))
            d["newton_T_f64"], d["newton_g_f64"] = Tn, gn
            out_files[f"refgen_{kinds.value}_n{n}"] = d

    # 5. known answers (test_solver.py:28-34,67-74,97-101)
    v_spec = PathSpec(start=[-1.0, 0.0, 0.0], end=[1.0, 0.0, 0.0],
                      surfaces=(make_plane([0.0, 0.0, 0.0], [1, 0, 0], [0, 1, 0]),))
    rep = bfgs_solve(v_spec, np.array([[0.5, 1.5]]))
    ls = line_search_alpha(v_spec, np.array([[0.0, 2.0]]), np.array([[0.0, -1.0]]), k=1)
    out_files["known_answers"] = dict(
        vpath_basis=v_spec.basis_tensor, vpath_anchor=v_spec.anchor_tensor,
        vpath_start=v_spec.start, vpath_end=v_spec.end, vpath_T0=np.array([[0.5, 1.5]]),
        vpath_T=rep.solution, vpath_L=rep.final_length, vpath_gnorm=rep.final_grad_norm,
        linesearch_alpha=ls)

    # 6. config 1 comparator: reference damped Newton vs BFGS on D-only batches
    for K in (1, 2, 3):
        b = datagen.gen_batch(K, ["D" * K], 256)
        arrs = (b.basis, b.anchor, b.start, b.end)
        d = dict(basis=b.basis, anchor=b.anchor, start=b.start, end=b.end, T0=b.T0)
        for it in (5, 10, 20):
            sc = _scene(b)
            Tn, gn = _newton_kernel(sc, b.T0, SolveOptions(iterations=it, precision=F32))
            d[f"newton_T_{it}"], d[f"newton_g_{it}"] = Tn, gn
            r = _fwd(arrs, b.T0, it, 1, F32)
            d[f"bfgs_T_{it}"], d[f"bfgs_g_{it}"] = r["T"], r["g"]
        out_files[f"config1_k{K}"] = d

    out_files.update(wide_fixtures())
    out_files.update(near_singular_fixture())
    for name, d in out_files.items():
        d = dict(d)
        d.update(meta)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
    total = sum(os.path.getsize(os.path.join(HERE, n + ".npz")) for n in out_files)
    print(f"wrote {len(out_files)} fixtures, {total / 1e6:.2f} MB")


def wide_fixtures():
    """7. orders 9..64 (the reference's MAX_INTERACTIONS; the warp-per-path solver):
    all-edge, all-plane and random R/D orderings, 100 iterations, fp32 + fp64,
    implicit gradients at the fp32 solution."""
    out = {}
    for K in (9, 12, 16, 33, 64):
        rng = np.random.default_rng([11, K])
        orders = ["D" * K, "R" * K] + ["".join(rng.choice(["R", "D"], size=K)) for _ in range(4)]
        b = datagen.gen_batch(900 + K, orders, 6)
        arrs = (b.basis, b.anchor, b.start, b.end)
        r32 = _fwd(arrs, b.T0, 100, 1, F32)
        r64 = _fwd(arrs, b.T0, 100, 1, F64)
        d = dict(basis=b.basis, anchor=b.anchor, start=b.start, end=b.end, T0=b.T0,
                 iterations=100, fp_iters=1)
        for k in ("T", "g", "L", "points"):
            d[k + "_f32"] = r32[k]
            d[k + "_f64"] = r64[k]
        specs = _specs_from_arrays(*arrs)
        gr = _grads_at(specs, r32["T"], np.random.default_rng([13, K]))
        d.update({"grad_" + k: v for k, v in gr.items() if k != "hess"})
        out[f"fwd_wide_k{K}"] = d
    return out


def near_singular_fixture():
    """8. _solve_sym's residual-check fallback (implicit_diff.py:55-71) on
    ill-conditioned active Hessians: a grazing reflection TX -> plane -> RX
    with TX/RX at height h over the plane z = 0 along the x axis and the
    plane's in-plane basis rotated by phi. At T* = 0 (exactly stationary by
    symmetry) H = R diag(2, 2 h^2 / (100 + h^2)) R^T / n, cond ~ 100 / h^2:
    from h ~ 1e-3 on, LAPACK's solution misses the 1e-8 (1 + |rhs|)
    residual bound and the reference re-solves with lambda = 1e-12 tr(H).
    K = 2 adds a well-conditioned second reflection after the grazing one
    (T* from reference_solve_batch). Records whether the fallback fired."""
    rng = np.random.default_rng(17)
    specs, Ts, fired = [], [], []
    for h in (1e-1, 1e-2, 1e-3, 3e-4, 1e-4, 3e-5):
        for phi in (0.3, 0.7854, 1.2):
            c, s = np.cos(phi), np.sin(phi)
            plane = make_plane([0.0, 0.0, 0.0], [c, s, 0.0], [-s, c, 0.0])
            specs.append(PathSpec(start=[-10.0, 0.0, h], end=[10.0, 0.0, h], surfaces=(plane,)))
            Ts.append(np.zeros((1, 2)))
    out = {}
    for K, group in ((1, (specs, Ts)),):
        sp, T = group
        arrs = _spec_arrays(sp)
        v = rng.normal(size=(len(sp), K, 2))
        u = np.stack([solve_stationary_system(s, t, vv) for s, t, vv in zip(sp, T, v)])
        for s, t, vv in zip(sp, T, v):
            H = hessian(s, t)
            x = np.linalg.solve(H, vv.ravel())
            fired.append(bool(np.linalg.norm(H @ x - vv.ravel()) > 1e-8 * (1 + np.linalg.norm(vv))))
        vj = [vjp_solution(s, t, vv) for s, t, vv in zip(sp, T, v)]
        out[f"near_singular_k{K}"] = dict(
            basis=arrs[0], anchor=arrs[1], start=arrs[2], end=arrs[3], T=np.stack(T), v=v, u=u,
            fired=np.array(fired), vjp_basis=np.stack([g.basis for g in vj]),
            vjp_anchor=np.stack([g.anchor for g in vj]), vjp_start=np.stack([g.start for g in vj]),
            vjp_end=np.stack([g.end for g in vj]))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--near-singular":
        meta = dict(numpy_version=np.__version__)
        for name, d in near_singular_fixture().items():
            d.update(meta)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
            print("wrote", name, "fallback fired on", int(d["fired"].sum()), "of", len(d["fired"]))
    elif len(sys.argv) > 1 and sys.argv[1] == "--wide":
        meta = dict(numpy_version=np.__version__)
        for name, d in wide_fixtures().items():
            d.update(meta)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
            print("wrote", name)
    else:
        main()

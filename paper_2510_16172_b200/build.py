"""Build the in-tree CUDA library `paper_2510_16172_b200/lib/libfermat_b200.so`.

Every translation unit is compiled for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`, IEEE div/sqrt, `-lineinfo`)
and linked into one shared library with a plain C ABI
(include/fermat_b200.h). The per-order kernel units build in parallel.

    python -m paper_2510_16172_b200.build [--force] [-j N]
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(REPO, "include")
OUT_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(OUT_DIR, "libfermat_b200.so")
OBJ_DIR = os.path.join(REPO, "build", "obj")

ORDERS = range(1, 9)
SPECIALISED_MAX_ORDER = 5  # fp_bucket.h kMaxSpecialisedOrder
TILE_MAX_ORDER = 5  # fp_abi.cu kMaxTileOrder (every mask of the order in one kernel)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC,
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build")
    return path


def _sources_digest() -> str:
    h = hashlib.sha256()
    for root in (CSRC, INCLUDE):
        for name in sorted(os.listdir(root)):
            if name.endswith((".cu", ".cuh", ".h")):
                with open(os.path.join(root, name), "rb") as fh:
                    h.update(name.encode())
                    h.update(fh.read())
    h.update(" ".join(ARCH + NVCC_FLAGS).encode())
    return h.hexdigest()


def _units(orders=ORDERS, obj_dir=None):
    obj_dir = obj_dir or OBJ_DIR
    units = [(os.path.join(CSRC, "fp_abi.cu"), os.path.join(obj_dir, "fp_abi.o"), [])]
    inst = os.path.join(CSRC, "fp_inst.cu")
    for k in orders:
        parts = (0, 1, 2) if k <= SPECIALISED_MAX_ORDER else (0,)
        if k <= TILE_MAX_ORDER:
            parts += (3, 4)
        for part in parts:
            units.append((inst, os.path.join(obj_dir, f"fp_inst_k{k}_p{part}.o"),
                          [f"-DFP_INST_K={k}", f"-DFP_INST_PART={part}"]))
    for extra in ("fp_enum.cu", "fp_bucket.cu", "fp_peak.cu", "fp_baselines.cu", "fp_visibility.cu",
                  "fp_wide.cu"):
        path = os.path.join(CSRC, extra)
        if os.path.exists(path):
            units.append((path, os.path.join(obj_dir, extra.replace(".cu", ".o")), []))
    # longest units first so the parallel build finishes sooner
    units.sort(key=lambda u: -sum(int(d.split("=")[1]) * (4 if ("FP_INST_PART=3" in " ".join(u[2]) or
                                                             "FP_INST_PART=4" in " ".join(u[2])) else 1)
                                  for d in u[2] if "FP_INST_K" in d))
    return units


def _compile(unit, extra=()):
    src, obj, defs = unit
    flags = NVCC_FLAGS
    if "-DFP_FMAD" in extra:  # A/B builds only: let nvcc contract mul + add
        flags = ["-fmad=true" if f == "-fmad=false" else f for f in flags]
    cmd = [nvcc(), *ARCH, *flags, *extra, *defs, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{res.stderr}")
    return obj


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    """Compile and link the library if sources changed; returns its path."""
    os.makedirs(OUT_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    stamp = os.path.join(OUT_DIR, ".build_digest")
    digest = _sources_digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == digest:
                return LIB
    units = _units()
    flags_stamp = os.path.join(OBJ_DIR, ".flags")
    flags = " ".join(ARCH + NVCC_FLAGS)
    same_flags = os.path.exists(flags_stamp) and open(flags_stamp).read() == flags
    headers = [os.path.join(d, n) for d in (CSRC, INCLUDE) for n in os.listdir(d)
               if n.endswith((".cuh", ".h"))]
    newest_header = max(os.path.getmtime(h) for h in headers)

    def stale(unit):
        # an object is reused only when it is newer than its source and every
        # shared header and was compiled with the same flags
        src, obj, _ = unit
        return (force or not same_flags or not os.path.exists(obj) or
                os.path.getmtime(obj) < max(os.path.getmtime(src), newest_header))

    todo = [u for u in units if stale(u)]
    jobs = jobs or max(1, min(len(todo), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        list(ex.map(_compile, todo))
    with open(flags_stamp, "w") as fh:
        fh.write(flags)
    objs = [u[1] for u in units]
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lcudart_static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(digest)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_variant(out: str, orders, defines=(), jobs=None) -> str:
    """Experimental library (subset of orders, extra -D flags) for A/B timing.

    Loaded instead of the default one with FERMAT_B200_LIB=<out>.
    """
    tag = os.path.splitext(os.path.basename(out))[0]
    obj_dir = os.path.join(REPO, "build", "variants", tag)
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    extra = [f"-D{d}" for d in defines]
    orders = list(orders)
    units = _units(orders, obj_dir)
    # orders missing from the variant still need their dispatch symbols: stub them
    stub = os.path.join(obj_dir, "stub.cu")
    with open(stub, "w") as fh:
        fh.write('#include "fp_kernels.cuh"\n#include "fp_dispatch.h"\nnamespace fp {\n')
        for k in ORDERS:
            if k in orders:
                continue
            for R in ("float", "double"):
                fh.write(f"template <> cudaError_t dispatch_dense<{R}, {k}>(const PathArgs<{R}>&, int, "
                         "cudaStream_t) { return cudaErrorNotSupported; }\n")
            if k <= TILE_MAX_ORDER:
                for R in ("float", "double"):
                    fh.write(f"template <> cudaError_t dispatch_tile<{R}, {k}>(const PathArgs<{R}>&, int, "
                             "cudaStream_t) { return cudaErrorNotSupported; }\n")
            if k <= SPECIALISED_MAX_ORDER:
                for fn in ("dispatch_masked_solve", "dispatch_masked_solve_vjp"):
                    fh.write(f"template <> cudaError_t {fn}<{k}>(const PathArgs<float>&, unsigned, "
                             "cudaStream_t) { return cudaErrorNotSupported; }\n")
        fh.write("}\n")
    units.append((stub, os.path.join(obj_dir, "stub.o"), []))
    jobs = jobs or min(len(units), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda u: _compile(u, extra), units))
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs, "-lcudart_static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--variant", help="output path of an experimental library")
    ap.add_argument("--orders", default="3", help="comma list of orders for --variant")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    args = ap.parse_args(argv)
    if args.variant:
        print(build_variant(args.variant, [int(k) for k in args.orders.split(",")], args.defines,
                            args.j))
        return
    build(force=args.force, jobs=args.j, verbose=True)


if __name__ == "__main__":
    sys.exit(main())

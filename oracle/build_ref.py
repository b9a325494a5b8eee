"""Install the genuine reference package into oracle/_ref — TEST/BENCH INFRASTRUCTURE.

The reference (`fermatpath`, /root/reference/pkg) is pure Python + numpy, so
"building" it is a plain offline pip install of its own sources into
``oracle/_ref`` (git-ignored, but not gpurun-ignored: it travels to the GPU
box with the built library). ``bench.py --impl reference`` then times the
reference's own code path on the box's host cores; the numpy restatement in
oracle/fermat_oracle.py stays as the bit-exact cross-check.

    python oracle/build_ref.py [--force]

Runs only where /root/reference exists (the build container); the tree is
read-only, so the install builds from a copy under /tmp. Nothing of the
reference is committed to this repository.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
TARGET = os.path.join(HERE, "_ref")


def installed() -> bool:
    return os.path.isfile(os.path.join(TARGET, "fermatpath", "solver.py"))


def build(force: bool = False) -> bool:
    """Install the reference into oracle/_ref; returns whether it is there."""
    if installed() and not force:
        return True
    if not os.path.isdir(REF_SRC):
        return installed()
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        stage = os.path.join(tmp, "target")
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", stage, src]
        res = subprocess.run(cmd, capture_output=True, text=True, cwd=tmp)
        if res.returncode != 0:
            print(res.stdout[-2000:], res.stderr[-2000:], file=sys.stderr)
            return installed()
        shutil.rmtree(TARGET, ignore_errors=True)
        shutil.copytree(stage, TARGET)
    return installed()


if __name__ == "__main__":
    ok = build(force="--force" in sys.argv)
    print(f"oracle/_ref: {'installed' if ok else 'unavailable'}")
    sys.exit(0 if ok else 1)

"""bench.py's reference arm runs on the CPU alone (no GPU needed): the line
keeps the contract's keys, times the reference package itself when
oracle/_ref is installed (else the bit-exact port), and cross-checks it with
the port (same converged count)."""

import json
import os
import subprocess
import sys

from oracle.cpu_baseline import reference_available

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--quick",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "paths/s"
    assert line["e2e"] == {"value": line["value"], "unit": "paths/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["cores"] >= 1
    if reference_available():
        assert cb["kind"] == "reference"
        assert cb["cross_check"]["equal"] is True
    else:
        assert cb["kind"] == "port"

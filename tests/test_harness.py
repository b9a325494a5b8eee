"""Harness host logic (no GPU): scene generator pinned to the reference, file formats, CLI."""

import io
import math

import numpy as np
import pytest

from paper_2510_16172_b200 import cli
from paper_2510_16172_b200.harness import (CSV_HEADER, BenchConfig, BenchRecord, Kinds, gen_scenes,
                                           load_scenes, read_records, save_scenes, write_records)

from parity import golden


@pytest.mark.parametrize("kinds", ["reflections", "diffractions", "mixed"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_gen_scenes_bit_exact_with_reference(kinds, n):
    """gen_scenes(41, n, kinds, 8) reproduces the reference's scenes bit for bit."""
    d = golden(f"refgen_{kinds}_n{n}")
    specs = gen_scenes(41, n, Kinds(kinds), 8)
    assert np.array_equal(np.stack([s.basis_tensor for s in specs]), d["basis"])
    assert np.array_equal(np.stack([s.anchor_tensor for s in specs]), d["anchor"])
    assert np.array_equal(np.stack([s.start for s in specs]), d["start"])
    assert np.array_equal(np.stack([s.end for s in specs]), d["end"])


def test_gen_scenes_properties():
    a, b = gen_scenes(7, 3, Kinds.MIXED, 5), gen_scenes(7, 3, Kinds.MIXED, 5)
    assert all(np.array_equal(x.basis_tensor, y.basis_tensor) for x, y in zip(a, b))
    assert not np.array_equal(gen_scenes(7, 3, Kinds.MIXED, 1)[0].start,
                              gen_scenes(8, 3, Kinds.MIXED, 1)[0].start)
    for spec in gen_scenes(9, 4, Kinds.MIXED, 3):
        kinds = [s.kind for s in spec.surfaces]
        assert all(x is not y for x, y in zip(kinds, kinds[1:]))
    with pytest.raises(ValueError):
        gen_scenes(0, 0, Kinds.MIXED, 1)


def test_yaml_and_csv_roundtrip():
    specs = gen_scenes(10, 2, Kinds.MIXED, 4)
    buf = io.StringIO()
    save_scenes(specs, buf)
    buf.seek(0)
    back = load_scenes(buf)
    for x, y in zip(specs, back):
        assert np.array_equal(x.basis_tensor, y.basis_tensor)
        assert np.array_equal(x.anchor_tensor, y.anchor_tensor)
        assert [s.kind for s in x.surfaces] == [s.kind for s in y.surfaces]
    recs = [BenchRecord("ours", 3, "mixed", 2, 100, 1, "single", 1.25e-4, 17.125),
            BenchRecord("image", 1, "reflections", 2, 0, 0, "double", float("nan"), 0.5)]
    buf = io.StringIO()
    write_records(recs, buf)
    assert buf.getvalue().splitlines()[0] == ",".join(CSV_HEADER)
    buf.seek(0)
    back = read_records(buf)
    assert back[0] == recs[0] and math.isnan(back[1].mean_error)
    with pytest.raises(ValueError):
        read_records(io.StringIO("a,b,c\n1,2,3\n"))


def test_bench_config_validation():
    for bad in (dict(solvers=("warp",)), dict(kinds=Kinds.MIXED, solvers=("image",)), dict(batch=0),
                dict(n_range=(0,))):
        with pytest.raises(ValueError):
            BenchConfig(seed=0, **bad)


def test_cli_gen_and_usage_errors(tmp_path, capsys):
    out = tmp_path / "s.yaml"
    assert cli.main(["gen", "--n", "2", "--count", "3", "--out", str(out)]) == 0
    with open(out) as fh:
        assert len(load_scenes(fh)) == 3
    assert cli.main(["gen", "--count", "0", "--out", str(out)]) == cli.USAGE_ERROR
    with pytest.raises(SystemExit) as e:
        cli.main(["bench", "--kinds", "nonsense"])
    assert e.value.code == cli.USAGE_ERROR
    assert cli.main(["grad-check", "--count", "0"]) == cli.USAGE_ERROR
    assert cli.main(["solve", str(tmp_path / "missing.yaml")]) == cli.USAGE_ERROR
    assert cli.main(["bench", "--solvers", "image", "--kinds", "mixed"]) == cli.USAGE_ERROR

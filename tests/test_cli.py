"""CLI mirror: same diagnostics/exit codes as the reference CLI (checked
against the reference package where importable), and `eval` writes the
container the reference writes (GPU)."""

import subprocess
import sys
from pathlib import Path

import pytest

from helpers import GOLDEN, manifest

ROOT = Path(__file__).resolve().parent.parent


def _cli(*args, module="paper_1804_10120_b200", env=None):
    return subprocess.run([sys.executable, "-m", module, *args], capture_output=True, text=True,
                          cwd=ROOT, timeout=600, env=env)


@pytest.mark.parametrize("k", range(len(manifest()["bad_programs"])))
def test_check_diagnostics_and_exit_code(k, tmp_path, capsys):
    from paper_1804_10120_b200.cli import main

    src = manifest()["bad_programs"][k]["source"]
    f = tmp_path / "p.tl"
    f.write_text(src)
    assert main(["check", str(f)]) == 1
    want = [f"{f}:{ln}:{col}: {msg}" for ln, col, msg in manifest()["bad_programs"][k]["diagnostics"]]
    assert capsys.readouterr().err.splitlines() == want


def test_check_validation_codes_and_io_errors(tmp_path):
    f = tmp_path / "p.tl"
    f.write_text("tensor A dim 3 rank 2;\nA(i, i) = 0;\n")
    res = _cli("check", str(f))
    assert res.returncode == 1 and "[repeated-lhs-index]" in res.stderr
    assert _cli("check", str(tmp_path / "missing.tl")).returncode == 2
    f.write_text(manifest()["cases"]["c4_p2"]["source"])
    assert _cli("check", str(f)).returncode == 0


def test_check_matches_reference_cli(tmp_path):
    pytest.importorskip("tlang.cli")
    import os

    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
    for src in (manifest()["cases"]["c4_p3"]["source"], "tensor A dim 3 rank 1;\nA(i) = B(i);\n",
                "tensor A dim 3 rank 1;\ntensor B dim 3 rank 2;\nA(i) = B(i);\n"):
        f = tmp_path / "p.tl"
        f.write_text(src)
        mine, ref = _cli("check", str(f)), _cli("check", str(f), module="tlang.cli", env=env)
        assert (mine.returncode, mine.stderr) == (ref.returncode, ref.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c4_p3", "c2_maxwell", "seq_augmented",
                                  "fused_literal_div_zero", "augmented_div_after_literal",
                                  "mixed_gridsize_read_before_resize",
                                  "mixed_gridsize_resize_first_use"])
@pytest.mark.parametrize("per_component", [False, True])
def test_eval_writes_the_reference_container(case, per_component, tmp_path):
    from paper_1804_10120_b200 import tldf

    spec = manifest()["cases"][case]
    f = tmp_path / "p.tl"
    f.write_text(spec["source"])
    out = tmp_path / "out.tldf"
    args = ["eval", str(f), "--data", str(GOLDEN / f"{case}.in.tldf"), "--out", str(out)]
    res = _cli(*args, *(["--per-component"] if per_component else []))
    assert res.returncode == 0, res.stderr
    # expected bytes: the input container with every target replaced by the
    # reference's output, in the same order (reference cli.py:77-104)
    env = tldf.read(GOLDEN / f"{case}.in.tldf", device="cpu")
    for name, fld in tldf.read(GOLDEN / f"{case}.out.tldf", device="cpu").items():
        env[name] = fld
    assert out.read_bytes() == tldf.dumps(env)


@pytest.mark.gpu
def test_eval_stops_where_the_reference_stops(tmp_path):
    # reference cli.py:96-102: an EvalError part-way through the program is a
    # diagnostic (EXIT_DIAGNOSTICS = 1, "<file>: <message>"), and no output is
    # written
    spec = manifest()["cases"]["error_after_first_statement"]
    f = tmp_path / "p.tl"
    f.write_text(spec["source"])
    out = tmp_path / "out.tldf"
    res = _cli("eval", str(f), "--data", str(GOLDEN / "error_after_first_statement.in.tldf"),
               "--out", str(out))
    assert res.returncode == 1
    assert res.stderr == f"{f}: {spec['raises']['message']}\n"
    assert not out.exists()


def test_bench_extended_row_arithmetic():
    # SURVEY.md §5 metrics: the device columns appended by `bench --extended`
    from paper_1804_10120_b200.bench import CSV_COLUMNS, EXT_COLUMNS, BenchResult

    r = BenchResult("s1_dtg", "whole-tensor", 1 << 20, 1e-3, 0.0, 22, 1, 176, 24)
    gpus, pts, hbm, frac, fp = r.extended_row(6455.0, 18400.0)
    assert gpus == 1 and pts == (1 << 20) / 1e-3
    assert hbm == 176 * (1 << 20) / 1e-3 / 1e9 and frac == hbm / 6455.0
    assert fp == 24 * (1 << 20) / 1e-3 / 1e9 / 18400.0
    assert len(CSV_COLUMNS + EXT_COLUMNS) == 12


@pytest.mark.gpu
@pytest.mark.parametrize("extended", [False, True])
def test_bench_subcommand_columns(tmp_path, extended):
    import json
    import subprocess
    import sys

    from paper_1804_10120_b200.bench import CSV_COLUMNS, DTG, EXT_COLUMNS

    src = tmp_path / "dtg.tl"
    src.write_text(DTG)
    cmd = [sys.executable, "-m", "paper_1804_10120_b200", "bench", "--file", str(src),
           "--grids", "4096", "--reps", "3", "--json"] + (["--extended"] if extended else [])
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    (row,) = json.loads(res.stdout)
    want = CSV_COLUMNS + (EXT_COLUMNS if extended else ())
    assert tuple(row) == want
    if extended:
        assert row["gpus"] == 1 and row["points_per_s"] > 0 and 0 < row["roofline_frac"] < 2

"""CLI harness (SPEC cli module) on the host: argument parsing and the usage-error exit code
(2), which are decided before any device work."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1111_6900_b200 import cli  # noqa: E402


@pytest.mark.parametrize("argv", [[], ["mul"], ["mul", "a"], ["echelonize", "x"], ["bench", "gemm", "2", "8"],
                                  ["mul", "a", "b", "c", "--backend", "winograd"], ["random", "2", "x", "3", "1", "o"]])
def test_usage_errors_exit_2(argv):
    with pytest.raises(SystemExit) as exc:
        cli.main(argv)
    assert exc.value.code == 2


@pytest.mark.parametrize("argv", [["selftest", "--e", "11"], ["selftest", "--sizes", "0"], ["selftest", "--e", "x"],
                                  ["random", "11", "2", "2", "1", "out.mat"], ["random", "4", "2", "2", "1", "o", "--f", "15"],
                                  ["bench", "mul", "1", "8"], ["mul", "/nonexistent/a.mat", "b", "c"],
                                  ["echelonize", "/nonexistent/a.mat", "out"]])
def test_bad_values_exit_2(argv, tmp_path):
    argv = [a if a not in ("out.mat", "o") else str(tmp_path / a) for a in argv]
    assert cli.main(argv) == 2


def test_crossover_env_must_be_int(monkeypatch):
    monkeypatch.setenv("GF2E_CROSSOVER", "big")
    with pytest.raises(cli.UsageError):
        cli._crossover(cli.build_parser().parse_args(["echelonize", "a", "b"]))
    monkeypatch.setenv("GF2E_CROSSOVER", "64")
    assert cli._crossover(cli.build_parser().parse_args(["echelonize", "a", "b"])) == 64
    assert cli._crossover(cli.build_parser().parse_args(["echelonize", "a", "b", "--crossover", "16"])) == 16


def test_module_help():
    out = subprocess.run([sys.executable, "-m", "paper_1111_6900_b200", "--help"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0
    for cmd in ("random", "mul", "echelonize", "selftest", "bench"):
        assert cmd in out.stdout

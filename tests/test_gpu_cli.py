"""CLI harness on the device (SPEC cli examples): files round-trip, identity products,
backend equivalence and counts, echelon ranks, self-test, and the bench line format."""

import os
import re
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def g():
    import torch

    import paper_1111_6900_b200 as g

    torch.cuda.set_device(0)
    return g


def _write(g, path, arr, e):
    g.save_matrix(path, g.PackedMatrix.from_array(g.field_new(e), np.asarray(arr, dtype=np.uint16)))


def test_random_deterministic(g, tmp_path):
    from paper_1111_6900_b200 import cli

    a, b = tmp_path / "a.mat", tmp_path / "b.mat"
    assert cli.main(["random", "8", "37", "70", "5", str(a)]) == 0
    assert cli.main(["random", "8", "37", "70", "5", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    M = g.load_matrix(str(a))
    assert M == g.PackedMatrix.random(g.field_new(8), 37, 70, 5)
    assert cli.main(["random", "3", "4", "5", "1", str(b), "--repr", "sliced"]) == 0
    assert b.read_text().startswith("gf2e-mat v1 e=3 f=b rows=4 cols=5 repr=sliced\n")


def test_mul_identity_and_backends(g, tmp_path, capsys):
    from paper_1111_6900_b200 import cli

    a, eye, out = str(tmp_path / "a.mat"), str(tmp_path / "i.mat"), str(tmp_path / "o.mat")
    assert cli.main(["random", "5", "70", "70", "9", a]) == 0
    _write(g, eye, np.eye(70), 5)
    assert cli.main(["mul", a, eye, out]) == 0
    assert open(out).read() == open(a).read()
    outs = {}
    for b in ("cubic", "nj", "strassen", "karatsuba"):
        p = str(tmp_path / f"{b}.mat")
        assert cli.main(["mul", a, a, p, "--backend", b, "--crossover", "16"]) == 0
        outs[b] = open(p).read()
    assert len(set(outs.values())) == 1
    x2 = str(tmp_path / "x2.mat")
    assert cli.main(["random", "2", "3", "3", "1", x2]) == 0
    capsys.readouterr()
    assert cli.main(["mul", x2, x2, out, "--counts"]) == 0
    assert "gf2_matmul_count=3" in capsys.readouterr().err


def test_mul_mismatch_exit_2(g, tmp_path):
    from paper_1111_6900_b200 import cli

    a, b, c = str(tmp_path / "a.mat"), str(tmp_path / "b.mat"), str(tmp_path / "c.mat")
    assert cli.main(["random", "4", "3", "5", "1", a]) == 0
    assert cli.main(["random", "4", "4", "5", "1", b]) == 0
    assert cli.main(["mul", a, b, str(tmp_path / "o.mat")]) == 2  # inner dimensions
    assert cli.main(["random", "3", "5", "5", "1", c]) == 0
    assert cli.main(["mul", a, c, str(tmp_path / "o.mat")]) == 2  # fields
    with open(b, "w") as fh:
        fh.write("gf2e-mat v1 e=4 f=13 rows=1 cols=2 repr=packed\n1 10\n")  # entry 16 >= 2^4
    assert cli.main(["mul", a, b, str(tmp_path / "o.mat")]) == 2


def test_echelonize_ranks(g, tmp_path, capsys):
    from paper_1111_6900_b200 import cli

    eye, zero, rnd = (str(tmp_path / f"{x}.mat") for x in ("i", "z", "r"))
    _write(g, eye, np.eye(40), 6)
    _write(g, zero, np.zeros((30, 50)), 6)
    assert cli.main(["random", "6", "90", "64", "3", rnd]) == 0
    res = {}
    for name, path in (("i", eye), ("z", zero), ("r", rnd)):
        for backend in ("nj", "ple"):
            capsys.readouterr()
            out = str(tmp_path / f"{name}_{backend}.mat")
            assert cli.main(["echelonize", path, out, "--full", "--backend", backend]) == 0
            res[name, backend] = (capsys.readouterr().out.strip(), open(out).read())
    assert res["i", "ple"][0] == "rank=40" and res["z", "ple"][0] == "rank=0" and res["r", "ple"][0] == "rank=64"
    for name in ("i", "z", "r"):
        assert res[name, "nj"] == res[name, "ple"]
    assert res["i", "ple"][1] == open(eye).read()


def test_selftest_passes(g, tmp_path):
    from paper_1111_6900_b200 import cli

    assert cli.main(["selftest", "--e", "2,5,8,10", "--sizes", "1,63,65,130", "--iters", "2",
                     "--out-dir", str(tmp_path)]) == 0
    assert not list(tmp_path.iterdir())


def test_bench_line(g, capsys):
    from paper_1111_6900_b200 import cli

    for op, muls in (("mul", "9"), ("addmul", "9"), ("ple", "na"), ("echelonize", "na"), ("trsm", "na")):
        capsys.readouterr()
        assert cli.main(["bench", op, "4", "300", "--reps", "2"]) == 0
        line = capsys.readouterr().out.strip()
        assert re.fullmatch(rf"bench op={op} e=4 n=300 reps=2 median_s=\d+\.\d+ gf2_muls={muls}", line), line

"""SURVEY §8f consumers of the hot path on device: triangular solves (the reference's
recursive TRSM, whose updates are addmul calls), sliced mul_by_x, packed scalar_mul.
Bit-exact against fixtures produced by the reference (tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch

    import paper_1111_6900_b200 as g

    torch.cuda.set_device(0)
    return g


def _tags(golden, key):
    return [str(t) for t in golden[key]]


def test_trsm_golden(g, golden):
    for tag in _tags(golden, "trsm_tags"):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        U = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/U"], m)
        L = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/L"], m)
        for fn, key, T in ((g.trsm_upper_left, "XU", U), (g.trsm_lower_left, "XL", L),
                           (g.trsm_lower_left_unit, "XLu", L)):
            B = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B"], n)
            fn(T, B)
            assert np.array_equal(B.to_numpy(), golden[f"{tag}/{key}"]), (tag, key)


@pytest.mark.parametrize("e,m,n", [(8, 1000, 3000), (4, 2048, 700), (10, 513, 1025), (8, 1100, 4200), (5, 2304, 4096)])
def test_trsm_identity_large(g, e, m, n):
    # U X = B and L X = B checked with the (separately verified) product kernel
    import torch

    ctx = g.field_new(e)
    R = g.PackedMatrix.random(ctx, m, m, 21).to_array()
    diag = (np.arange(m) % (ctx.order - 1)) + 1
    up, lo = np.triu(R, 1), np.tril(R, -1)
    np.fill_diagonal(up, diag)
    np.fill_diagonal(lo, diag)
    U = g.PackedMatrix.from_array(ctx, up)
    L = g.PackedMatrix.from_array(ctx, lo)
    B0 = g.PackedMatrix.random(ctx, m, n, 23)
    for T in (U, L):
        X = B0.copy()
        (g.trsm_upper_left if T is U else g.trsm_lower_left)(T, X)
        assert g.karatsuba_mul_packed(T, X) == B0
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", range(int(os.environ.get("GF2E_FUZZ_SEEDS", "12"))))
def test_trsm_fuzz(g, seed):
    # random field, shapes, triangle, unit/non-unit diagonal (random nonzero pivots):
    # T X = B checked with the separately verified product kernel
    rng = np.random.default_rng(9000 + seed)
    e = int(rng.integers(2, 11))
    m, n = int(rng.integers(1, 1400)), int(rng.integers(1, 1400))
    ctx = g.field_new(e)
    R = g.PackedMatrix.random(ctx, m, m, 40 + seed).to_array()
    upper, unit = bool(seed & 1), (seed % 4 == 2)
    T = np.triu(R, 1) if upper else np.tril(R, -1)
    np.fill_diagonal(T, 1 if unit else rng.integers(1, ctx.order, size=m))
    Tm = g.PackedMatrix.from_array(ctx, T)
    B0 = g.PackedMatrix.random(ctx, m, n, 41 + seed)
    X = B0.copy()
    if upper:
        g.trsm_upper_left(Tm, X)
    elif unit:
        g.trsm_lower_left_unit(Tm, X)
    else:
        g.trsm_lower_left(Tm, X)
    assert g.karatsuba_mul_packed(Tm, X) == B0, (e, m, n, upper, unit)


def test_trsm_singular(g):
    ctx = g.field_new(5)
    arr = np.triu(g.PackedMatrix.random(ctx, 300, 300, 3).to_array(), 1)
    np.fill_diagonal(arr, 1)
    arr[200, 200] = 0
    arr[250, 250] = 0
    U = g.PackedMatrix.from_array(ctx, arr)
    B = g.PackedMatrix.random(ctx, 300, 10, 4)
    before = B.to_numpy()
    with pytest.raises(g.SingularMatrixError) as ei:
        g.trsm_upper_left(U, B)
    assert ei.value.index == 200 and isinstance(ei.value, ValueError)
    assert np.array_equal(B.to_numpy(), before)  # untouched
    # the unit-diagonal lower solve ignores the stored diagonal
    g.trsm_lower_left_unit(g.PackedMatrix.from_array(ctx, arr.T.copy()), B)
    with pytest.raises(ValueError, match="square"):
        g.trsm_upper_left(g.PackedMatrix.random(ctx, 3, 4, 1), B)


def test_mul_by_x_and_scalar_mul_golden(g, golden):
    for tag in _tags(golden, "scal_tags"):
        e = int(tag.split("/e")[1])
        ctx = g.field_new(e)
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A"], 70)
        xA = g.mul_by_x(g.slice_packed(A))
        assert np.array_equal(xA.to_numpy(), golden[f"{tag}/xA"]), tag
        for c, ref in zip(golden[f"{tag}/c"], golden[f"{tag}/cA"]):
            assert np.array_equal(A.scalar_mul(int(c)).to_numpy(), ref), (tag, int(c))
        with pytest.raises(ValueError):
            A.scalar_mul(ctx.order)


@pytest.mark.parametrize("e", range(2, 11))
def test_matrix_file_roundtrip(g, e, tmp_path):
    # SPEC cli MatrixFile: parse(serialize(A)) == A, canonical text round-trips byte for byte
    ctx = g.field_new(e)
    for (m, n) in [(7, 65), (1, 1), (0, 3), (4, 0), (33, 128)]:
        A = g.PackedMatrix.random(ctx, m, n, 5 + e)
        text = g.serialize_matrix(A)
        assert text.startswith(f"gf2e-mat v1 e={e} f={ctx.f:x} rows={m} cols={n} repr=packed\n")
        B = g.parse_matrix(text)
        assert isinstance(B, g.PackedMatrix) and B == A
        assert g.serialize_matrix(B) == text
        S = g.slice_packed(A)
        p = tmp_path / f"s{e}_{m}_{n}.txt"
        g.save_matrix(p, S)
        T = g.load_matrix(p)
        assert isinstance(T, g.SlicedMatrix) and np.array_equal(T.to_numpy(), S.to_numpy())
    ok = "gf2e-mat v1 e=2 f=7 rows=1 cols=2 repr=packed\n1 3\n"
    assert g.parse_matrix(ok).to_array().tolist() == [[1, 3]]
    for bad in ["gf2e-mat v1 e=2 f=7 rows=1 cols=2 repr=packed\n1 4\n",   # entry >= 2^e
                "gf2e-mat v1 e=2 f=7 rows=2 cols=2 repr=packed\n1 3\n",   # missing row
                "gf2e-mat v1 e=2 f=7 rows=1 cols=2 repr=packed\n1  3\n",  # double space
                "gf2e-mat v1 e=2 f=7 rows=1 cols=2 repr=packed\n1 A\n",   # uppercase
                "gf2e-mat v2 e=2 f=7 rows=1 cols=2 repr=packed\n1 3\n",   # version
                "gf2e-mat v1 e=2 f=5 rows=1 cols=2 repr=packed\n1 3\n",   # reducible f
                "gf2e-mat v1 e=2 f=7 rows=1 cols=2 repr=packed\n1 3"]:    # no trailing newline
        with pytest.raises(ValueError):
            g.parse_matrix(bad)

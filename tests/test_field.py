"""Host field arithmetic (paper_1111_6900_b200.gf2e) against brute-force restatements of the
reference's definitions (gf2e.py:35-106): trial-division irreducibility, the order walk for
primitivity, and shift-and-reduce products.  No GPU needed."""

import numpy as np
import pytest

from paper_1111_6900_b200 import gf2e as G


def _clmul(a, b):
    r = 0
    i = 0
    while b >> i:
        if (b >> i) & 1:
            r ^= a << i
        i += 1
    return r


def _mod(a, m):
    dm = m.bit_length() - 1
    while a.bit_length() - 1 >= dm:
        a ^= m << (a.bit_length() - 1 - dm)
    return a


def _irreducible_bf(f):
    d = f.bit_length() - 1
    if d < 1:
        return False
    if d == 1:
        return True
    return all(_mod(f, g) != 0 for g in range(2, 1 << (d // 2 + 1)))


def _primitive_bf(f):
    e = f.bit_length() - 1
    n = (1 << e) - 1
    acc = 2 % (1 << e) if e > 1 else 1
    for _ in range(1, n):
        if acc == 1:
            return False
        acc = _mod(_clmul(acc, 2), f)
    return acc == 1


def test_irreducible_and_primitive_all_degrees_to_10():
    counts = {}
    for f in range(1, 1 << 11):
        irr = G.is_irreducible(f)
        assert irr == _irreducible_bf(f), f
        if irr:
            counts[f.bit_length() - 1] = counts.get(f.bit_length() - 1, 0) + 1
            assert G.is_primitive(f) == _primitive_bf(f), f
    # number of irreducible binary polynomials of degree 1..10 (necklace counting)
    assert [counts[d] for d in range(1, 11)] == [2, 1, 2, 3, 6, 9, 18, 30, 56, 99]
    assert G.is_irreducible(0) is False


def test_default_polys_are_primitive():
    for e, f in G.DEFAULT_POLYS.items():
        assert f.bit_length() - 1 == e and G.is_irreducible(f) and G.is_primitive(f)


@pytest.mark.parametrize("e,f", [(e, None) for e in range(2, 11)] + [(4, 0x19), (8, 0x11B), (10, 0x40F)])
def test_tables_match_shift_and_reduce(e, f):
    ctx = G.FieldCtx(e, f)
    q = 1 << e
    rng = np.random.default_rng(e)
    pairs = rng.integers(0, q, size=(400, 2))
    for a, b in pairs:
        assert ctx.mul(int(a), int(b)) == _mod(_clmul(int(a), int(b)), ctx.f)
    assert ctx.mul_table.dtype == np.uint16 and ctx.mul_table.shape == (q, q)
    assert np.array_equal(ctx.mul_table, ctx.mul_table.T)
    assert not ctx.mul_table[0].any() and not ctx.mul_table[:, 0].any()
    a = np.arange(1, q)
    assert (ctx.mul_table[a, ctx.inv_table[a]] == 1).all() and ctx.inv_table[0] == 0
    with pytest.raises(ZeroDivisionError):
        ctx.inv(0)


def test_poly_helpers():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        a, b = (int(x) for x in rng.integers(0, 1 << 30, size=2))
        m = int(rng.integers(1, 1 << 12)) | 1
        assert G.poly_mul(a, b) == _clmul(a, b)
        assert G.poly_mod(a, m) == _mod(a, m)
    assert G.poly_degree(0) == -1 and G.poly_degree(1) == 0


def test_field_errors_and_cache():
    with pytest.raises(ValueError, match="extension degree must be in 2..10, got 11"):
        G.field_new(11)
    with pytest.raises(ValueError, match="modulus 0x15 is not irreducible over GF\\(2\\)"):
        G.FieldCtx(4, 0x15)
    with pytest.raises(ValueError, match="modulus 0x13 has degree 4, expected 3"):
        G.FieldCtx(3, 0x13)
    assert G.field_new(8) is G.field_new(8, 0x11D)
    assert G.field_new(8) == G.FieldCtx(8) and hash(G.field_new(8)) == hash((8, 0x11D))

"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/gf2e_b200.h declares, and its host-side logic (schedule, validation, workspace
sizing) matches the oracle and the reference's error behaviour."""

import ctypes
import os
import re

import pytest

import oracle
from paper_1111_6900_b200 import _lib
import paper_1111_6900_b200 as g

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gf2e_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(gf2e_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 17
    for name in syms:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes signature table"
    assert set(_lib.SIGNATURES) == set(syms)


def test_version_and_pack_width():
    assert b"sm_100a" in _lib.load().gf2e_version()
    assert [_lib.load().gf2e_pack_width(e) for e in range(1, 12)] == [-1, 2, 4, 4, 8, 8, 8, 8, 16, 16, -1]


@pytest.mark.parametrize("e", range(2, 11))
def test_native_schedule_matches_oracle(e):
    s = g.schedule(e)
    o = oracle.schedule(e)
    assert list(s.subsets) == o.subsets
    assert list(s.outmap) == o.outmap
    assert s.counters == (o.counters.gf2_matmul_count, o.counters.additions, o.counters.peak_live_products)


@pytest.mark.parametrize("e,f", [(4, 0b11001), (8, 0x11B), (10, 0b10000001111), (5, 0b111101)])
def test_native_schedule_custom_f(e, f):
    s = g.schedule(e, f)
    o = oracle.schedule(e, f)
    assert list(s.outmap) == o.outmap and list(s.subsets) == o.subsets


@pytest.mark.parametrize("e,f", [(e, None) for e in range(2, 11)] + [(4, 0b11001), (8, 0x11B), (10, 0b10000001111)])
def test_run_grouping_reproduces_outmap(e, f):
    # the running-sum form's drain groups: every output plane b must receive exactly the
    # products of outmap[b], i.e. for each product t the XOR of the masks of the groups it is
    # accumulated into is its column of M (oracle schedule, poly_mul.py:245-259)
    o = oracle.schedule(e, f)
    seq, gsize, gmask, load = g._lib.run_schedule(e, o.f)
    K = len(o.subsets)
    assert sum(gsize) == len(seq) and all(0 <= t < K for t in seq)
    col = [0] * K
    i = 0
    buf = [0, 0]
    for gi, (n, m) in enumerate(zip(gsize, gmask)):
        for t in seq[i:i + n]:
            col[t] ^= m
        buf[gi & 1] += n
        i += n
    want = [sum(((o.outmap[b] >> t) & 1) << b for b in range(e)) for t in range(K)]
    assert col == want
    assert load == max(buf) and len(gsize) <= K


def test_schedule_rejects_bad_fields():
    n = ctypes.c_int()
    L = _lib.load()
    assert L.gf2e_schedule(11, 0x805, ctypes.byref(n), None, None, None) == _lib.GF2E_EINVAL
    assert "2..10" in _lib.last_error()
    assert L.gf2e_schedule(4, 0b10101, ctypes.byref(n), None, None, None) == _lib.GF2E_EINVAL  # reducible
    assert "irreducible" in _lib.last_error()
    assert L.gf2e_schedule(4, 0b111, ctypes.byref(n), None, None, None) == _lib.GF2E_EINVAL  # wrong degree
    with pytest.raises(ValueError):
        g.schedule(4, 0b10101)


def test_count_products_host_only():
    # poly_mul.count_products (poly_mul.py:262-272) answered without a GPU
    assert [g.count_products(e) for e in range(2, 11)] == [3, 6, 9, 15, 18, 24, 27, 39, 45]


def test_workspace_sizes():
    L = _lib.load()
    # tensor-core layout: K(e) * (m_pad * k_pad + n_pad * k_pad) / 8 bytes, bounded over the
    # forms the call may pick (n padded to 256-column tiles, or 192 for the running-sum form;
    # k to 256-bit stages)
    def rup(x, q):
        return -(-x // q) * q

    ws = L.gf2e_slice_mul_workspace(8, 0x11D, 16384, 16384, 16384, 0)
    assert ws == 27 * (16384 + 16384) * 16384 // 8  # long k: the 256-column fp4 forms only
    assert L.gf2e_slice_mul_workspace(8, 0x11D, 0, 5, 5, 0) == 0
    assert L.gf2e_slice_mul_workspace(8, 0x11D, 5, 5, 5, 1 << 7) == -1  # bad flag
    assert L.gf2e_slice_mul_workspace(8, 0x11D, 5, 5, 5, _lib.TC_INT8 | _lib.TC_RUN) == -1  # conflicting
    # m padded to the 256-row CTA-pair tile; short k: the running-sum form's B^T is stored
    # nibble-expanded (4 bits per bit)
    assert L.gf2e_plane_mul_workspace(100, 1, 300, 0) == (256 * 256 + max(rup(300, 256), rup(300, 192)) * 256 * 4) // 8


def test_invalid_arguments_fail_before_device():
    L = _lib.load()
    rc = L.gf2e_slice_mul(12, 0x1, None, 1, 1, None, 1, 1, None, 1, 1, 4, 4, 4, 0, None, 0, None)
    assert rc == _lib.GF2E_EINVAL
    rc = L.gf2e_slice_mul(4, 0x13, None, 1, 1, None, 1, 1, None, 1, 1, 4, 4, 4, 0, None, 0, None)
    assert rc == _lib.GF2E_EINVAL and "NULL" in _lib.last_error()


def test_field_api_mirrors_reference():
    with pytest.raises(ValueError, match="2..10"):
        g.field_new(1)
    with pytest.raises(ValueError, match="irreducible"):
        g.FieldCtx(4, 0b10101)
    ctx = g.field_new(2)
    assert ctx.mul(2, 2) == 3 and ctx.inv(2) == 3
    with pytest.raises(ZeroDivisionError):
        ctx.inv(0)
    assert g.pack_width(5) == 8
    with pytest.raises(ValueError):
        g.pack_width(11)


def test_field_tables_match_reference(golden):
    import numpy as np

    for e in (2, 3, 4):
        assert np.array_equal(g.field_new(e).mul_table, golden[f"field/e{e}/mul"])


def test_host_buffer_api_rejects_bad_shapes():
    # karatsuba_mul_packed_host validates every host array before the library touches it
    # (a short C would otherwise be read / written past its end by the H2D / D2H copies)
    import numpy as np

    ctx = g.field_new(8)
    m, k, n = 10, 70, 90
    A = np.zeros((m, g.words_for(k * 8)), dtype=np.uint64)
    B = np.zeros((k, g.words_for(n * 8)), dtype=np.uint64)
    C = np.zeros((m, g.words_for(n * 8)), dtype=np.uint64)
    with pytest.raises(ValueError, match="shape"):
        g.karatsuba_mul_packed_host(ctx, A, k, B, n, C_words=C[:m - 1].copy())
    with pytest.raises(ValueError, match="shape"):
        g.karatsuba_mul_packed_host(ctx, A, k, B, n, out=np.zeros((m, 3), dtype=np.uint64))
    with pytest.raises(ValueError, match="shape"):
        g.karatsuba_mul_packed_host(ctx, A, k, B, n, C_words=C.reshape(-1))
    with pytest.raises(ValueError, match="C-contiguous uint64"):
        g.karatsuba_mul_packed_host(ctx, A, k, B, n, C_words=C.astype(np.int64))
    with pytest.raises(ValueError, match="words per row"):
        g.karatsuba_mul_packed_host(ctx, A[:, :1], k, B, n)
    with pytest.raises(ValueError, match="words per row"):
        g.karatsuba_mul_packed_host(ctx, A, k, B[:, :2], n)
    with pytest.raises(ValueError, match="inner dimensions differ"):
        g.karatsuba_mul_packed_host(ctx, A, k + 1, B, n)

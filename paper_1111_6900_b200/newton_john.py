"""Newton-John (Gray-code multiple table) API on the B200 — drop-in for ``gf2elin.newton_john``
(SURVEY §8f rank 2).

The reference uses these table-based routines below its 64 crossover (``tuning.py:24``) and as
the quadratic base cases of PLE and TRSM.  Here the functions keep their names, arguments,
results and exceptions and run on the device:

* ``make_table`` (``newton_john.py:55-88``): all 2^e scalar multiples of a row in one
  ``gf2e_row_scales`` launch (broadcast row x scalars 0 .. 2^e - 1);
* ``nj_mul`` / ``cubic_mul`` (``:124-164``): the reference's own algorithm — a table of the 2^e
  multiples of every row of B, one lookup-and-XOR per (row of A, row of B) — on packed words
  in one launch (``gf2e_nj_mul``, ``csrc/nj.cu``) when B's rows fit its shared-memory tables
  (n <= 64 at e = 9, 10; more at smaller e), else the tensor-core product (the product is
  unique, so the results are bit-identical);
* ``nj_gauss`` (``:167-204``): ``echelonize`` (the reference documents that its PLE-based
  echelon forms match the table-based elimination bit for bit, ``ple_echelon.py:349-352``);
* ``nj_ple`` (``:207-260``): the device PLE, whose 64-column panel kernel is this algorithm
  (same pivot rule, same in-place layout);
* ``nj_trsm_upper_left`` (``:263-291``): the device TRSM.

``RowOpCounters``: ``make_table`` and ``nj_mul`` count the tables their kernels build (e scalar
row multiplications and 2^e - 1 row additions per table, as the reference).  ``nj_gauss``,
``nj_ple`` and ``nj_trsm_upper_left`` report the reference-equivalent accounting of the
table algorithm for the same input (one table per pivot / solved row), not the device's
different blocked work.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device, _lib
from .mat_gf2 import RowOpCounters
from .mat_packed import PackedMatrix
from .mat_sliced import cling, slice_packed
from .ple_echelon import SingularMatrixError, echelonize, ple_sliced, trsm_upper_left
from .poly_mul import karatsuba_mul_packed, nj_fits, nj_mul_packed


def _count_tables(ctx, counters: RowOpCounters | None, ntables: int) -> None:
    if counters is not None and ntables > 0:
        counters.scalar_row_muls += ctx.e * ntables
        counters.row_adds += ((1 << ctx.e) - 1) * ntables


class NJTable:
    """All 2^e scalar multiples of one source row, indexed by scalar (newton_john.py:34-52).
    ``words`` is a device tensor [2^e, row words]."""

    __slots__ = ("ctx", "ncols", "words")

    def __init__(self, ctx, ncols: int, words):
        self.ctx = ctx
        self.ncols = ncols
        self.words = words

    def row(self, x: int) -> PackedMatrix:
        out = PackedMatrix(self.ctx, 1, self.ncols)
        out.storage.words[0].copy_(self.words[x])
        return out

    def as_matrix(self) -> PackedMatrix:
        out = PackedMatrix(self.ctx, self.words.shape[0], self.ncols)
        out.storage.words.copy_(self.words)
        return out


def make_table(row: PackedMatrix, counters: RowOpCounters | None = None) -> NJTable:
    """Table of all 2^e multiples of a 1 x n row (newton_john.py:77-88); row x = x * row."""
    if row.nrows != 1:
        raise ValueError(f"expected a single row, got {row.nrows} rows")
    ctx = row.ctx
    q = 1 << ctx.e
    src = row.storage.words
    width = src.shape[1]
    words = _device.zeros_words((q, width))
    if width:
        cs = np.arange(q, dtype=np.uint32)
        _lib.call("gf2e_row_scales", ctx.e, ctx.f, _device.ptr(src), width, 1,
                  cs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), _device.ptr(words), width, q, row.ncols,
                  _device.stream_handle())
    _count_tables(ctx, counters, 1)
    return NJTable(ctx, row.ncols, words)


def _check_mul_operands(A: PackedMatrix, B: PackedMatrix) -> None:
    if A.ctx != B.ctx:
        raise ValueError(f"field mismatch: {A.ctx} vs {B.ctx}")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")


def _device_mul(A: PackedMatrix, B: PackedMatrix) -> PackedMatrix:
    # the packed-domain Newton-John kernel (gf2e_nj_mul: the reference's table algorithm, one
    # launch) whenever B's rows fit it; the tensor-core product otherwise (same result)
    if nj_fits(A.ctx.e, B.ncols):
        return nj_mul_packed(A, B)
    return karatsuba_mul_packed(A, B, backend="tc")


def cubic_mul(A: PackedMatrix, B: PackedMatrix) -> PackedMatrix:
    """Schoolbook product (newton_john.py:124-142): the unique product, computed on device."""
    _check_mul_operands(A, B)
    return _device_mul(A, B)


def nj_mul(A: PackedMatrix, B: PackedMatrix, counters: RowOpCounters | None = None,
           table_count: int | None = None) -> PackedMatrix:
    """Table-based product (newton_john.py:145-164): the same tables-per-row-of-B algorithm in
    one device launch (gf2e_nj_mul) when B's rows fit it, else the device product.  counters:
    the reference's accounting (one table per row of B: e scalar row multiplications and
    2^e - 1 row additions each); the kernel builds exactly those tables."""
    _check_mul_operands(A, B)
    if A.nrows == 0 or A.ncols == 0 or B.ncols == 0:
        return PackedMatrix(A.ctx, A.nrows, B.ncols)
    _count_tables(A.ctx, counters, B.nrows)
    return _device_mul(A, B)


def nj_gauss(A: PackedMatrix, full: bool = True, counters: RowOpCounters | None = None) -> int:
    """In-place Gaussian elimination, returns the rank (newton_john.py:167-204): reduced row
    echelon form (full) or row echelon form with leading ones."""
    if A.nrows == 0 or A.ncols == 0:
        return 0
    r = echelonize(A, full=full)
    _count_tables(A.ctx, counters, r)
    return r


def nj_ple(A: PackedMatrix, counters: RowOpCounters | None = None):
    """In-place PLE (newton_john.py:207-260); returns (P, Q, r): int64 swap vectors of length
    min(m, n) and the rank."""
    S = slice_packed(A)
    P, Q, r = ple_sliced(S)
    cling(S, out=A)
    _count_tables(A.ctx, counters, r)
    return P.entries, Q.entries, r


def nj_trsm_upper_left(U: PackedMatrix, B: PackedMatrix, counters: RowOpCounters | None = None) -> None:
    """Solve U X = B in place (newton_john.py:263-291)."""
    trsm_upper_left(U, B)
    _count_tables(U.ctx, counters, U.nrows - 1)


__all__ = ["SingularMatrixError", "NJTable", "make_table", "cubic_mul", "nj_mul", "nj_gauss", "nj_ple",
           "nj_trsm_upper_left"]

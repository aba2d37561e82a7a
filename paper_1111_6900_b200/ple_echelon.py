"""Triangular solves over GF(2^e) on the B200 — the first consumer of the hot path.

Drop-in for ``trsm_upper_left``, ``trsm_lower_left``, ``trsm_lower_left_unit`` and
``SingularMatrixError`` of ``gf2elin.ple_echelon`` / ``newton_john``
(``ple_echelon.py:138-217``, ``newton_john.py:26-31``): solve T X = B in place on packed
matrices.  One ``gf2e_trsm`` call: the matrices are sliced once, the blocked recursion
(128-row aligned splits) does every off-diagonal update ``B_i ^= T_ij X_j`` with the fused
tensor-core ``addmul`` and applies device-inverted diagonal blocks with the same kernel, then
the result is clung back into B.  X is unique, so the result is bit-identical to the
reference for any crossover (accepted and ignored).  Singular factors raise before B is
modified; the index reported is the smallest zero diagonal row.
"""

from __future__ import annotations

import ctypes

from . import _device, _lib
from .mat_gf2 import words_for
from .mat_packed import PackedMatrix
from .mat_sliced import SlicedMatrix, cling, slice_packed
from .poly_mul import MulCounters


class SingularMatrixError(ValueError):
    """A triangular solve met a zero diagonal entry (newton_john.py:26-31)."""

    def __init__(self, index: int):
        super().__init__(f"zero diagonal entry at index {index}")
        self.index = index


def _check(T: PackedMatrix, B: PackedMatrix) -> None:
    if T.ctx != B.ctx:
        raise ValueError(f"field mismatch: {T.ctx} vs {B.ctx}")
    m = T.nrows
    if T.ncols != m:
        raise ValueError(f"triangular factor must be square, got {T.nrows}x{T.ncols}")
    if B.nrows != m:
        raise ValueError(f"dimension mismatch: {m}x{m} solve against {B.nrows} rows")


def trsm_sliced(T: SlicedMatrix, B: SlicedMatrix, upper: bool, unit_diag: bool = False) -> None:
    """Solve T X = B in place on sliced matrices (X overwrites B)."""
    ctx = T.ctx
    m, n = T.nrows, B.ncols
    if m == 0 or n == 0:
        return
    L = _lib.load()
    ws_bytes = int(L.gf2e_trsm_workspace(ctx.e, ctx.f, m, n))
    ws = _device.workspace.get(ws_bytes)
    bad = ctypes.c_int64(-1)
    ldt, ldb = T.planes.shape[2], B.planes.shape[2]
    rc = L.gf2e_trsm(ctx.e, ctx.f, int(upper), int(unit_diag), _device.ptr(T.planes), ldt, m * ldt,
                     _device.ptr(B.planes), ldb, m * ldb, m, n, ws.data_ptr(), ws.numel(), _device.stream_handle(),
                     ctypes.byref(bad))
    if rc == _lib.GF2E_ESINGULAR:
        raise SingularMatrixError(int(bad.value))
    _lib.check(rc, "gf2e_trsm")


def _trsm_packed(T: PackedMatrix, B: PackedMatrix, upper: bool, unit_diag: bool) -> None:
    _check(T, B)
    if T.nrows == 0 or B.ncols == 0:
        return
    Bs = slice_packed(B)
    trsm_sliced(slice_packed(T), Bs, upper, unit_diag)
    cling(Bs, out=B)


def trsm_upper_left(U: PackedMatrix, B: PackedMatrix, crossover: int | None = None,
                    counters: MulCounters | None = None) -> None:
    """Solve U X = B in place for upper triangular U (ple_echelon.py:187-198)."""
    _trsm_packed(U, B, True, False)


def trsm_lower_left(L: PackedMatrix, B: PackedMatrix, unit_diag: bool = False, crossover: int | None = None,
                    counters: MulCounters | None = None) -> None:
    """Solve L X = B in place for lower triangular L (ple_echelon.py:138-156)."""
    _trsm_packed(L, B, False, unit_diag)


def trsm_lower_left_unit(L: PackedMatrix, B: PackedMatrix, crossover: int | None = None,
                         counters: MulCounters | None = None) -> None:
    """Solve L X = B with L unit lower triangular (diagonal implicit; ple_echelon.py:178-184)."""
    _trsm_packed(L, B, False, True)


__all__ = ["SingularMatrixError", "trsm_sliced", "trsm_upper_left", "trsm_lower_left", "trsm_lower_left_unit",
           "words_for"]

"""Triangular solves, PLE decomposition and echelon forms over GF(2^e) on the B200 — the
consumers of the hot path.

Drop-in for ``trsm_upper_left``, ``trsm_lower_left``, ``trsm_lower_left_unit`` and
``SingularMatrixError`` of ``gf2elin.ple_echelon`` / ``newton_john``
(``ple_echelon.py:138-217``, ``newton_john.py:26-31``): solve T X = B in place on packed
matrices.  One ``gf2e_trsm`` call: the matrices are sliced once, the blocked recursion
(128-row aligned splits) does every off-diagonal update ``B_i ^= T_ij X_j`` with the fused
tensor-core ``addmul`` and applies device-inverted diagonal blocks with the same kernel, then
the result is clung back into B.  X is unique, so the result is bit-identical to the
reference for any crossover (accepted and ignored).  Singular factors raise before B is
modified; the index reported is the smallest zero diagonal row.

``ple`` / ``echelonize`` (``ple_echelon.py:240-374``) run ``gf2e_ple`` / ``gf2e_echelonize``:
the reference's column-halving recursion with 64-column-aligned splits (its result is
crossover-independent, ``ple_echelon.py:8-10``), 64-column base panels factored on device by
the two-phase ``nj_ple`` kernel, Schur updates through the fused addmul and corner solves
through the device TRSM.  Same pivot rule, same in-place storage (L below the diagonal with
the pivots on it, E above), same LAPACK-style swap vectors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

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


# -- reference MulCounters accounting (ple_echelon.py:130-136, 159-217, 240-287) -------------
# The device recursion splits at tile-aligned points and multiplies every block on the tensor
# cores, so it cannot count what the reference counts.  The reference's counters are a pure
# function of the shapes, the crossover and (for PLE) the column rank profile: _dispatch_mul
# runs karatsuba_mul (K(e) products + the schedule's additions) iff min(m, k, n) > crossover.
# These replays reproduce them; device_products receives the products actually launched.
DEFAULT_PLE_CROSSOVER = 64  # tuning.py:24


def _crossover(crossover: int | None) -> int:
    return max(1, DEFAULT_PLE_CROSSOVER if crossover is None else int(crossover))


def _ref_trsm_calls(m: int, n: int, cx: int) -> int:
    """Karatsuba calls of _trsm_lower_rec / _trsm_upper_rec (ple_echelon.py:159-175,201-217)
    on an m x m triangle against n columns; both split at h = m // 2 and dispatch one
    (m-h) x h x n (lower) or h x (m-h) x n (upper) update."""
    if m <= cx:
        return 0
    h = m // 2
    return (_ref_trsm_calls(h, n, cx) + _ref_trsm_calls(m - h, n, cx)
            + (1 if min(m - h, h, n) > cx else 0))


def _ref_ple_calls(m: int, n: int, c0: int, pivots: np.ndarray, cx: int) -> int:
    """Karatsuba calls of _ple_rec (ple_echelon.py:240-287) on rows m, columns [c0, c0 + n):
    the left half's rank r1 is the number of pivot columns it holds (PLE finds the column rank
    profile, and a node's Schur complement keeps the global profile's columns)."""
    if n <= cx or n < 2:
        return 0
    n1 = n // 2
    calls = _ref_ple_calls(m, n1, c0, pivots, cx)
    r1 = int(np.count_nonzero((pivots >= c0) & (pivots < c0 + n1)))
    if r1 > 0:
        calls += _ref_trsm_calls(r1, n - n1, cx)
        if m - r1 > 0 and min(m - r1, r1, n - n1) > cx:
            calls += 1
    if m - r1 > 0:
        calls += _ref_ple_calls(m - r1, n - n1, c0 + n1, pivots, cx)
    return calls


def _account(counters: MulCounters | None, ctx, calls: int, device: int) -> None:
    from .poly_mul import _bump

    _bump(counters, ctx, calls, device_products=device)


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


def _trsm_packed(T: PackedMatrix, B: PackedMatrix, upper: bool, unit_diag: bool, crossover: int | None,
                 counters: MulCounters | None) -> None:
    _check(T, B)
    if T.nrows == 0 or B.ncols == 0:
        return
    Bs = slice_packed(B)
    Ts = slice_packed(T)
    trsm_sliced(Ts, Bs, upper, unit_diag)
    device = _lib.last_gf2_products()  # before cling (every library call resets it)
    cling(Bs, out=B)
    _account(counters, T.ctx, _ref_trsm_calls(T.nrows, B.ncols, _crossover(crossover)), device)


def trsm_upper_left(U: PackedMatrix, B: PackedMatrix, crossover: int | None = None,
                    counters: MulCounters | None = None) -> None:
    """Solve U X = B in place for upper triangular U (ple_echelon.py:187-198)."""
    _trsm_packed(U, B, True, False, crossover, counters)


def trsm_lower_left(L: PackedMatrix, B: PackedMatrix, unit_diag: bool = False, crossover: int | None = None,
                    counters: MulCounters | None = None) -> None:
    """Solve L X = B in place for lower triangular L (ple_echelon.py:138-156)."""
    _trsm_packed(L, B, False, unit_diag, crossover, counters)


def trsm_lower_left_unit(L: PackedMatrix, B: PackedMatrix, crossover: int | None = None,
                         counters: MulCounters | None = None) -> None:
    """Solve L X = B with L unit lower triangular (diagonal implicit; ple_echelon.py:178-184)."""
    _trsm_packed(L, B, False, True, crossover, counters)


# -- permutations (ple_echelon.py:36-107) ----------------------------------------------------


class PermVector:
    """LAPACK-style swap vector; entry i >= i for all i (ple_echelon.py:36-65)."""

    __slots__ = ("entries",)

    def __init__(self, entries):
        arr = np.asarray(entries, dtype=np.int64).copy()
        if arr.ndim != 1:
            raise ValueError("permutation vector must be one-dimensional")
        if np.any(arr < np.arange(arr.size)):
            bad = int(np.nonzero(arr < np.arange(arr.size))[0][0])
            raise ValueError(f"entry {int(arr[bad])} at index {bad} violates P_i >= i")
        self.entries = arr

    def __len__(self) -> int:
        return self.entries.size

    def __getitem__(self, i: int) -> int:
        return int(self.entries[i])

    def __eq__(self, other) -> bool:
        return isinstance(other, PermVector) and np.array_equal(self.entries, other.entries)

    def __repr__(self) -> str:
        return f"PermVector({self.entries.tolist()})"

    @classmethod
    def identity(cls, n: int) -> "PermVector":
        return cls(np.arange(n, dtype=np.int64))


@dataclass
class PleFactors:
    """In-place PLE result: swap vectors, rank, and the matrix (ple_echelon.py:68-74)."""

    P: PermVector
    Q: PermVector
    rank: int
    matrix: PackedMatrix


def _entries(P) -> np.ndarray:
    return np.ascontiguousarray(P.entries if isinstance(P, PermVector) else np.asarray(P, dtype=np.int64),
                                dtype=np.int64)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def apply_perm_rows(A, P, forward: bool = True) -> None:
    """Apply (forward) or undo (backward) a row swap vector in place (ple_echelon.py:81-91).
    A: PackedMatrix or SlicedMatrix; the swaps run on device."""
    ent = _entries(P)
    m = A.nrows
    for i, j in enumerate(ent.tolist()):
        if j < i or j >= m:
            raise ValueError(f"swap target {j} at index {i} invalid for {m} rows")
    if ent.size == 0:
        return
    if isinstance(A, SlicedMatrix):
        t, planes = A.planes, A.ctx.e
        ld, ps, nw = t.shape[2], t.shape[1] * t.shape[2], t.shape[2]
    else:
        t, planes = A.storage.words, 1
        ld, ps, nw = t.shape[1], 0, t.shape[1]
    _lib.call("gf2e_row_swaps", planes, _device.ptr(t), ld, ps, m, nw, _i64p(ent), ent.size, int(not forward),
              _device.stream_handle())


def _col_swaps(A, triples: list[tuple[int, int, int]]) -> None:
    if not triples:
        return
    tr = np.ascontiguousarray(np.asarray(triples, dtype=np.int64).reshape(-1))
    if isinstance(A, SlicedMatrix):
        t, planes, w = A.planes, A.ctx.e, 1
        ld, ps = t.shape[2], t.shape[1] * t.shape[2]
    else:
        t, planes, w = A.storage.words, 1, A.w
        ld, ps = t.shape[1], 0
    _lib.call("gf2e_col_swaps", planes, w, _device.ptr(t), ld, ps, A.nrows, A.ncols, _i64p(tr), len(triples),
              _device.stream_handle())


def col_swap(A, i: int, j: int, row_start: int = 0) -> None:
    """Swap columns i and j in rows >= row_start (PackedMatrix.col_swap), on device."""
    for c in (i, j):
        if not 0 <= c < A.ncols:
            raise IndexError(f"column {c} outside {A.nrows}x{A.ncols}")
    _col_swaps(A, [(i, j, row_start)])


def apply_perm_cols(A, Q, forward: bool = True) -> None:
    """Apply (forward) or undo (backward) a column swap vector in place (ple_echelon.py:94-107)."""
    ent = _entries(Q)
    n = A.ncols
    for i, j in enumerate(ent.tolist()):
        if j < i or j >= n:
            raise ValueError(f"swap target {j} at index {i} invalid for {n} columns")
    order = range(ent.size) if forward else range(ent.size - 1, -1, -1)
    _col_swaps(A, [(i, int(ent[i]), 0) for i in order if int(ent[i]) != i])


# -- PLE and echelon forms (ple_echelon.py:240-374) ---------------------------------------------


def _planes_args(S: SlicedMatrix):
    t = S.planes
    return _device.ptr(t), t.shape[2], t.shape[1] * t.shape[2]


def ple_sliced(S: SlicedMatrix) -> tuple[PermVector, PermVector, int]:
    """In-place PLE of a sliced matrix; returns (P, Q, rank)."""
    m, n = S.nrows, S.ncols
    k = min(m, n)
    P = np.arange(k, dtype=np.int64)
    Q = np.arange(k, dtype=np.int64)
    r = ctypes.c_int64(0)
    if k:
        ptr, ld, ps = _planes_args(S)
        _lib.call("gf2e_ple", S.ctx.e, S.ctx.f, ptr, ld, ps, m, n, _i64p(P), _i64p(Q), ctypes.byref(r),
                  _device.stream_handle())
    return PermVector(P), PermVector(Q), int(r.value)


def ple(A: PackedMatrix, crossover: int | None = None, counters: MulCounters | None = None) -> PleFactors:
    """In-place PLE decomposition of A (ple_echelon.py:290-300).  crossover is accepted for
    API parity; like the reference's, it cannot change the result."""
    S = slice_packed(A)
    P, Q, r = ple_sliced(S)
    device = _lib.last_gf2_products()
    cling(S, out=A)
    if counters is not None:
        from .poly_mul import _bump

        calls = _ref_ple_calls(A.nrows, A.ncols, 0, Q.entries[:r], _crossover(crossover))
        _bump(counters, A.ctx, calls, device_products=device)
    return PleFactors(P, Q, r, A)


def ple_unpack(factors: PleFactors) -> tuple[PackedMatrix, PackedMatrix]:
    """Expand an in-place PLE into explicit L (m x m) and E (m x n) (ple_echelon.py:303-324)."""
    A = factors.matrix
    P, Q, r = factors.P, factors.Q, factors.rank
    m, n = A.nrows, A.ncols
    work = A.copy()
    _col_swaps(work, [(t, Q[t], t) for t in range(r - 1, -1, -1) if Q[t] != t])
    arr = work.to_array()
    larr = np.zeros((m, m), dtype=np.uint16)
    np.fill_diagonal(larr, 1)
    earr = np.zeros((m, n), dtype=np.uint16)
    for t in range(r):
        j = Q[t]
        larr[t:, t] = arr[t:, j]
        earr[t, j] = 1
        earr[t, j + 1:] = arr[t, j + 1:]
    return PackedMatrix.from_array(A.ctx, larr), PackedMatrix.from_array(A.ctx, earr)


def ple_reconstruct(factors: PleFactors) -> PackedMatrix:
    """P * L * E from an in-place PLE (ple_echelon.py:327-332), product on device."""
    from .poly_mul import karatsuba_mul_packed

    L, E = ple_unpack(factors)
    M = karatsuba_mul_packed(L, E)
    apply_perm_rows(M, factors.P, forward=False)
    return M


def echelonize_sliced(S: SlicedMatrix, full: bool = True) -> int:
    m, n = S.nrows, S.ncols
    if m == 0 or n == 0:
        return 0
    r = ctypes.c_int64(0)
    ptr, ld, ps = _planes_args(S)
    _lib.call("gf2e_echelonize", S.ctx.e, S.ctx.f, ptr, ld, ps, m, n, int(bool(full)), ctypes.byref(r),
              _device.stream_handle())
    return int(r.value)


def echelonize(A: PackedMatrix, full: bool = True, crossover: int | None = None,
               counters: MulCounters | None = None) -> int:
    """Reduce A in place via PLE; returns the rank (ple_echelon.py:343-374).  full=False leaves
    the row echelon form, full=True the reduced row echelon form."""
    S = slice_packed(A)
    if counters is None:
        r = echelonize_sliced(S, full)
        cling(S, out=A)
        return r
    # the accounting needs the column rank profile: PLE + the echelon steps on the same planes
    from .poly_mul import _bump

    cx = _crossover(crossover)
    m, n = A.nrows, A.ncols
    r = echelonize_sliced(S, full)
    device = _lib.last_gf2_products()
    cling(S, out=A)
    # pivot columns = the leading entry of each of the first r rows of the echelon form
    lead = A.to_array()[:r] != 0
    pivots = np.argmax(lead, axis=1) if r else np.zeros(0, dtype=np.int64)
    calls = _ref_ple_calls(m, n, 0, pivots, cx)
    if full and r > 0:
        calls += _ref_trsm_calls(r, n, cx)
    _bump(counters, A.ctx, calls, device_products=device)
    return r


__all__ = ["SingularMatrixError", "trsm_sliced", "trsm_upper_left", "trsm_lower_left", "trsm_lower_left_unit",
           "words_for", "PermVector", "PleFactors", "apply_perm_rows", "apply_perm_cols", "col_swap", "ple",
           "ple_sliced", "ple_unpack", "ple_reconstruct", "echelonize", "echelonize_sliced"]

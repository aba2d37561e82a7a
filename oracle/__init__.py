"""CPU oracle for the GF(2^e) bitsliced-Karatsuba hot path — TEST INFRASTRUCTURE ONLY.

This package is the parity checker (and the "port" CPU baseline) for the CUDA library in
``paper_1111_6900_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it; the product path never does.

Two halves:

* ``liboracle.so`` (``oracle/gf2e_oracle.c``) — a C restatement of the reference functions
  (generator, slice, cling, M4RM GF(2) product, recursive Karatsuba, reduce mod f, the PLE
  base case nj_ple), wrapped
  here with numpy.  Each C function cites the reference file:line it follows.
* ``schedule`` — a symbolic replay of the reference Karatsuba recursion
  (``poly_mul.py:166-242``) that yields the operand subsets S_t, the combine map Γ, the
  fold R_f and the counters, used to check the library's native schedule.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against fixtures in
``tests/golden/`` that ``tests/golden/make_golden.py`` produced by importing the reference
package itself (``/root/reference/pkg/src/gf2elin``), plus the SPEC known-answer vectors.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

U64P = ctypes.POINTER(ctypes.c_uint64)
I64 = ctypes.c_int64


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_word_stream.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, U64P]
        L.orc_pack_width.argtypes = [ctypes.c_int]
        L.orc_packed_random.argtypes = [ctypes.c_int, I64, I64, ctypes.c_uint64, I64, I64, I64, U64P, I64]
        L.orc_sliced_random.argtypes = [ctypes.c_int, I64, I64, ctypes.c_uint64, I64, I64, I64, U64P, I64, I64]
        L.orc_slice.argtypes = [ctypes.c_int, I64, I64, U64P, I64, U64P, I64, I64]
        L.orc_cling.argtypes = [ctypes.c_int, I64, I64, U64P, I64, I64, U64P, I64]
        L.orc_gf2_mul.argtypes = [U64P, I64, U64P, I64, U64P, I64, I64, I64, I64, ctypes.c_int, ctypes.c_int]
        L.orc_karatsuba.argtypes = [ctypes.c_int, ctypes.c_uint32, U64P, I64, I64, U64P, I64, I64,
                                    U64P, I64, I64, I64, I64, I64, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int64)]
        L.orc_karatsuba.restype = ctypes.c_int
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_ple.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint16), I64, I64,
                              ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.orc_ple.restype = I64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(U64P)


def words_for(ncols: int) -> int:
    """mat_gf2.py:44"""
    return (ncols + 63) >> 6


def pack_width(e: int) -> int:
    """mat_packed.py:26-33"""
    w = lib().orc_pack_width(e)
    if w < 0:
        raise ValueError(f"extension degree must be in 2..10, got {e}")
    return w


DEFAULT_POLYS = {2: 0b111, 3: 0b1011, 4: 0b10011, 5: 0b100101, 6: 0b1000011,
                 7: 0b10000011, 8: 0b100011101, 9: 0b1000010001, 10: 0b10000001001}
"""gf2e.py:22-32 (restated)."""


def max_threads() -> int:
    return int(lib().orc_max_threads())


# -- generator (rng.py:20-35, mat_packed.py:253-259) ------------------------------------

def word_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    if count:
        lib().orc_word_stream(seed & (2**64 - 1), start, count, _p(out))
    return out


def packed_random(e: int, rows: int, cols: int, seed: int, row0: int = 0, col0: int = 0,
                  gcols: int | None = None) -> np.ndarray:
    """Packed words of the window [row0, row0+rows) x [col0, col0+cols) of the reference
    ``PackedMatrix.random(ctx, *, gcols, seed)`` (gcols = full column count)."""
    w = pack_width(e)
    ld = words_for(cols * w)
    out = np.zeros((rows, ld), dtype=np.uint64)
    if rows and cols:
        lib().orc_packed_random(e, rows, cols, seed, row0, col0, cols if gcols is None else gcols,
                                _p(out), ld)
    return out


def sliced_random(e: int, rows: int, cols: int, seed: int, row0: int = 0, col0: int = 0,
                  gcols: int | None = None) -> np.ndarray:
    """Planes [e, rows, words_for(cols)] of ``slice_packed(PackedMatrix.random(...))``."""
    ld = words_for(cols)
    out = np.zeros((e, rows, ld), dtype=np.uint64)
    if rows and cols:
        lib().orc_sliced_random(e, rows, cols, seed, row0, col0, cols if gcols is None else gcols,
                                _p(out), ld, rows * ld)
    return out


# -- representation conversions (mat_sliced.py:97-106) ----------------------------------

def slice_words(e: int, rows: int, cols: int, packed: np.ndarray) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint64)
    ld = words_for(cols)
    out = np.zeros((e, rows, ld), dtype=np.uint64)
    if rows and cols:
        lib().orc_slice(e, rows, cols, _p(packed), packed.shape[1], _p(out), ld, rows * ld)
    return out


def cling_words(e: int, rows: int, cols: int, planes: np.ndarray) -> np.ndarray:
    planes = np.ascontiguousarray(planes, dtype=np.uint64)
    w = pack_width(e)
    ldp = words_for(cols * w)
    out = np.zeros((rows, ldp), dtype=np.uint64)
    if rows and cols:
        lib().orc_cling(e, rows, cols, _p(planes), planes.shape[2], rows * planes.shape[2],
                        _p(out), ldp)
    return out


# -- GF(2) product (mat_gf2.py:348-366) and Karatsuba (poly_mul.py:166-259) -------------

def gf2_mul(A: np.ndarray, B: np.ndarray, m: int, k: int, n: int, C: np.ndarray | None = None,
            nthreads: int = 0) -> np.ndarray:
    """C = A*B over GF(2) (or C ^= A*B when C is given).  A: (m, words_for(k)), B: (k, words_for(n))."""
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    acc = C is not None
    if C is None:
        C = np.zeros((m, words_for(n)), dtype=np.uint64)
    lib().orc_gf2_mul(_p(A), A.shape[1] if A.ndim == 2 else 0, _p(B), B.shape[1] if B.ndim == 2 else 0,
                      _p(C), C.shape[1], m, k, n, int(acc), nthreads)
    return C


@dataclass
class Counters:
    """poly_mul.py:32-43"""
    gf2_matmul_count: int = 0
    additions: int = 0
    peak_live_products: int = 0


def karatsuba(e: int, f: int, A: np.ndarray, B: np.ndarray, m: int, k: int, n: int,
              C0: np.ndarray | None = None, nthreads: int = 0) -> tuple[np.ndarray, Counters]:
    """karatsuba_mul on plane stacks A [e, m, words(k)], B [e, k, words(n)]; with C0 the
    addmul C0 ^ A*B.  Returns (planes [e, m, words(n)], counters)."""
    A = np.ascontiguousarray(A, dtype=np.uint64)
    B = np.ascontiguousarray(B, dtype=np.uint64)
    nw = words_for(n)
    C = np.zeros((e, m, nw), dtype=np.uint64) if C0 is None else np.array(C0, dtype=np.uint64, copy=True)
    cnt = (ctypes.c_int64 * 3)()
    lda = A.shape[2] if A.size else words_for(k)
    ldb = B.shape[2] if B.size else nw
    Ap = A if A.size else np.zeros(1, dtype=np.uint64)
    Bp = B if B.size else np.zeros(1, dtype=np.uint64)
    Cp = C if C.size else np.zeros(1, dtype=np.uint64)
    rc = lib().orc_karatsuba(e, f, _p(Ap), lda, m * lda, _p(Bp), ldb, k * ldb, _p(Cp), nw, m * nw,
                             m, k, n, int(C0 is not None), nthreads, cnt)
    if rc != 0:
        raise ValueError(f"extension degree must be in 2..10, got {e}")
    return C, Counters(int(cnt[0]), int(cnt[1]), int(cnt[2]))


# -- symbolic schedule replay (poly_mul.py:128-242) -------------------------------------

@dataclass
class Schedule:
    e: int
    f: int
    subsets: list[int]        # S_t as a bitmask over the e input planes, reference order
    gamma: list[int]          # unreduced output d (0..2e-2) as a bitmask over products
    fold: list[int]           # reduced plane j as a bitmask over unreduced outputs d
    outmap: list[int]         # M = R_f . Gamma: reduced plane j as a bitmask over products
    counters: Counters

    @property
    def n_products(self) -> int:
        return len(self.subsets)


def schedule(e: int, f: int | None = None) -> Schedule:
    """Replay ``_kara`` + ``reduce_mod_f`` on symbols: every operand plane is the XOR of a
    subset of input planes (bitmask), every product output is the XOR of a set of products
    (bitmask).  Counter bookkeeping follows poly_mul.py line by line."""
    if f is None:
        f = DEFAULT_POLYS[e]
    subsets: list[int] = []
    cnt = Counters()
    live = [0, 0]  # live, peak (poly_mul.py:128-143)

    def grab(k=1):
        live[0] += k
        live[1] = max(live[1], live[0])

    def base(a, b):  # poly_mul.py:146-150
        assert a == b
        subsets.append(a)
        cnt.gf2_matmul_count += 1
        grab()
        return 1 << (len(subsets) - 1)

    def add_lists(xs, ys):  # poly_mul.py:153-163
        if len(xs) < len(ys):
            xs, ys = ys, xs
        out = list(xs)
        for i, y in enumerate(ys):
            out[i] ^= y
        cnt.additions += len(ys)
        return out

    def kara(a, b):  # poly_mul.py:166-220
        ka = len(a)
        if ka == 1:
            return [base(a[0], b[0])]
        if ka == 3:
            d0 = base(a[0], b[0]); d1 = base(a[1], b[1]); d2 = base(a[2], b[2])
            d01 = base(a[0] ^ a[1], b[0] ^ b[1])
            d02 = base(a[0] ^ a[2], b[0] ^ b[2])
            d12 = base(a[1] ^ a[2], b[1] ^ b[2])
            cnt.additions += 6 + 7
            live[0] -= 6
            grab(5)
            return [d0, d01 ^ d0 ^ d1, d02 ^ d0 ^ d1 ^ d2, d12 ^ d1 ^ d2, d2]
        h = (ka + 1) // 2
        lo = kara(a[:h], b[:h])
        hi = kara(a[h:], b[h:])
        mid = kara(add_lists(a[:h], a[h:]), add_lists(b[:h], b[h:]))
        for i, x in enumerate(lo):
            mid[i] ^= x
        for i, x in enumerate(hi):
            mid[i] ^= x
        cnt.additions += len(lo) + len(hi)
        out = [0] * (2 * ka - 1)
        for i, x in enumerate(lo):
            out[i] ^= x
        for i, x in enumerate(mid):
            out[h + i] ^= x
        for i, x in enumerate(hi):
            out[2 * h + i] ^= x
        cnt.additions += len(lo) + len(mid) + len(hi)
        live[0] -= len(lo) + len(hi) + len(mid)
        grab(len(out))
        return out

    planes = [1 << i for i in range(e)]
    gamma = kara(planes, planes)
    cnt.peak_live_products = live[1]
    # reduce_mod_f (poly_mul.py:223-242) on symbols: work[d] = set of unreduced outputs
    work = [1 << d for d in range(2 * e - 1)]
    low_bits = [k for k in range(e) if (f >> k) & 1]
    for d in range(2 * e - 2, e - 1, -1):
        for k in low_bits:
            work[d - e + k] ^= work[d]
            cnt.additions += 1
    fold = work[:e]
    outmap = []
    for j in range(e):
        acc = 0
        for d in range(2 * e - 1):
            if (fold[j] >> d) & 1:
                acc ^= gamma[d]
        outmap.append(acc)
    return Schedule(e, f, subsets, gamma, fold, outmap, cnt)


def apply_schedule(sch: Schedule, A: np.ndarray, B: np.ndarray, m: int, k: int, n: int) -> np.ndarray:
    """Evaluate C = sum_j x^j * XOR_{t in M[j]} (XOR_{i in S_t} A_i)(XOR_{i in S_t} B_i) with
    the oracle's GF(2) product — an independent route to karatsuba_mul's result."""
    e = sch.e
    nw = words_for(n)
    C = np.zeros((e, m, nw), dtype=np.uint64)
    for t, s in enumerate(sch.subsets):
        Ac = np.zeros((m, words_for(k)), dtype=np.uint64)
        Bc = np.zeros((k, nw), dtype=np.uint64)
        for i in range(e):
            if (s >> i) & 1:
                Ac ^= A[i]
                Bc ^= B[i]
        P = gf2_mul(Ac, Bc, m, k, n)
        for j in range(e):
            if (sch.outmap[j] >> t) & 1:
                C[j] ^= P
    return C


def ple(e: int, f: int, arr: np.ndarray):
    """nj_ple (newton_john.py:207-260) on an element array; returns (factored array, P, Q, rank).
    Equals the reference's recursive ple() for every crossover (ple_echelon.py:8-10)."""
    a = np.ascontiguousarray(arr, dtype=np.uint16).copy()
    m, n = a.shape
    k = min(m, n)
    P = np.zeros(k, dtype=np.int64)
    Q = np.zeros(k, dtype=np.int64)
    r = lib().orc_ple(e, f, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), m, n,
                      P.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), Q.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return a, P, Q, int(r)

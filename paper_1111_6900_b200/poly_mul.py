"""★ The hot path: GF(2^e) matrix multiply(-accumulate) via bitsliced Karatsuba on the B200.

Drop-in for the Karatsuba half of ``gf2elin.poly_mul`` (``poly_mul.py:32-43,128-278``):
``MulCounters``, ``karatsuba_mul``, ``reduce_mod_f``, ``count_products``,
``karatsuba_mul_packed`` keep their names, arguments, return types and errors; ``addmul``
/ ``addmul_packed`` add the C += A*B form the reference writes inline
(``ple_echelon.py:130-136,259``).  M4RIE names are aliases (``mzd_slice_mul`` ...).

One call = one ``gf2e_slice_mul`` into libgf2e_b200.so: operand combinations (K3), then the
fused tensor-core product + Karatsuba combine + mod-f fold (+ addmul XOR) kernel (K4/K5).
Counters are replayed from the native schedule (``gf2e_schedule``) and equal the
reference's ``MulCounters`` exactly.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

from . import _device, _lib
from .gf2e import FieldCtx, field_new
from .mat_gf2 import BitMatrix, words_for
from .mat_packed import PackedMatrix
from .mat_sliced import SlicedMatrix, cling, slice_packed

_BACKENDS = {"tc": _lib.BACKEND_TC, "tc_i8": _lib.BACKEND_TC | _lib.TC_INT8, "tc_fp4": _lib.BACKEND_TC | _lib.TC_FP4,
             "tc_run": _lib.BACKEND_TC | _lib.TC_RUN, "m4rm": _lib.BACKEND_M4RM}
DEFAULT_BACKEND = os.environ.get("GF2E_BACKEND", "tc")


def _resolve_backend(backend: str | None) -> int:
    b = DEFAULT_BACKEND if backend is None else backend
    if b not in _BACKENDS:
        raise ValueError(f"unknown backend {b!r}; expected one of {sorted(_BACKENDS)}")
    return _BACKENDS[b]


@dataclass
class MulCounters:
    """Operation counts accumulated over one multiplication call (poly_mul.py:32-43).

    The three reference fields carry the reference's accounting exactly: every Karatsuba
    multiplication the reference would perform adds K(e) GF(2) products and the schedule's
    additions (replayed from the same schedule), including those inside TRSM / PLE /
    echelonize, where the reference's recursion with the given crossover is replayed on the
    factorisation's rank profile (ple_echelon.py:130-136).  ``device_products`` (not part of
    equality) counts the GF(2) plane products this library actually launched on the GPU."""

    gf2_matmul_count: int = 0
    additions: int = 0
    peak_live_products: int = 0
    device_products: int = field(default=0, compare=False)

    def reset(self) -> None:
        self.gf2_matmul_count = 0
        self.additions = 0
        self.peak_live_products = 0
        self.device_products = 0


@dataclass(frozen=True)
class Schedule:
    """The Karatsuba schedule for (e, f) as computed natively by the library."""

    e: int
    f: int
    subsets: tuple[int, ...]   # operand t = XOR of input planes in subsets[t]
    outmap: tuple[int, ...]    # output plane j = XOR of products in outmap[j] (M = R_f . Gamma)
    counters: tuple[int, int, int]

    @property
    def n_products(self) -> int:
        return len(self.subsets)


_SCHED_CACHE: dict[tuple[int, int], Schedule] = {}


def schedule(e: int, f: int | None = None) -> Schedule:
    """Native schedule (no GPU needed): symbolic replay of poly_mul.py:166-242 in C++."""
    ctx = field_new(e, f)
    key = (ctx.e, ctx.f)
    s = _SCHED_CACHE.get(key)
    if s is None:
        n = ctypes.c_int()
        subsets = (ctypes.c_uint64 * 64)()
        outmap = (ctypes.c_uint64 * 10)()
        cnt = (ctypes.c_int64 * 3)()
        _lib.check(_lib.load().gf2e_schedule(ctx.e, ctx.f, ctypes.byref(n), subsets, outmap, cnt), "gf2e_schedule")
        s = Schedule(ctx.e, ctx.f, tuple(int(subsets[t]) for t in range(n.value)),
                     tuple(int(outmap[j]) for j in range(ctx.e)), (int(cnt[0]), int(cnt[1]), int(cnt[2])))
        _SCHED_CACHE[key] = s
    return s


def _bump(counters: MulCounters | None, ctx: FieldCtx, calls: int = 1, device_products: int | None = None) -> None:
    """Add `calls` reference Karatsuba multiplications (poly_mul.py:146-150 / 245-259
    bookkeeping) and the GF(2) products launched on the device (default: K(e) per call)."""
    if counters is None:
        return
    g, adds, peak = schedule(ctx.e, ctx.f).counters
    counters.gf2_matmul_count += g * calls
    counters.additions += adds * calls
    if calls and peak > counters.peak_live_products:
        counters.peak_live_products = peak
    counters.device_products += g * calls if device_products is None else device_products


def _check_operands(A: SlicedMatrix, B: SlicedMatrix) -> None:
    if A.ctx != B.ctx:
        raise ValueError(f"field mismatch: {A.ctx} vs {B.ctx}")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")


def _slice_mul(A: SlicedMatrix, B: SlicedMatrix, C: SlicedMatrix, accumulate: bool, backend: str | None) -> None:
    ctx = A.ctx
    m, k, n = A.nrows, A.ncols, B.ncols
    flags = _resolve_backend(backend) | (_lib.ACCUMULATE if accumulate else 0)
    L = _lib.load()
    ws_bytes = int(L.gf2e_slice_mul_workspace(ctx.e, ctx.f, m, k, n, flags))
    if ws_bytes < 0:
        _lib.check(_lib.GF2E_EINVAL, "gf2e_slice_mul_workspace")
    stream = _device.stream_handle()
    ws = _device.workspace.get(ws_bytes, stream)
    lda, ldb, ldc = A.planes.shape[2], B.planes.shape[2], C.planes.shape[2]
    _lib.call("gf2e_slice_mul", ctx.e, ctx.f, _device.ptr(A.planes), lda, m * lda, _device.ptr(B.planes), ldb,
              k * ldb, _device.ptr(C.planes), ldc, m * ldc, m, k, n, flags, ws.data_ptr(), ws.numel(), stream)


def karatsuba_mul(A: SlicedMatrix, B: SlicedMatrix, counters: MulCounters | None = None,
                  backend: str | None = None) -> SlicedMatrix:
    """GF(2^e) product via slice-polynomial Karatsuba plus reduction (poly_mul.py:245-259)."""
    _check_operands(A, B)
    C = SlicedMatrix(A.ctx, A.nrows, B.ncols, _device.empty_words((A.ctx.e, A.nrows, words_for(B.ncols))))
    _slice_mul(A, B, C, False, backend)
    _bump(counters, A.ctx)
    return C


def addmul(C: SlicedMatrix, A: SlicedMatrix, B: SlicedMatrix, counters: MulCounters | None = None,
           backend: str | None = None) -> SlicedMatrix:
    """C ^= A*B in place (mzd_slice_addmul) — the reference's ``X ^= karatsuba_mul(A, B)``."""
    _check_operands(A, B)
    if C.ctx != A.ctx:
        raise ValueError(f"field mismatch: {C.ctx} vs {A.ctx}")
    if C.shape != (A.nrows, B.ncols):
        raise ValueError(f"dimension mismatch: {C.shape} vs {(A.nrows, B.ncols)}")
    _slice_mul(A, B, C, True, backend)
    _bump(counters, A.ctx)
    return C


def reduce_mod_f(slices: list[BitMatrix], ctx: FieldCtx, counters: MulCounters | None = None) -> list[BitMatrix]:
    """Fold a degree-(2e-2) slice polynomial to degree < e (poly_mul.py:223-242), on device."""
    e = ctx.e
    if len(slices) != 2 * e - 1:
        raise ValueError(f"expected {2 * e - 1} coefficient slices, got {len(slices)}")
    m, n = slices[0].shape
    work = _device.empty_words((2 * e - 1, m, words_for(n)))
    for d, s in enumerate(slices):
        work[d].copy_(s.words)
    nw = words_for(n)
    if m and nw:
        _lib.call("gf2e_reduce_mod_f", e, ctx.f, _device.ptr(work), m, nw, nw, m * nw, _device.stream_handle())
    if counters is not None:
        counters.additions += sum(1 for _ in range(2 * e - 2, e - 1, -1) for k in range(e) if (ctx.f >> k) & 1)
    return [BitMatrix(m, n, work[j].clone()) for j in range(e)]


def count_products(e: int, f: int | None = None) -> int:
    """GF(2) products per Karatsuba multiplication (poly_mul.py:262-272); host-only."""
    return schedule(e, f).n_products


# Up to this size (max of m, k, n) per field degree, products of packed matrices take the
# one-launch packed-domain Newton-John kernel (gf2e_nj_mul) instead of slice -> combos ->
# product -> cling.  Measured crossovers of square products on the B200
# (tools/nj_crossover.py, profiles/r02/nj_crossover.jsonl): the table kernel wins up to these
# sizes; GF2E_NJ_CROSSOVER overrides all degrees.
NJ_CROSSOVER = {2: 256, 3: 128, 4: 128, 5: 96, 6: 96, 7: 96, 8: 64, 9: 32, 10: 32}
if os.environ.get("GF2E_NJ_CROSSOVER"):
    NJ_CROSSOVER = {e: int(os.environ["GF2E_NJ_CROSSOVER"]) for e in NJ_CROSSOVER}


def nj_fits(e: int, n: int) -> bool:
    from .mat_packed import pack_width

    return words_for(n * pack_width(e)) <= 16


def nj_mul_packed(A: PackedMatrix, B: PackedMatrix, C: PackedMatrix | None = None) -> PackedMatrix:
    """C = A*B (or C ^= A*B when C is given) on packed words in one launch (gf2e_nj_mul):
    Newton-John tables of the rows of B in shared memory (newton_john.py:145-164)."""
    ctx = A.ctx
    m, k, n = A.nrows, A.ncols, B.ncols
    acc = C is not None
    if C is None:
        C = PackedMatrix(ctx, m, n)
    aw, bw, cw = A.storage.words, B.storage.words, C.storage.words
    _lib.call("gf2e_nj_mul", ctx.e, ctx.f, _device.ptr(aw), aw.shape[1], _device.ptr(bw), bw.shape[1],
              _device.ptr(cw), cw.shape[1], m, k, n, _lib.ACCUMULATE if acc else 0, _device.stream_handle())
    return C


def nj_mul_sliced(A: SlicedMatrix, B: SlicedMatrix, C: SlicedMatrix | None = None) -> SlicedMatrix:
    """C = A*B (or C ^= A*B when C is given) on bit planes in one launch (gf2e_nj_slice_mul):
    the Newton-John table product that PLE and TRSM use for their small updates."""
    _check_operands(A, B)
    ctx = A.ctx
    m, k, n = A.nrows, A.ncols, B.ncols
    acc = C is not None
    if C is None:
        C = SlicedMatrix(ctx, m, n)
    lda, ldb, ldc = A.planes.shape[2], B.planes.shape[2], C.planes.shape[2]
    _lib.call("gf2e_nj_slice_mul", ctx.e, ctx.f, _device.ptr(A.planes), lda, m * lda, _device.ptr(B.planes), ldb,
              k * ldb, _device.ptr(C.planes), ldc, m * ldc, m, k, n, _lib.ACCUMULATE if acc else 0,
              _device.stream_handle())
    return C


def _small(A: PackedMatrix, B: PackedMatrix, backend: str | None) -> bool:
    return (backend is None and max(A.nrows, A.ncols, B.ncols) <= NJ_CROSSOVER[A.ctx.e]
            and nj_fits(A.ctx.e, B.ncols))


def karatsuba_mul_packed(A: PackedMatrix, B: PackedMatrix, counters: MulCounters | None = None,
                         backend: str | None = None) -> PackedMatrix:
    """Slice, multiply, cling back (poly_mul.py:275-278): K1 -> K3/K4/K5 -> K2; below
    NJ_CROSSOVER the packed-domain Newton-John kernel (same product, one launch)."""
    if _small(A, B, backend):
        if A.ctx != B.ctx:
            raise ValueError(f"field mismatch: {A.ctx} vs {B.ctx}")
        if A.ncols != B.nrows:
            raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")
        C = nj_mul_packed(A, B)
        _bump(counters, A.ctx, 1, device_products=0)
        return C
    return cling(karatsuba_mul(slice_packed(A), slice_packed(B), counters, backend))


def addmul_packed(C: PackedMatrix, A: PackedMatrix, B: PackedMatrix, counters: MulCounters | None = None,
                  backend: str | None = None) -> PackedMatrix:
    """C ^= A*B on packed matrices (mzed_addmul), through the sliced path; C updated in place."""
    if A.ctx != B.ctx or C.ctx != A.ctx:
        raise ValueError(f"field mismatch: {A.ctx} vs {B.ctx}")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")
    if C.shape != (A.nrows, B.ncols):
        raise ValueError(f"dimension mismatch: {C.shape} vs {(A.nrows, B.ncols)}")
    if _small(A, B, backend):
        nj_mul_packed(A, B, C)
        _bump(counters, A.ctx, 1, device_products=0)
        return C
    Cs = slice_packed(C)
    addmul(Cs, slice_packed(A), slice_packed(B), counters, backend)
    cling(Cs, out=C)
    return C


def karatsuba_mul_packed_host(ctx: FieldCtx, A_words, k: int, B_words, n: int, C_words=None,
                              chunk_rows: int = 0, counters: MulCounters | None = None, out=None):
    """mzed_mul / mzed_addmul on HOST packed words (reference ``PackedMatrix.storage.words``):
    returns (C words, device ms).  With ``C_words`` the product is XOR-ed into it in place.
    One synchronous ``gf2e_mzed_mul_host`` call: B uploaded and prepared once, rows of A
    streamed in chunks with copies overlapping the kernels (use pinned arrays for overlap).
    ``out``: optional preallocated (pinned) result array for C = A*B."""
    import numpy as np

    from .mat_packed import pack_width

    import torch

    A = np.ascontiguousarray(A_words, dtype=np.uint64)
    b_dev = isinstance(B_words, torch.Tensor) and B_words.is_cuda
    if b_dev:  # B already on this GPU (e.g. broadcast by the multi-GPU path): no upload
        if B_words.dtype != torch.int64 or B_words.dim() != 2 or not B_words.is_contiguous():
            raise ValueError("a device B_words must be a contiguous 2-D int64 tensor of packed words")
        B = B_words
        torch.cuda.current_stream().synchronize()  # the call runs on its own streams
    else:
        B = np.ascontiguousarray(B_words, dtype=np.uint64)
    w = pack_width(ctx.e)
    wa, wb = words_for(k * w), words_for(n * w)
    if A.ndim != 2 or B.ndim != 2:
        raise ValueError("A_words and B_words must be 2-D arrays of packed words")
    m = A.shape[0]
    if B.shape[0] != k:
        raise ValueError(f"inner dimensions differ: {m}x{k} times {B.shape[0]}x{n}")
    if A.shape[1] < wa:
        raise ValueError(f"A_words has {A.shape[1]} words per row, need {wa} for {k} columns")
    if B.shape[1] < wb:
        raise ValueError(f"B_words has {B.shape[1]} words per row, need {wb} for {n} columns")

    def _check_out(C, name):
        if not isinstance(C, np.ndarray) or C.dtype != np.uint64 or not C.flags.c_contiguous:
            raise ValueError(f"{name} must be a C-contiguous uint64 array")
        if C.ndim != 2 or C.shape[0] != m or C.shape[1] < wb:
            raise ValueError(f"{name} must have shape ({m}, >= {wb}), got {C.shape}")
        if not C.flags.writeable:
            raise ValueError(f"{name} must be writeable")

    acc = C_words is not None
    if acc:
        C = C_words
        _check_out(C, "C_words")
    elif out is not None:
        C = out
        _check_out(C, "out")
    else:
        C = np.empty((m, wb), dtype=np.uint64)
    ms = ctypes.c_double()
    flags = (_lib.ACCUMULATE if acc else 0) | (_lib.B_DEVICE if b_dev else 0)
    _lib.call("gf2e_mzed_mul_host", ctx.e, ctx.f, A.ctypes.data, A.shape[1],
              B.data_ptr() if b_dev else B.ctypes.data, B.shape[1], C.ctypes.data, C.shape[1], m, k, n, flags,
              chunk_rows, ctypes.byref(ms))
    _bump(counters, ctx)
    return C, ms.value


# M4RIE vocabulary (BASELINE.json north star)
mzd_slice_mul = karatsuba_mul
mzd_slice_addmul = addmul
mzed_mul = karatsuba_mul_packed
mzed_addmul = addmul_packed
mzed_mul_host = karatsuba_mul_packed_host

"""Dense GF(2) matrices (M4RI ``mzd_t``) resident in HBM — drop-in for ``gf2elin.mat_gf2``.

Layout is the reference's (``mat_gf2.py:3-7``): entry (i, j) is bit j % 64 of word j // 64
of row i, bits past ``ncols`` zero.  ``words`` is a CUDA int64 tensor of shape
(nrows, ceil(ncols/64)) holding exactly the reference's uint64 words, so
``BitMatrix.to_numpy()`` equals the reference ``BitMatrix.words`` bit for bit.

``mul`` / ``addmul`` run the GF(2) plane product on the B200 (``gf2e_plane_mul``); the
reference's CPU strategies ("auto", "cubic", "m4rm", "strassen") are accepted for API
compatibility — all give bit-identical results there (``mat_gf2.py:435-436``) and here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib


@dataclass
class RowOpCounters:
    """mat_gf2.py:32-41 (kept for API parity)."""

    row_adds: int = 0
    scalar_row_muls: int = 0

    def reset(self) -> None:
        self.row_adds = 0
        self.scalar_row_muls = 0


def words_for(ncols: int) -> int:
    return (ncols + 63) >> 6


def tail_mask(ncols: int) -> int:
    r = ncols & 63
    return (1 << 64) - 1 if r == 0 else (1 << r) - 1


class BitMatrix:
    """A dense GF(2) matrix stored as an (nrows, words) int64 tensor on the GPU."""

    __slots__ = ("nrows", "ncols", "words")

    def __init__(self, nrows: int, ncols: int, words: torch.Tensor | np.ndarray | None = None):
        if nrows < 0 or ncols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        self.nrows = nrows
        self.ncols = ncols
        width = words_for(ncols)
        if words is None:
            self.words = _device.zeros_words((nrows, width))
        else:
            if isinstance(words, np.ndarray):
                if words.shape != (nrows, width) or words.dtype != np.uint64:
                    raise ValueError("backing array has the wrong shape or dtype")
                words = _device.to_device_words(words)
            elif tuple(words.shape) != (nrows, width) or words.dtype != torch.int64 or not words.is_cuda:
                raise ValueError("backing array has the wrong shape or dtype")
            self.words = words

    # -- construction / interop ------------------------------------------------------
    @classmethod
    def from_numpy(cls, words: np.ndarray, ncols: int) -> "BitMatrix":
        """From reference-layout uint64 words (e.g. a reference ``BitMatrix.words``)."""
        words = np.asarray(words, dtype=np.uint64)
        return cls(words.shape[0], ncols, np.ascontiguousarray(words))

    def to_numpy(self) -> np.ndarray:
        return _device.to_host_words(self.words)

    @classmethod
    def from_array(cls, arr) -> "BitMatrix":
        """From an (m, n) array of 0/1 values (mat_gf2.py:92-103)."""
        arr = np.asarray(arr)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d array")
        m, n = arr.shape
        words = np.zeros((m, words_for(n)), dtype=np.uint64)
        if m and n:
            packed = np.packbits(arr.astype(np.uint8) & 1, axis=1, bitorder="little")
            words.view(np.uint8)[:, : packed.shape[1]] = packed
        return cls(m, n, words)

    def to_array(self) -> np.ndarray:
        if self.nrows == 0 or self.ncols == 0:
            return np.zeros((self.nrows, self.ncols), dtype=np.uint8)
        bits = np.unpackbits(self.to_numpy().view(np.uint8), axis=1, bitorder="little")
        return np.ascontiguousarray(bits[:, : self.ncols])

    @classmethod
    def identity(cls, n: int) -> "BitMatrix":
        return cls.from_array(np.eye(n, dtype=np.uint8))

    @classmethod
    def random(cls, nrows: int, ncols: int, seed: int) -> "BitMatrix":
        """Reproducible bits, identical to the reference BitMatrix.random (mat_gf2.py:194-206)."""
        out = cls(nrows, ncols)
        out.randomize(seed)
        return out

    def randomize(self, seed: int) -> None:
        _device.require_cuda()
        _lib.call("gf2e_random_words", self.nrows, self.ncols, seed & (2**64 - 1), _device.ptr(self.words),
                  self.words.shape[1], _device.stream_handle())

    def copy(self) -> "BitMatrix":
        return BitMatrix(self.nrows, self.ncols, self.words.clone())

    # -- protocol -----------------------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def __eq__(self, other) -> bool:
        return (isinstance(other, BitMatrix) and self.shape == other.shape
                and bool(torch.equal(self.words, other.words)))

    def __repr__(self) -> str:
        return f"BitMatrix({self.nrows}x{self.ncols}, cuda)"

    def _check_index(self, i: int, j: int) -> None:
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError(f"index ({i}, {j}) outside {self.nrows}x{self.ncols}")

    def get(self, i: int, j: int) -> int:
        self._check_index(i, j)
        w, s = divmod(j, 64)
        return (int(self.words[i, w].item()) >> s) & 1

    def set(self, i: int, j: int, value: int) -> None:
        self._check_index(i, j)
        w, s = divmod(j, 64)
        cur = int(self.words[i, w].item()) & ((1 << 64) - 1)
        cur = (cur | (1 << s)) if value & 1 else (cur & ~(1 << s))
        self.words[i, w] = np.uint64(cur).astype(np.int64).item()

    # -- arithmetic ---------------------------------------------------------------------
    def add(self, other: "BitMatrix") -> "BitMatrix":
        """Entrywise XOR (mat_gf2.py:151-157)."""
        if self.shape != other.shape:
            raise ValueError(f"dimension mismatch: {self.shape} vs {other.shape}")
        out = self.copy()
        out.iadd(other)
        return out

    __xor__ = add

    def iadd(self, other: "BitMatrix") -> None:
        if self.shape != other.shape:
            raise ValueError(f"dimension mismatch: {self.shape} vs {other.shape}")
        nw = self.words.shape[1]
        _lib.call("gf2e_xor", _device.ptr(self.words), nw, _device.ptr(other.words), nw, self.nrows, nw,
                  _device.stream_handle())

    def is_zero(self) -> bool:
        return not bool(self.words.any().item())


_STRATEGIES = ("auto", "cubic", "m4rm", "strassen")


def _backend_flags(backend: str | None) -> int:
    from .poly_mul import _resolve_backend

    return _resolve_backend(backend)


def _plane_mul(A: BitMatrix, B: BitMatrix, C: BitMatrix, accumulate: bool, backend: str | None) -> None:
    flags = _backend_flags(backend) | (_lib.ACCUMULATE if accumulate else 0)
    m, k, n = A.nrows, A.ncols, B.ncols
    L = _lib.load()
    ws_bytes = int(L.gf2e_plane_mul_workspace(m, k, n, flags))
    ws = _device.workspace.get(ws_bytes)
    _lib.call("gf2e_plane_mul", _device.ptr(A.words), A.words.shape[1], _device.ptr(B.words), B.words.shape[1],
              _device.ptr(C.words), C.words.shape[1], m, k, n, flags, ws.data_ptr(), ws.numel(),
              _device.stream_handle())


def mul(A: BitMatrix, B: BitMatrix, strategy: str = "auto", crossover: int | None = None,
        m4rm_k: int | None = None, counters=None, backend: str | None = None) -> BitMatrix:
    """GF(2) product A*B (mzd_mul; reference mat_gf2.py:425-455), computed on the B200."""
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")
    if strategy not in _STRATEGIES:
        raise ValueError(f"unknown multiplication strategy: {strategy!r}")
    if counters is not None:
        counters.gf2_matmul_count += 1
    C = BitMatrix(A.nrows, B.ncols, _device.empty_words((A.nrows, words_for(B.ncols))))
    _plane_mul(A, B, C, False, backend)
    return C


def addmul(C: BitMatrix, A: BitMatrix, B: BitMatrix, counters=None, backend: str | None = None) -> BitMatrix:
    """C ^= A*B in place (mzd_addmul; the reference's iadd-after-mul pattern, mat_gf2.py:161-164)."""
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")
    if C.shape != (A.nrows, B.ncols):
        raise ValueError(f"dimension mismatch: {C.shape} vs {(A.nrows, B.ncols)}")
    if counters is not None:
        counters.gf2_matmul_count += 1
    _plane_mul(A, B, C, True, backend)
    return C


mzd_mul = mul
mzd_addmul = addmul

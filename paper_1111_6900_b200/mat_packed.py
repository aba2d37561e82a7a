"""Bit-packed GF(2^e) matrices (M4RIE ``mzed_t``) in HBM — drop-in for ``gf2elin.mat_packed``.

Element (i, j) occupies bits [j*w, j*w + e) of the packed row, w = ``pack_width(e)`` the
smallest divisor of 64 >= e, pad bits zero (``mat_packed.py:1-33``).  The storage is a
device ``BitMatrix`` of nrows x (ncols*w) bits, word-identical to the reference.
``PackedMatrix.random`` runs the reference's counter-mode splitmix64 generator
(``rng.py:20-35``, ``mat_packed.py:253-265``) on the GPU (kernel K7), bit-exact.
"""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from .gf2e import FieldCtx
from .mat_gf2 import BitMatrix, words_for

_PACK_WIDTHS = (1, 2, 4, 8, 16, 32, 64)


def pack_width(e: int) -> int:
    """Smallest divisor of 64 that fits an e-bit element (mat_packed.py:26-33)."""
    if not 2 <= e <= 10:
        raise ValueError(f"extension degree must be in 2..10, got {e}")
    for w in _PACK_WIDTHS:
        if w >= e:
            return w
    raise AssertionError("unreachable")


class PackedMatrix:
    """GF(2^e) matrix with w-bit packed elements over a device BitMatrix."""

    __slots__ = ("ctx", "nrows", "ncols", "w", "storage")

    def __init__(self, ctx: FieldCtx, nrows: int, ncols: int, storage: BitMatrix | None = None):
        self.ctx = ctx
        self.nrows = nrows
        self.ncols = ncols
        self.w = pack_width(ctx.e)
        if storage is None:
            storage = BitMatrix(nrows, ncols * self.w)
        elif storage.shape != (nrows, ncols * self.w):
            raise ValueError("backing BitMatrix has the wrong shape")
        self.storage = storage

    # -- construction / interop ------------------------------------------------------
    @classmethod
    def from_array(cls, ctx: FieldCtx, arr) -> "PackedMatrix":
        """From an (m, n) array of field elements < 2^e (mat_packed.py:95-112)."""
        arr = np.asarray(arr)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d array")
        if arr.size and int(arr.max()) >= ctx.order:
            raise ValueError(f"element {int(arr.max())} out of range for GF(2^{ctx.e})")
        m, n = arr.shape
        w = pack_width(ctx.e)
        per = 64 // w
        words = np.zeros((m, words_for(n * w)), dtype=np.uint64)
        a = arr.astype(np.uint64)
        for s in range(per):
            cols = a[:, s::per]
            words[:, : cols.shape[1]] |= cols << np.uint64(s * w)
        return cls(ctx, m, n, BitMatrix(m, n * w, words))

    @classmethod
    def from_numpy(cls, ctx: FieldCtx, words: np.ndarray, ncols: int) -> "PackedMatrix":
        """From reference packed storage words (a reference ``PackedMatrix.storage.words``)."""
        w = pack_width(ctx.e)
        return cls(ctx, words.shape[0], ncols, BitMatrix.from_numpy(words, ncols * w))

    def to_numpy(self) -> np.ndarray:
        return self.storage.to_numpy()

    def to_array(self) -> np.ndarray:
        """(m, n) uint16 element values (mat_packed.py:114-122)."""
        m, n, w = self.nrows, self.ncols, self.w
        if m == 0 or n == 0:
            return np.zeros((m, n), dtype=np.uint16)
        words = self.to_numpy()
        per = 64 // w
        out = np.zeros((m, n), dtype=np.uint16)
        mask = np.uint64((1 << self.ctx.e) - 1)
        for s in range(per):
            cols = (words >> np.uint64(s * w)) & mask
            k = out[:, s::per].shape[1]
            out[:, s::per] = cols[:, :k].astype(np.uint16)
        return out

    @classmethod
    def identity(cls, ctx: FieldCtx, n: int) -> "PackedMatrix":
        return cls.from_array(ctx, np.eye(n, dtype=np.uint16))

    def randomize(self, seed: int) -> None:
        """Reference-identical pseudo-random elements (mat_packed.py:253-259), generated on device."""
        if self.nrows == 0 or self.ncols == 0:
            return
        _lib.call("gf2e_random_packed", self.ctx.e, self.nrows, self.ncols, seed & (2**64 - 1), 0, 0, self.ncols,
                  _device.ptr(self.storage.words), self.storage.words.shape[1], _device.stream_handle())

    @classmethod
    def random(cls, ctx: FieldCtx, nrows: int, ncols: int, seed: int) -> "PackedMatrix":
        out = cls(ctx, nrows, ncols, BitMatrix(nrows, ncols * pack_width(ctx.e),
                                               _device.empty_words((nrows, words_for(ncols * pack_width(ctx.e))))))
        if nrows and ncols:
            out.randomize(seed)
        else:
            out.storage.words.zero_()
        return out

    def copy(self) -> "PackedMatrix":
        return PackedMatrix(self.ctx, self.nrows, self.ncols, self.storage.copy())

    # -- protocol -------------------------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def __eq__(self, other) -> bool:
        return (isinstance(other, PackedMatrix) and self.ctx == other.ctx and self.shape == other.shape
                and self.storage == other.storage)

    def __repr__(self) -> str:
        return f"PackedMatrix(GF(2^{self.ctx.e}), {self.nrows}x{self.ncols}, cuda)"

    def _check_index(self, i: int, j: int) -> None:
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError(f"index ({i}, {j}) outside {self.nrows}x{self.ncols}")

    def get(self, i: int, j: int) -> int:
        self._check_index(i, j)
        wrd, s = divmod(j * self.w, 64)
        return (int(self.storage.words[i, wrd].item()) >> s) & ((1 << self.w) - 1)

    def set(self, i: int, j: int, value: int) -> None:
        self._check_index(i, j)
        if not 0 <= value < self.ctx.order:
            raise ValueError(f"element {value} out of range for GF(2^{self.ctx.e})")
        wrd, s = divmod(j * self.w, 64)
        cur = int(self.storage.words[i, wrd].item()) & ((1 << 64) - 1)
        slot = ((1 << self.w) - 1) << s
        cur = (cur & ~slot) | (value << s)
        self.storage.words[i, wrd] = np.uint64(cur).astype(np.int64).item()

    # -- arithmetic -----------------------------------------------------------------------
    def _check_compat(self, other: "PackedMatrix") -> None:
        if self.ctx != other.ctx:
            raise ValueError(f"field mismatch: {self.ctx} vs {other.ctx}")
        if self.shape != other.shape:
            raise ValueError(f"dimension mismatch: {self.shape} vs {other.shape}")

    def add(self, other: "PackedMatrix") -> "PackedMatrix":
        """Entrywise field addition: one XOR sweep (mat_packed.py:180-186)."""
        self._check_compat(other)
        return PackedMatrix(self.ctx, self.nrows, self.ncols, self.storage.add(other.storage))

    __xor__ = add

    def iadd(self, other: "PackedMatrix") -> None:
        self._check_compat(other)
        self.storage.iadd(other.storage)

    def is_zero(self) -> bool:
        return self.storage.is_zero()

    def scalar_mul(self, c: int) -> "PackedMatrix":
        """Every entry multiplied by the scalar c (mat_packed.py:192-199), on device."""
        if not 0 <= c < self.ctx.order:
            raise ValueError(f"scalar {c} out of range for GF(2^{self.ctx.e})")
        ld = self.storage.words.shape[1]
        out = PackedMatrix(self.ctx, self.nrows, self.ncols,
                           BitMatrix(self.nrows, self.ncols * self.w, _device.empty_words((self.nrows, ld))))
        if self.nrows and ld:
            _lib.call("gf2e_scalar_mul", self.ctx.e, self.ctx.f, c, _device.ptr(self.storage.words), ld,
                      _device.ptr(out.storage.words), ld, self.nrows, self.ncols, _device.stream_handle())
        return out

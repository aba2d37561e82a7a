"""Bitsliced GF(2^e) matrices (M4RIE ``mzd_slice_t``) in HBM — drop-in for ``gf2elin.mat_sliced``.

Device layout: ONE (e, nrows, ceil(ncols/64)) int64 tensor; plane t holds the x^t
coefficient of every entry in the reference BitMatrix word layout.  ``slices`` returns
BitMatrix views of the planes (writes through), so code written against the reference's
``list[BitMatrix]`` keeps working.  ``slice_packed`` / ``cling`` are kernels K1 / K2.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .gf2e import FieldCtx
from .mat_gf2 import BitMatrix, words_for
from .mat_packed import PackedMatrix, pack_width


class SlicedMatrix:
    """GF(2^e) matrix stored as e coefficient planes of equal shape (mat_sliced.py:22-94)."""

    __slots__ = ("ctx", "nrows", "ncols", "planes")

    def __init__(self, ctx: FieldCtx, nrows: int, ncols: int, slices=None):
        self.ctx = ctx
        self.nrows = nrows
        self.ncols = ncols
        nw = words_for(ncols)
        if slices is None:
            self.planes = _device.zeros_words((ctx.e, nrows, nw))
        elif isinstance(slices, torch.Tensor):
            if tuple(slices.shape) != (ctx.e, nrows, nw) or slices.dtype != torch.int64:
                raise ValueError("need e slices of identical shape")
            self.planes = slices
        else:
            slices = list(slices)
            if len(slices) != ctx.e or any(s.shape != (nrows, ncols) for s in slices):
                raise ValueError("need e slices of identical shape")
            self.planes = (torch.stack([s.words for s in slices]) if slices
                           else _device.zeros_words((0, nrows, nw)))

    @property
    def slices(self) -> list[BitMatrix]:
        return [BitMatrix(self.nrows, self.ncols, self.planes[t]) for t in range(self.ctx.e)]

    # -- interop ----------------------------------------------------------------------
    @classmethod
    def from_numpy(cls, ctx: FieldCtx, planes: np.ndarray, ncols: int) -> "SlicedMatrix":
        planes = np.ascontiguousarray(planes, dtype=np.uint64)
        return cls(ctx, planes.shape[1], ncols, _device.to_device_words(planes))

    def to_numpy(self) -> np.ndarray:
        return _device.to_host_words(self.planes)

    def to_array(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols), dtype=np.uint16)
        for k, s in enumerate(self.slices):
            out |= s.to_array().astype(np.uint16) << k
        return out

    # -- protocol -----------------------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def __eq__(self, other) -> bool:
        return (isinstance(other, SlicedMatrix) and self.ctx == other.ctx and self.shape == other.shape
                and bool(torch.equal(self.planes, other.planes)))

    def __repr__(self) -> str:
        return f"SlicedMatrix(GF(2^{self.ctx.e}), {self.nrows}x{self.ncols}, cuda)"

    def copy(self) -> "SlicedMatrix":
        return SlicedMatrix(self.ctx, self.nrows, self.ncols, self.planes.clone())

    def get(self, i: int, j: int) -> int:
        return sum(s.get(i, j) << k for k, s in enumerate(self.slices))

    def set(self, i: int, j: int, value: int) -> None:
        if not 0 <= value < self.ctx.order:
            raise ValueError(f"element {value} out of range for GF(2^{self.ctx.e})")
        for k, s in enumerate(self.slices):
            s.set(i, j, (value >> k) & 1)

    def _check_compat(self, other: "SlicedMatrix") -> None:
        if self.ctx != other.ctx:
            raise ValueError(f"field mismatch: {self.ctx} vs {other.ctx}")
        if self.shape != other.shape:
            raise ValueError(f"dimension mismatch: {self.shape} vs {other.shape}")

    def iadd(self, other: "SlicedMatrix") -> None:
        self._check_compat(other)
        rows = self.ctx.e * self.nrows
        nw = self.planes.shape[2]
        _lib.call("gf2e_xor", _device.ptr(self.planes), nw, _device.ptr(other.planes), nw, rows, nw,
                  _device.stream_handle())

    def add(self, other: "SlicedMatrix") -> "SlicedMatrix":
        """Slicewise XOR (mat_sliced.py:69-72)."""
        self._check_compat(other)
        out = self.copy()
        out.iadd(other)
        return out

    __xor__ = add

    @classmethod
    def random(cls, ctx: FieldCtx, nrows: int, ncols: int, seed: int, row0: int = 0,
               gcols: int | None = None) -> "SlicedMatrix":
        """slice_packed(PackedMatrix.random(ctx, nrows, ncols, seed)) generated directly as planes
        (K7).  With row0/gcols: the row block [row0, row0+nrows) of an (* x gcols) matrix."""
        nw = words_for(ncols)
        out = cls(ctx, nrows, ncols, _device.empty_words((ctx.e, nrows, nw)))
        if nrows and nw:
            _lib.call("gf2e_random_sliced", ctx.e, nrows, ncols, seed & (2**64 - 1), row0, 0,
                      ncols if gcols is None else gcols, _device.ptr(out.planes), nw, nrows * nw,
                      _device.stream_handle())
        else:
            out.planes.zero_()
        return out


def slice_packed(A: PackedMatrix, out: SlicedMatrix | None = None) -> SlicedMatrix:
    """Packed -> sliced (mzed -> mzd_slice; mat_sliced.py:97-101), kernel K1."""
    e, m, n = A.ctx.e, A.nrows, A.ncols
    nw = words_for(n)
    if out is None:
        out = SlicedMatrix(A.ctx, m, n, _device.empty_words((e, m, nw)))
    elif out.ctx != A.ctx or out.shape != A.shape:
        raise ValueError("output has the wrong field or shape")
    if m and nw:
        _lib.call("gf2e_slice", e, m, n, _device.ptr(A.storage.words), A.storage.words.shape[1],
                  _device.ptr(out.planes), nw, m * nw, _device.stream_handle())
    return out


def cling(S: SlicedMatrix, out: PackedMatrix | None = None) -> PackedMatrix:
    """Sliced -> packed, pad bits zero (mzd_slice -> mzed; mat_sliced.py:104-106), kernel K2."""
    e, m, n = S.ctx.e, S.nrows, S.ncols
    w = pack_width(e)
    ldp = words_for(n * w)
    if out is None:
        out = PackedMatrix(S.ctx, m, n, BitMatrix(m, n * w, _device.empty_words((m, ldp))))
    elif out.ctx != S.ctx or out.shape != S.shape:
        raise ValueError("output has the wrong field or shape")
    if m and ldp:
        nw = S.planes.shape[2]
        _lib.call("gf2e_cling", e, m, n, _device.ptr(S.planes), nw, m * nw, _device.ptr(out.storage.words), ldp,
                  _device.stream_handle())
    return out


def mul_by_x(S: SlicedMatrix) -> SlicedMatrix:
    """Every entry times alpha (the class of x), reduced mod f (mat_sliced.py:109-122), on device."""
    out = SlicedMatrix(S.ctx, S.nrows, S.ncols, _device.empty_words(tuple(S.planes.shape)))
    nw = S.planes.shape[2]
    if S.nrows and nw:
        _lib.call("gf2e_mul_by_x", S.ctx.e, S.ctx.f, _device.ptr(S.planes), nw, S.nrows * nw,
                  _device.ptr(out.planes), S.nrows * nw, S.nrows, S.ncols, _device.stream_handle())
    return out


mzed_slice = slice_packed
mzed_cling = cling

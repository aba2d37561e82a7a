"""Multi-GPU partitioning of the hot path: C row-blocks across ranks, B broadcast once.

SURVEY §8e.  Rows of C are independent (C[r, :] = A[r, :] . B (+ C0[r, :])), so rank g owns
rows [row0_g, row0_g + rows_g) of A, C0 and C and needs all of B.  The only collective on the
data path is the broadcast of B's e planes from the source rank (NCCL over NVLink/NVSwitch on
a B200 box; gloo in the CPU tests).  There is no reduction: results stay sharded;
``all_gather_rows`` exists for verification only.

The broadcast is split into column parts (``col_parts``): part p is its own contiguous plane
stack, broadcast on a side stream, and the product consumes the parts as they arrive
(``gf2e_slice_mul_parts``: A's operand combinations once, then after each part the product of
every column tile whose columns have all arrived), so only the first part's transfer is
exposed.

Everything here works on plane tensors ([e, rows, words] int64), device-agnostic, so the same
code runs under NCCL (CUDA tensors) and gloo (CPU tensors).  ``sharded_mul`` computes the local
block with the device kernel unless a ``compute`` callable is injected (the CPU tests inject
the oracle — test infrastructure only).
"""

from __future__ import annotations

import ctypes
import math
from typing import Callable

import torch
import torch.distributed as dist

from .mat_gf2 import words_for

ROW_ALIGN = 256  # one CTA-pair tile of C rows


def row_partition(m: int, world: int, align: int = ROW_ALIGN) -> list[tuple[int, int]]:
    """(row0, rows) per rank: whole `align`-row tiles dealt out as evenly as possible (the
    first ranks take one extra tile), the last non-empty block trimmed so the union is exactly
    [0, m).  With fewer tiles than ranks the tile shrinks (64 rows, then 1) so that no rank is
    left empty unless m < world."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if m < 0:
        raise ValueError("row count must be non-negative")
    while align > 1 and -(-m // align) < world:
        align = 64 if align > 64 else 1
    tiles = -(-m // align)
    base, extra = divmod(tiles, world)
    out, t0 = [], 0
    for g in range(world):
        nt = base + (1 if g < extra else 0)
        r0 = min(t0 * align, m)
        r1 = min((t0 + nt) * align, m)
        out.append((r0, r1 - r0))
        t0 += nt
    return out


def col_parts(n: int, parts: int, first_fraction: float = 0.125, tile: int = 768, rows: int | None = None,
              pairs: int | None = None) -> list[int]:
    """Column bounds of B's broadcast parts.  The first part is small (its transfer is the only
    one not hidden behind products); interior bounds are multiples of `tile` (whole product
    tiles, so no tile waits for two parts; 768 suits both the 256- and the 192-column forms).
    With `rows` (this rank's rows of C) and `pairs` (CTA pairs of the GPU) the first part is the
    smallest whole number of waves of tiles, so splitting the product costs no partial wave."""
    if parts <= 1 or n <= 2 * tile:
        return [0, n]
    first = max(tile, int(n * first_fraction) // tile * tile)
    if rows and pairs:
        rt = -(-rows // 256)
        step = pairs // math.gcd(rt, pairs)  # column tiles per whole wave
        c = step
        while c * tile < int(n * first_fraction):
            c += step
        if c * tile < n:
            first = c * tile
    bounds = [0, first]
    rest = n - first
    for p in range(1, parts - 1):
        b = first + -(-rest * p // (parts - 1) // tile) * tile
        if bounds[-1] < b < n:
            bounds.append(b)
    bounds.append(n)
    return bounds


def broadcast_planes(planes: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of a plane stack from `src` (the one data-path collective)."""
    if dist.is_initialized():
        dist.broadcast(planes, src=src, group=group)
    return planes


def split_parts(B: torch.Tensor, bounds: list[int]) -> list[torch.Tensor]:
    """Contiguous copies of B's column parts [bounds[p], bounds[p+1]) (word-aligned bounds)."""
    return [B[:, :, b0 // 64:words_for(b1)].contiguous() for b0, b1 in zip(bounds, bounds[1:])]


def broadcast_parts(B: torch.Tensor | None, shape: tuple[int, int, int], bounds: list[int], src: int = 0,
                    group=None, stream=None, device=None, src_parts: list[torch.Tensor] | None = None):
    """Broadcast B [e, k, words(n)] as contiguous column parts (one per `bounds` interval).
    On `src`, B holds the matrix; elsewhere it may be None.  Returns (parts, events): on CUDA
    the broadcasts are issued on `stream` (a side stream) and events[p] fires when part p has
    arrived; on CPU (gloo) the calls are synchronous and events are None.  src_parts: the
    source's parts already split (split_parts), so no copy is made on `src`."""
    e, k, _ = shape
    rank = dist.get_rank(group) if dist.is_initialized() else src
    dev = B.device if B is not None else (device or torch.device("cuda", torch.cuda.current_device()))
    if rank == src:
        parts = src_parts if src_parts is not None else split_parts(B, bounds)
    else:
        parts = [torch.empty((e, k, words_for(b1) - b0 // 64), dtype=torch.int64, device=dev)
                 for b0, b1 in zip(bounds, bounds[1:])]
    if dev.type != "cuda":
        for t in parts:
            broadcast_planes(t, src, group)
        return parts, [None] * len(parts)
    side = stream or torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))  # the part copies above
    events = []
    with torch.cuda.stream(side):
        for t in parts:
            if dist.is_initialized():
                work = dist.broadcast(t, src=src, group=group, async_op=True)
                work.wait()  # the side stream waits for NCCL's stream
            ev = torch.cuda.Event()
            ev.record(side)
            events.append(ev)
    for t in parts:  # the parts are used on the current stream: keep the allocator honest
        t.record_stream(side)
    return parts, events


def all_gather_rows(block: torch.Tensor, m: int, group=None, align: int = ROW_ALIGN) -> torch.Tensor:
    """Reassemble [e, m, words] from per-rank row blocks (verification only)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return block
    parts = row_partition(m, world, align)
    maxrows = max(r for _, r in parts)
    e, _, nw = block.shape
    padded = torch.zeros((e, maxrows, nw), dtype=block.dtype, device=block.device)
    padded[:, : block.shape[1]] = block
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([b[:, :r] for b, (_, r) in zip(bufs, parts)], dim=1)


def mul_parts(e: int, f: int, A: torch.Tensor, parts: list[torch.Tensor], events, bounds: list[int], k: int,
              n: int, C: torch.Tensor, accumulate: bool = False, backend: str | None = None) -> torch.Tensor:
    """C (^)= A . B with B given as column parts (gf2e_slice_mul_parts), each gated by its
    event.  A [e, m, words(k)], C [e, m, words(n)] contiguous."""
    from . import _device, _lib
    from .poly_mul import _resolve_backend

    m = A.shape[1]
    flags = _resolve_backend(backend) | (_lib.ACCUMULATE if accumulate else 0)
    L = _lib.load()
    ws_bytes = int(L.gf2e_slice_mul_workspace(e, f, m, k, n, flags))
    if ws_bytes < 0:
        _lib.check(_lib.GF2E_EINVAL, "gf2e_slice_mul_workspace")
    ws = _device.workspace.get(ws_bytes)
    np_ = len(parts)
    cb = (ctypes.c_int64 * (np_ + 1))(*bounds)
    bp = (ctypes.c_void_p * np_)(*[t.data_ptr() if t.numel() else None for t in parts])
    ldb = (ctypes.c_int64 * np_)(*[t.shape[2] for t in parts])
    pb = (ctypes.c_int64 * np_)(*[t.shape[1] * t.shape[2] for t in parts])
    evs = (ctypes.c_void_p * np_)(*[ev.cuda_event if ev is not None else None for ev in events])
    lda, ldc = A.shape[2], C.shape[2]
    _lib.call("gf2e_slice_mul_parts", e, f, _device.ptr(A), lda, m * lda, np_, cb, bp, ldb, pb, evs,
              _device.ptr(C), ldc, m * ldc, m, k, n, flags, ws.data_ptr(), ws.numel(), _device.stream_handle())
    return C


def _device_compute(e: int, f: int, A: torch.Tensor, B: torch.Tensor, C0: torch.Tensor | None, k: int, n: int,
                    backend: str | None) -> torch.Tensor:
    from .gf2e import field_new
    from .mat_sliced import SlicedMatrix
    from .poly_mul import addmul, karatsuba_mul

    ctx = field_new(e, f)
    SA = SlicedMatrix(ctx, A.shape[1], k, A)
    SB = SlicedMatrix(ctx, k, n, B)
    if C0 is not None:
        SC = SlicedMatrix(ctx, A.shape[1], n, C0)
        addmul(SC, SA, SB, backend=backend)
        return SC.planes
    return karatsuba_mul(SA, SB, backend=backend).planes


def sharded_mul(e: int, f: int, A_block: torch.Tensor, B: torch.Tensor | None, k: int, n: int, *, C0_block=None,
                src: int = 0, group=None, backend: str | None = None, parts: int = 1,
                compute: Callable | None = None) -> torch.Tensor:
    """This rank's C row-block = A_block . B (^ C0_block), with B broadcast from `src`.

    A_block: [e, rows_g, words(k)] planes of this rank's rows.  B: [e, k, words(n)] planes,
    valid on `src`.  parts == 1: B is broadcast in place (it must exist on every rank) and
    multiplied once.  parts > 1: B travels in column parts on a side stream and the product
    consumes them as they arrive (B may be None off `src`).  Returns [e, rows_g, words(n)]."""
    rank = dist.get_rank(group) if dist.is_initialized() else src
    if (B is not None or rank == src) and B is not None and tuple(B.shape) != (e, k, words_for(n)):
        raise ValueError(f"B planes must have shape {(e, k, words_for(n))}, got {tuple(B.shape)}")
    if A_block.shape[0] != e or A_block.shape[2] != words_for(k):
        raise ValueError("A block planes have the wrong shape")
    if parts <= 1:
        if B is None:
            raise ValueError("B must be allocated on every rank when parts == 1")
        broadcast_planes(B, src=src, group=group)
        fn = compute or (lambda *a: _device_compute(*a, backend))
        return fn(e, f, A_block, B, C0_block, k, n)
    bounds = col_parts(n, parts)
    pieces, events = broadcast_parts(B, (e, k, words_for(n)), bounds, src=src, group=group, device=A_block.device)
    if compute is not None or A_block.device.type != "cuda":
        Bfull = torch.cat(pieces, dim=2) if len(pieces) > 1 else pieces[0]
        fn = compute or (lambda *a: _device_compute(*a, backend))
        return fn(e, f, A_block, Bfull, C0_block, k, n)
    rows = A_block.shape[1]
    if C0_block is not None:
        return mul_parts(e, f, A_block, pieces, events, bounds, k, n, C0_block, True, backend)
    C = torch.empty((e, rows, words_for(n)), dtype=torch.int64, device=A_block.device)
    return mul_parts(e, f, A_block, pieces, events, bounds, k, n, C, False, backend)

"""Multi-GPU partitioning of the hot path: C row-blocks across ranks, B broadcast once.

SURVEY §8e.  Rows of C are independent (C[r, :] = A[r, :] . B (+ C0[r, :])), so rank g owns
rows [row0_g, row0_g + rows_g) of A, C0 and C and needs all of B.  The only collective on the
data path is one broadcast of B's e planes from the source rank (NCCL over NVLink/NVSwitch on
a B200 box; gloo in the CPU tests).  There is no reduction: results stay sharded;
``all_gather_rows`` exists for verification only.

Everything here works on plane tensors ([e, rows, words] int64), device-agnostic, so the same
code runs under NCCL (CUDA tensors) and gloo (CPU tensors).  ``sharded_mul`` computes the local
block with the device kernel (``karatsuba_mul`` / ``addmul``) unless a ``compute`` callable is
injected (the CPU tests inject the oracle — test infrastructure only).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .mat_gf2 import words_for

ROW_ALIGN = 256  # one CTA-pair tile of C rows


def row_partition(m: int, world: int, align: int = ROW_ALIGN) -> list[tuple[int, int]]:
    """(row0, rows) per rank: equal blocks rounded to `align` rows, the remainder on the last
    ranks' blocks trimmed so the union is exactly [0, m)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    per = -(-m // world)
    per = -(-per // align) * align if per else 0
    out = []
    for g in range(world):
        r0 = min(g * per, m)
        r1 = min(r0 + per, m)
        out.append((r0, r1 - r0))
    return out


def broadcast_planes(planes: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of a plane stack from `src` (the one data-path collective)."""
    if dist.is_initialized():
        dist.broadcast(planes, src=src, group=group)
    return planes


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


def sharded_mul(e: int, f: int, A_block: torch.Tensor, B: torch.Tensor, k: int, n: int, *, C0_block=None,
                src: int = 0, group=None, backend: str | None = None,
                compute: Callable | None = None) -> torch.Tensor:
    """This rank's C row-block = A_block . B (^ C0_block), after broadcasting B from `src`.

    A_block: [e, rows_g, words(k)] planes of this rank's rows; B: [e, k, words(n)] planes, valid
    on `src` (overwritten elsewhere by the broadcast).  Returns [e, rows_g, words(n)]."""
    if tuple(B.shape) != (e, k, words_for(n)):
        raise ValueError(f"B planes must have shape {(e, k, words_for(n))}, got {tuple(B.shape)}")
    if A_block.shape[0] != e or A_block.shape[2] != words_for(k):
        raise ValueError("A block planes have the wrong shape")
    broadcast_planes(B, src=src, group=group)
    fn = compute or (lambda *a: _device_compute(*a, backend))
    return fn(e, f, A_block, B, C0_block, k, n)

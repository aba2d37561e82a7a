"""Device plumbing: CUDA device/stream handles and the workspace cache.

PyTorch is used only for device memory and streams; all arithmetic runs in
libgf2e_b200.so.  There is no CPU path: without an sm_100 GPU every call raises.
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch


_CUDA_CHECKED = False


def require_cuda() -> torch.device:
    global _CUDA_CHECKED
    if not _CUDA_CHECKED:  # once per process (the per-call check was a measurable host cost)
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1111_6900_b200 needs a CUDA (sm_100) device; there is no CPU fallback")
        _CUDA_CHECKED = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr() if t.numel() else 0


def empty_words(shape, device=None) -> torch.Tensor:
    return torch.empty(shape, dtype=torch.int64, device=device or require_cuda())


def zeros_words(shape, device=None) -> torch.Tensor:
    return torch.zeros(shape, dtype=torch.int64, device=device or require_cuda())


def to_device_words(arr: np.ndarray, device=None) -> torch.Tensor:
    a = np.ascontiguousarray(arr, dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(device or require_cuda())


def to_host_words(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().cpu().numpy().view(np.uint64)


# scratch requests above this size are not kept between calls (GF2E_WORKSPACE_KEEP bytes)
WORKSPACE_KEEP = int(os.environ.get("GF2E_WORKSPACE_KEEP", str(4 << 30)))


class _Workspace(threading.local):
    """Per-thread, per-(device, stream) scratch buffer, reused across calls up to
    WORKSPACE_KEEP bytes; a larger request gets a one-call tensor (back to PyTorch's caching
    allocator when the call returns), so one huge product does not pin its scratch."""

    def __init__(self):
        self.bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, nbytes: int, stream: int | None = None) -> torch.Tensor:
        dev = require_cuda()
        if nbytes > WORKSPACE_KEEP:
            return torch.empty(nbytes, dtype=torch.uint8, device=dev)
        key = (dev.index, stream_handle() if stream is None else stream)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            self.bufs[key] = buf
        return buf

    def clear(self) -> None:
        self.bufs.clear()


def release_workspace() -> None:
    """Drop the kept scratch buffers of this thread, return PyTorch's cached blocks to the
    driver and trim the library's own pool (gf2e_trim_pool)."""
    workspace.clear()
    if torch.cuda.is_available():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        from . import _lib

        _lib.load().gf2e_trim_pool(0)


workspace = _Workspace()

"""ctypes binding of libgf2e_b200.so (the C ABI declared in include/gf2e_b200.h).

There is no CPU fallback: if the shared library is missing, or there is no sm_100 GPU,
every device entry point raises.  Status codes map to the reference's exception types:
GF2E_EINVAL -> ValueError (poly_mul.py:248-253, gf2e.py:126-137), everything else ->
RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GF2E_LIB_PATH") or os.path.join(_HERE, "libgf2e_b200.so")  # env: dev A/B builds

GF2E_OK, GF2E_EINVAL, GF2E_ECUDA, GF2E_ENOMEM, GF2E_ENODEV, GF2E_ESINGULAR = 0, 1, 2, 3, 4, 5
ACCUMULATE = 1
BACKEND_TC = 0
BACKEND_M4RM = 2
TC_INT8 = 4
TC_FP4 = 8
TC_RUN = 16
B_DEVICE = 32

_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_P = ctypes.c_void_p
_INT = ctypes.c_int
_U32 = ctypes.c_uint32

# name -> (restype, argtypes); mirrors include/gf2e_b200.h one for one
SIGNATURES = {
    "gf2e_last_error": (ctypes.c_char_p, []),
    "gf2e_version": (ctypes.c_char_p, []),
    "gf2e_pack_width": (_INT, [_INT]),
    "gf2e_schedule": (_INT, [_INT, _U32, ctypes.POINTER(_INT), ctypes.POINTER(_U64), ctypes.POINTER(_U64),
                             ctypes.POINTER(_I64)]),
    "gf2e_random_packed": (_INT, [_INT, _I64, _I64, _U64, _I64, _I64, _I64, _P, _I64, _P]),
    "gf2e_random_sliced": (_INT, [_INT, _I64, _I64, _U64, _I64, _I64, _I64, _P, _I64, _I64, _P]),
    "gf2e_random_words": (_INT, [_I64, _I64, _U64, _P, _I64, _P]),
    "gf2e_slice": (_INT, [_INT, _I64, _I64, _P, _I64, _P, _I64, _I64, _P]),
    "gf2e_cling": (_INT, [_INT, _I64, _I64, _P, _I64, _I64, _P, _I64, _P]),
    "gf2e_xor": (_INT, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "gf2e_reduce_mod_f": (_INT, [_INT, _U32, _P, _I64, _I64, _I64, _I64, _P]),
    "gf2e_slice_mul_workspace": (_I64, [_INT, _U32, _I64, _I64, _I64, _U32]),
    "gf2e_plane_mul_workspace": (_I64, [_I64, _I64, _I64, _U32]),
    "gf2e_slice_mul": (_INT, [_INT, _U32, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64,
                              _U32, _P, _I64, _P]),
    "gf2e_nj_mul": (_INT, [_INT, _U32, _P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _U32, _P]),
    "gf2e_run_schedule": (_INT, [_INT, _U32, _P, _P, _P, _P, _P, _P]),
    "gf2e_nj_slice_mul": (_INT, [_INT, _U32, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64,
                                 _U32, _P]),
    "gf2e_slice_mul_parts": (_INT, [_INT, _U32, _P, _I64, _I64, _INT, ctypes.POINTER(_I64), ctypes.POINTER(_P),
                                    ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_P), _P, _I64, _I64,
                                    _I64, _I64, _I64, _U32, _P, _I64, _P]),
    "gf2e_mzed_mul_host": (_INT, [_INT, _U32, _P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _U32, _I64,
                                  ctypes.POINTER(ctypes.c_double)]),
    "gf2e_trsm_workspace": (_I64, [_INT, _U32, _I64, _I64]),
    "gf2e_trsm": (_INT, [_INT, _U32, _INT, _INT, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _P,
                         ctypes.POINTER(_I64)]),
    "gf2e_ple": (_INT, [_INT, _U32, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                        ctypes.POINTER(_I64), _P]),
    "gf2e_echelonize": (_INT, [_INT, _U32, _P, _I64, _I64, _I64, _I64, _INT, ctypes.POINTER(_I64), _P]),
    "gf2e_row_swaps": (_INT, [_INT, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(_I64), _I64, _INT, _P]),
    "gf2e_col_swaps": (_INT, [_INT, _INT, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(_I64), _I64, _P]),
    "gf2e_row_scales": (_INT, [_INT, _U32, _P, _I64, _INT, ctypes.POINTER(_U32), _P, _I64, _I64, _I64, _P]),
    "gf2e_mul_by_x": (_INT, [_INT, _U32, _P, _I64, _I64, _P, _I64, _I64, _I64, _P]),
    "gf2e_scalar_mul": (_INT, [_INT, _U32, _U32, _P, _I64, _P, _I64, _I64, _I64, _P]),
    "gf2e_plane_mul": (_INT, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _U32, _P, _I64, _P]),
    "gf2e_last_launch_count": (_INT, []),
    "gf2e_last_gf2_products": (_I64, []),
    "gf2e_last_product_kernel": (ctypes.c_char_p, []),
    "gf2e_profile_enable": (_INT, [_INT]),
    "gf2e_profile_read": (_INT, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_INT)]),
    "gf2e_dev_fp4_probe": (_INT, [_INT, _INT, _P, _P, _P, ctypes.POINTER(ctypes.c_double), _P]),
    "gf2e_mma_peak": (_INT, [_INT, _INT, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), _P]),
    "gf2e_trim_pool": (_INT, [_I64]),
    "gf2e_tile_cols": (_I64, [_INT, _U32, _I64, _U32]),
    "gf2e_int_peak": (_INT, [_INT, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), _P]),
    "gf2e_fp4_selfcheck": (_INT, [_INT, _INT, ctypes.POINTER(_INT)]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree shared library (built by __graft_entry__.build / csrc/Makefile)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libgf2e_b200.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().gf2e_last_error().decode()


def check(rc: int, what: str) -> None:
    if rc == GF2E_OK:
        return
    msg = last_error()
    if rc == GF2E_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def last_launch_count() -> int:
    return int(load().gf2e_last_launch_count())


def last_gf2_products() -> int:
    """GF(2) plane products the last library call launched (K(e) per fused product launch)."""
    return int(load().gf2e_last_gf2_products())


def profile_enable(on: bool) -> None:
    load().gf2e_profile_enable(1 if on else 0)


def profile_read() -> tuple[float, int]:
    """(summed product-kernel ms, launches) since the last read; synchronises the events."""
    ms = ctypes.c_double()
    n = ctypes.c_int()
    check(load().gf2e_profile_read(ctypes.byref(ms), ctypes.byref(n)), "gf2e_profile_read")
    return ms.value, n.value


def mma_peak(cta_group: int = 1, iters: int = 20000) -> tuple[float, float]:
    """Measured dense kind::i8 tensor rate (TOPS) and launch ms (gf2e_mma_peak)."""
    import torch

    tops = ctypes.c_double()
    ms = ctypes.c_double()
    check(load().gf2e_mma_peak(cta_group, iters, ctypes.byref(tops), ctypes.byref(ms),
                               torch.cuda.current_stream().cuda_stream), "gf2e_mma_peak")
    return tops.value, ms.value


def mma_peak_fp4(iters: int = 20000, operands: str = "zero") -> float:
    """Measured dense kind::mxf4 (block-scaled e2m1) tensor rate in TOPS: pure MMA loop on all
    SMs (gf2e_dev_fp4_probe).  operands="zero": all-zero tiles (burst rate, lowest power);
    "random": random GF(2) bits in the product kernel's e2m1 encoding (A nibbles 0 or
    0.5/1/2/1, B nibbles 0 or 2/1/0.5/1) -- with a long loop this is the sustained rate the
    product kernel can meet under the board power limit."""
    import numpy as np
    import torch

    if operands == "zero":
        a = torch.zeros(128 * 128, dtype=torch.uint8, device="cuda")
        b = torch.zeros(256 * 128, dtype=torch.uint8, device="cuda")
    elif operands == "random":
        rng = np.random.default_rng(7)

        def img(rows, vals):
            bits = rng.integers(0, 2, size=(rows, 32, 4, 2), dtype=np.uint8)  # [row][word][byte][nibble]
            plane = (np.arange(32) % 4)[None, :, None, None]
            v = np.asarray(vals, dtype=np.uint8)[plane] * bits
            return torch.from_numpy((v[..., 0] | (v[..., 1] << 4)).reshape(-1).copy()).cuda()

        a = img(128, [1, 2, 4, 2])
        b = img(256, [4, 2, 1, 2])
    else:
        raise ValueError("operands must be 'zero' or 'random'")
    out = torch.empty(128 * 256, dtype=torch.int32, device="cuda")
    tops = ctypes.c_double()
    check(load().gf2e_dev_fp4_probe(iters, 0, a.data_ptr(), b.data_ptr(), out.data_ptr(), ctypes.byref(tops),
                                    torch.cuda.current_stream().cuda_stream), "gf2e_dev_fp4_probe")
    return tops.value


def fp4_selfcheck(rerun: bool = False, inject_fault: bool = False) -> int:
    """Run (once per device, or again with rerun) the fp4 exactness self-check: 1 = the fp4
    forms matched the int8 form bit for bit and stay in use, -1 = mismatch, fp4 disabled."""
    ok = ctypes.c_int()
    check(load().gf2e_fp4_selfcheck(1 if rerun else 0, 1 if inject_fault else 0, ctypes.byref(ok)),
          "gf2e_fp4_selfcheck")
    return ok.value


def int_peak(iters: int = 2000) -> tuple[float, float]:
    """(LDS.128 bytes/s of the whole GPU, the M4RM form's GF(2) Tbit-op/s bound) measured live."""
    import torch

    bps = ctypes.c_double()
    tops = ctypes.c_double()
    check(load().gf2e_int_peak(iters, ctypes.byref(bps), ctypes.byref(tops),
                               torch.cuda.current_stream().cuda_stream), "gf2e_int_peak")
    return bps.value, tops.value


def run_schedule(e: int, f: int) -> tuple[list[int], list[int], list[int], int]:
    """The running-sum form's drain grouping: (seq, gsize, gmask, run_load)."""
    n, g, load_ = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    seq, gsize, gmask = (ctypes.c_int * 128)(), (ctypes.c_int * 128)(), (ctypes.c_uint32 * 128)()
    check(load().gf2e_run_schedule(e, f, ctypes.byref(n), ctypes.byref(g), ctypes.byref(load_), seq, gsize, gmask),
          "gf2e_run_schedule")
    return list(seq[:n.value]), list(gsize[:g.value]), list(gmask[:g.value]), load_.value


def last_product_kernel() -> str:
    return load().gf2e_last_product_kernel().decode()

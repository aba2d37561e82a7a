"""Probe of the block-scaled FP4 tensor path for GF(2) products (dev tool).

Checks exactness of fp32 accumulation of 0/1 e2m1 products and the mxf4 rate."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1111_6900_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
L = _lib.load()


def run(a, b, iters, mode=0):
    da = torch.from_numpy(a.copy()).cuda()
    db = torch.from_numpy(b.copy()).cuda()
    out = torch.zeros((128, 256), dtype=torch.int32, device="cuda")
    tops = ctypes.c_double()
    _lib.check(L.gf2e_dev_fp4_probe(iters, mode, da.data_ptr(), db.data_ptr(), out.data_ptr(), ctypes.byref(tops),
                                    torch.cuda.current_stream().cuda_stream), "probe")
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32), tops.value


def expect(a, b):
    # element k of a row: byte k//2, low nibble first (order is irrelevant: A and B share it)
    def vals(x):
        lo, hi = x & 0xF, x >> 4
        v = np.stack([lo, hi], axis=-1).reshape(x.shape[0], -1)
        return (v == 2).astype(np.int64)  # only codes 0 and 2 (1.0) are used
    return vals(a) @ vals(b).T


rng = np.random.default_rng(0)
ones_a = np.full((128, 128), 0x22, np.uint8)
ones_b = np.full((256, 128), 0x22, np.uint8)
for iters in (1, 16, 256, 4096, 65536):
    out, tops = run(ones_a, ones_b, iters)
    f = out.view(np.float32)
    want = 256.0 * iters
    print(f"all-ones iters={iters:6d} count={int(want):9d}  exact={bool(np.all(f == want))}  "
          f"sample={f[0,0]}  TOPS={tops:.0f}")
for iters in (1, 7, 100, 255):
    out, _ = run(ones_a, ones_b, iters, mode=1)
    want = np.uint32(0x47800000 + (256 * iters << 7)) if 256 * iters < 65536 else None
    print(f"init65536 iters={iters:4d} bit7-parity ok={want is None or bool(np.all(out == want))} word={hex(out[0,0])}")
for trial in range(3):
    bits_a = rng.integers(0, 2, size=(128, 256))
    bits_b = rng.integers(0, 2, size=(256, 256))
    pack = lambda bits: ((bits[:, 0::2] * 2) | ((bits[:, 1::2] * 2) << 4)).astype(np.uint8)
    a, b = pack(bits_a), pack(bits_b)
    iters = [1, 33, 250][trial]
    out, _ = run(a, b, iters)
    exp = expect(a, b) * iters
    got = out.view(np.float32)
    print(f"random trial {trial} iters={iters}: exact={bool(np.all(got == exp))} max={exp.max()}")
    out, _ = run(a, b, iters, mode=1)
    par = (out >> 7) & 1
    print(f"   init65536 parity-at-bit-7 ok={bool(np.all(par == (exp & 1)))}")

"""Dev tool: per-role wait-cycle counters of the product kernel (library built with
-DGF2E_INSTR=1, loaded through GF2E_LIB_PATH).  python tools/instr.py e m k n"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import _lib  # noqa: E402

e, m, k, n = (int(x) for x in sys.argv[1:5])
ctx = g.field_new(e)
A = g.SlicedMatrix.random(ctx, m, k, 1)
B = g.SlicedMatrix.random(ctx, k, n, 2)
for _ in range(2):
    g.karatsuba_mul(A, B)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (1024 * 16))()
assert lib.gf2e_debug_instr(buf, 1024) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.float64)
nb = int((a[:, 2] > 0).sum())
a = a[:nb]
names = ["exp_empty", "exp_bfull", "exp_total", "epi_tfull", "epi_total", "mma_full", "mma_tempty", "mma_total"]
for i, nm in enumerate(names):
    col = a[:, i] if "mma" not in nm else a[0::2, i]  # MMA issuer only on the leader CTA
    print(f"{nm:12s} mean {col.mean():14.0f} cycles  ({100 * col.mean() / a[:, 2].mean():5.1f}% of expander total)")
ns = a[0::2, 8].mean()
ops = g.count_products(e) * m * n * k * 2.0 / (2 * (m // 256) * (n // 256) / nb) if False else None
cyc = a[0::2, 7].mean()
ideal = g.count_products(e) * (m // 256) * (n // 256) / (nb // 2) * (k // 256) * 512  # 4 x 128-cycle MMAs per stage
print(f"per-cycle MMA efficiency (ideal {ideal:.0f} / MMA-thread cycles): {ideal / cyc:.3f}")
print(f"effective SM clock (MMA thread cycles / globaltimer): {a[0::2, 7].mean() / ns:.3f} GHz over {ns / 1e6:.2f} ms")

"""Dev tool: per-role wait / work cycle counters of k_product_run (library variant built with
tools/build_variant.sh NAME -DGF2E_INSTR=1 product_run.cu, loaded through GF2E_LIB_PATH).
    GF2E_LIB_PATH=build/variants/lib_NAME.so python tools/instr_run.py e m k n [--acc]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import _lib  # noqa: E402

e, m, k, n = (int(x) for x in sys.argv[1:5])
acc = "--acc" in sys.argv
ctx = g.field_new(e)
A = g.SlicedMatrix.random(ctx, m, k, 1)
B = g.SlicedMatrix.random(ctx, k, n, 2)
C = g.SlicedMatrix.random(ctx, m, n, 3)
for _ in range(2):
    if acc:
        g.addmul(C, A, B, backend="tc_run")
    else:
        g.karatsuba_mul(A, B, backend="tc_run")
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (1024 * 32))()
assert lib.gf2e_debug_instr_run(buf, 1024) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 32).astype(np.float64)
nb = int((a[:, 3] > 0).sum())
a = a[:nb]
tot = a[:, 3].mean()
names = {0: "exp wait empty", 1: "exp wait bfull", 2: "exp work (expand+wait_st)", 3: "exp total",
         4: "epi wait tfull", 5: "epi drain (ld..arrive)", 6: "epi C store", 7: "epi total",
         8: "mma wait full", 9: "mma wait tempty", 10: "mma total",
         12: "  exp: A expand + STTM issue", 13: "  exp: B expand + STS", 14: "  exp: wait::st + fences",
         16: "  epi: ld 0,1 + wait::ld", 17: "  epi: fold 0,1 + ld 2", 18: "  epi: wait::ld 2",
         19: "  epi: init/fence/arrive", 20: "  epi: fold 2"}
for i, nm in names.items():
    col = a[0::2, i] if 8 <= i <= 11 else a[:, i]
    print(f"{nm:28s} {col.mean():14.0f} cycles  {100 * col.mean() / tot:5.1f}%")
K = len(_lib.run_schedule(e, ctx.f)[0])  # entries (MMA products) per tile of the grouped sequence
if os.environ.get("GF2E_RUN_DRAINS") and int(os.environ["GF2E_RUN_DRAINS"]) >= g.count_products(e):
    K = g.count_products(e)
tiles = (-(-m // 256)) * (-(-n // 192))
per_pair = tiles / (nb // 2) * K
print(f"entries per CTA pair {per_pair:.0f}; cycles per entry (MMA thread): {a[0::2, 10].mean() / per_pair:.0f}; "
      f"SM clock {a[0::2, 10].mean() / a[0::2, 11].mean():.3f} GHz over {a[0::2, 11].mean() / 1e6:.2f} ms")

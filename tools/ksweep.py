"""Product-kernel time vs k (int8 form) at m = n = 16384, e = 8: per-product overhead."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import _lib  # noqa: E402

ctx = g.field_new(int(os.environ.get("E", "8")))
m = n = 16384
backend = os.environ.get("BACKEND", "tc_i8")
for k in (128, 256, 512, 1024, 2048, 4096):
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    C = g.SlicedMatrix.random(ctx, m, n, 3)
    for _ in range(2):
        g.addmul(C, A, B, backend=backend)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    _lib.profile_read()
    for _ in range(5):
        g.addmul(C, A, B, backend=backend)
    torch.cuda.synchronize()
    ms, cnt = _lib.profile_read()
    _lib.profile_enable(False)
    per = ms / cnt
    K = g.count_products(ctx.e)
    tiles = (m // 256) * (n // 256)
    prods_per_pair = K * tiles / 74
    cyc = per * 1e-3 * 1.842e9 / prods_per_pair
    ideal = 1024 * k / 256
    print(f"k={k:5d} [{_lib.last_product_kernel()}]: {per:8.3f} ms, {cyc:7.0f} cycles/product (ideal {ideal:.0f}), "
          f"overhead {cyc - ideal:6.0f}", flush=True)
    del A, B, C

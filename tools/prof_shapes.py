"""Product-kernel time per launch for a few shapes (e=8): python tools/prof_shapes.py m,k,n ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import _lib  # noqa: E402

ctx = g.field_new(8)
for spec in sys.argv[1:]:
    m, k, n = (int(x) for x in spec.split(","))
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    for _ in range(3):
        g.karatsuba_mul(A, B)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    reps = 10
    for _ in range(reps):
        g.karatsuba_mul(A, B)
    torch.cuda.synchronize()
    ms, cnt = _lib.profile_read()
    _lib.profile_enable(False)
    per = ms / max(cnt, 1)
    ops = 27 * 2 * m * k * n
    print(f"{m}x{k}x{n}: product {per:.4f} ms/launch ({cnt} launches) {ops / per / 1e9:.0f} Tbit-op/s "
          f"[{_lib.last_product_kernel()}]", flush=True)
    del A, B

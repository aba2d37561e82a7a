"""Dev: device time of one karatsuba_mul per tensor-core form at mid-size k (where the
default switches from the running-sum form to the single-accumulator fp4 form).
    python tools/form_cross.py E M N k1,k2,..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e, m, n = (int(x) for x in sys.argv[1:4])
ks = [int(x) for x in sys.argv[4].split(",")]
ctx = g.field_new(e)
for k in ks:
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    res = {}
    for be in ("tc", "tc_run", "tc_fp4"):
        for _ in range(3):
            C = g.karatsuba_mul(A, B, backend=be)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(10):
            C = g.karatsuba_mul(A, B, backend=be)
        ev1.record()
        torch.cuda.synchronize()
        res[be] = (ev0.elapsed_time(ev1) / 10, g._lib.last_product_kernel())
    print(f"e={e} {m}x{k}x{n}: " + "  ".join(f"{b} {t:.3f} ms ({kn})" for b, (t, kn) in res.items()), flush=True)

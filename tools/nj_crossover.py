"""Small-product crossover: the one-launch packed Newton-John kernel
(gf2e_nj_mul) against the sliced tensor-core path (slice A, slice B, combos, product, cling)
for square s x s x s packed products, every e.  Device time per call by CUDA events over many
back-to-back calls.   python tools/nj_crossover.py > profiles/r02/nj_crossover.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import poly_mul  # noqa: E402

torch.cuda.set_device(0)


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


for e in range(2, 11):
    ctx = g.field_new(e)
    for s in (8, 16, 32, 64, 96, 128, 256, 512):
        if not poly_mul.nj_fits(e, s):
            continue
        A = g.PackedMatrix.random(ctx, s, s, 1)
        B = g.PackedMatrix.random(ctx, s, s, 2)
        assert poly_mul.nj_mul_packed(A, B) == g.karatsuba_mul_packed(A, B, backend="tc")
        t_nj = timed(lambda: poly_mul.nj_mul_packed(A, B))
        t_sl = timed(lambda: g.karatsuba_mul_packed(A, B, backend="tc"))
        print(json.dumps({"e": e, "size": s, "nj_us": round(t_nj, 2), "sliced_us": round(t_sl, 2),
                          "winner": "nj" if t_nj < t_sl else "sliced"}), flush=True)

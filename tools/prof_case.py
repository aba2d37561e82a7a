"""Run one karatsuba_mul / addmul shape a few times (for ncu / compute-sanitizer captures).

    python tools/prof_case.py E M K N [--acc] [--reps R] [--backend tc|m4rm]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("e", type=int)
ap.add_argument("m", type=int)
ap.add_argument("k", type=int)
ap.add_argument("n", type=int)
ap.add_argument("--acc", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--backend", default=None)
a = ap.parse_args()
ctx = g.field_new(a.e)
A = g.SlicedMatrix.random(ctx, a.m, a.k, 1)
B = g.SlicedMatrix.random(ctx, a.k, a.n, 2)
C = g.SlicedMatrix.random(ctx, a.m, a.n, 3)
for _ in range(a.reps):
    if a.acc:
        g.addmul(C, A, B, backend=a.backend)
    else:
        g.karatsuba_mul(A, B, backend=a.backend)
torch.cuda.synchronize()
print("ok", g._lib.last_product_kernel())

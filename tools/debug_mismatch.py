"""Compare karatsuba_mul on GPU with the oracle and report mismatching 256x256 tiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1111_6900_b200 as g  # noqa: E402

e, m, k, n = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
ctx = g.field_new(e)
A = g.SlicedMatrix.random(ctx, m, k, 1)
B = g.SlicedMatrix.random(ctx, k, n, 2)
ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2), m, k, n)
for r in range(reps):
    C = g.karatsuba_mul(A, B).to_numpy()
    bad = C != ref  # [e, m, nw]
    if not bad.any():
        print(f"rep {r}: OK")
        continue
    planes, rows, words = np.nonzero(bad)
    tiles = sorted(set(zip((rows // 256).tolist(), (words // 4).tolist())))
    print(f"rep {r}: {bad.sum()} bad words, planes {sorted(set(planes.tolist()))}, "
          f"{len(tiles)} bad tiles of {((m + 255) // 256) * ((n + 255) // 256)}: {tiles[:20]}")
    rr = rows - (rows // 256) * 256
    print("   row-in-tile histogram (CTA half 0/1):", np.bincount(rr // 128, minlength=2).tolist(),
          " word-in-tile:", np.bincount(words % 4, minlength=4).tolist())

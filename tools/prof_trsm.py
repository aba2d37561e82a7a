"""Dev: one upper TRSM m x m \\ m x n (sliced) for launch-list profiling.  python tools/prof_trsm.py e m n"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e, m, n = (int(x) for x in sys.argv[1:4])
ctx = g.field_new(e)
R = g.PackedMatrix.random(ctx, m, m, 7).to_array()
up = np.triu(R, 1)
np.fill_diagonal(up, (np.arange(m) % (ctx.order - 1)) + 1)
Us = g.slice_packed(g.PackedMatrix.from_array(ctx, up))
B0 = g.SlicedMatrix.random(ctx, m, n, 8)
X = B0.copy()
g.trsm_sliced(Us, X, upper=True)
for _ in range(3):
    X.planes.copy_(B0.planes)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.trsm_sliced(Us, X, upper=True)
    torch.cuda.synchronize()
    print(f"trsm e={e} {m}x{m} \\\\ {m}x{n}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)

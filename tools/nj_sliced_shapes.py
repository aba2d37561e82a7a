"""Dev: the sliced Newton-John product (gf2e_nj_slice_mul) against the tensor-core addmul at the
shapes of PLE's / TRSM's updates; device time per call from a launch list (run under ncu), or
events over many calls.  python tools/nj_sliced_shapes.py e"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402
from paper_1111_6900_b200 import poly_mul  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = g.field_new(e)
shapes = [(8128, 64, 64), (4000, 64, 64), (500, 64, 64), (8064, 128, 128), (2000, 128, 128), (128, 128, 8064),
          (128, 128, 2048), (128, 64, 4096), (7936, 256, 256), (256, 256, 4096)]
reps = int(os.environ.get("REPS", "50"))
for (m, k, n) in shapes:
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    C = g.SlicedMatrix.random(ctx, m, n, 3)
    res = {}
    for name, fn in (("nj", lambda: poly_mul.nj_mul_sliced(A, B, C)), ("tc", lambda: g.addmul(C, A, B))):
        fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        # events around a burst: host-bound for small shapes, so also report the graph-free
        # per-call time from the launch list when run under ncu
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) * 1e3 / reps
    print(f"e={e} m={m} k={k} n={n}: nj {res['nj']:.1f} us, tc {res['tc']:.1f} us (event bursts)", flush=True)

"""Dev: device time of small sliced products C ^= A * B (m x k x n) through gf2e_slice_mul, the
shapes PLE's recursion and TRSM issue.  python tools/small_products.py e"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = g.field_new(e)
for (m, k, n) in [(8128, 64, 64), (4096, 64, 64), (1024, 64, 64), (8064, 128, 128), (2048, 128, 128),
                  (7936, 256, 256), (7680, 512, 512), (7168, 1024, 1024), (6144, 2048, 2048), (4096, 4096, 4096),
                  (128, 128, 4096), (128, 128, 8064)]:
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    C = g.SlicedMatrix.random(ctx, m, n, 3)
    for _ in range(3):
        g.addmul(C, A, B)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    ev0.record()
    for _ in range(reps):
        g.addmul(C, A, B)
    ev1.record()
    torch.cuda.synchronize()
    print(f"e={e} m={m} k={k} n={n}: {1e3 * ev0.elapsed_time(ev1) / reps:.1f} us", flush=True)

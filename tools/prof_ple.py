"""Dev: one PLE of n x n (sliced) for launch-list profiling.  python tools/prof_ple.py e n"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e, n = int(sys.argv[1]), int(sys.argv[2])
ctx = g.field_new(e)
S0 = g.slice_packed(g.PackedMatrix.random(ctx, n, n, 11))
S = S0.copy()
g.ple_sliced(S)
torch.cuda.synchronize()
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for _ in range(reps):
    S.planes.copy_(S0.planes)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    P, Q, r = g.ple_sliced(S)
    ev1.record()
    torch.cuda.synchronize()
    print(f"ple e={e} n={n}: {1e3 * (time.perf_counter() - t0):.2f} ms wall, {ev0.elapsed_time(ev1):.2f} ms "
          f"default-stream events, rank {r}", flush=True)

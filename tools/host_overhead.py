"""Dev: host-side cost per call of karatsuba_mul at small sizes (BASELINE config 1), and a
cProfile of the Python path.  python tools/host_overhead.py [e m k n]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e, m, k, n = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (2, 1024, 1024, 1024)
ctx = g.field_new(e)
A = g.SlicedMatrix.random(ctx, m, k, 1)
B = g.SlicedMatrix.random(ctx, k, n, 2)
for _ in range(20):
    g.karatsuba_mul(A, B)
torch.cuda.synchronize()
N = 300
t0 = time.perf_counter()
for _ in range(N):
    g.karatsuba_mul(A, B)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / N:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / N:.1f} us/call")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# device time per call when the host is not the bottleneck: a CUDA graph is not used by the
# library; instead time a burst after pre-enqueueing (device runs behind the host)
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    g.karatsuba_mul(A, B)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

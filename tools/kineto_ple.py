"""Dev: real (not ncu-serialised) kernel times and device idle of one PLE (or echelonize with
--ech), from torch.profiler (CUPTI activity records).  python tools/kineto_ple.py e n [--ech]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402

e, n = int(sys.argv[1]), int(sys.argv[2])
ctx = g.field_new(e)
S0 = g.slice_packed(g.PackedMatrix.random(ctx, n, n, 11))
S = S0.copy()
op = (lambda X: g.echelonize_sliced(X, True)) if "--ech" in sys.argv else g.ple_sliced
op(S)
torch.cuda.synchronize()
S.planes.copy_(S0.planes)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    op(S)
    torch.cuda.synchronize()
evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
kern = [(ev.time_range.start, ev.time_range.end, ev.name) for ev in evs]
kern.sort()
t0, t1 = kern[0][0], max(k[1] for k in kern)
busy, last = 0.0, t0
for s, t, _ in kern:  # union of intervals (streams may overlap)
    if t > last:
        busy += t - max(s, last)
        last = t
tot = collections.defaultdict(lambda: [0, 0.0])
for s, t, name in kern:
    short = name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    tot[short][0] += 1
    tot[short][1] += t - s
print(f"span {(t1 - t0) / 1e3:.2f} ms, device busy {busy / 1e3:.2f} ms, idle {(t1 - t0 - busy) / 1e3:.2f} ms, "
      f"{len(kern)} records")
for name, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{name[:60]:60s} {c:6d} {us / 1e3:9.2f} ms {us / c:8.1f} us")

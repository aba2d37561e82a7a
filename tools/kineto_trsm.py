"""Dev: CUPTI kernel times of one upper TRSM m x m \\ m x n (sliced).  python tools/kineto_trsm.py e m n"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

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
torch.cuda.synchronize()
X.planes.copy_(B0.planes)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    g.trsm_sliced(Us, X, upper=True)
    torch.cuda.synchronize()
kern = sorted((ev.time_range.start, ev.time_range.end, ev.name) for ev in prof.events()
              if ev.device_type == torch.autograd.DeviceType.CUDA)
t0, t1 = kern[0][0], max(k[1] for k in kern)
tot = collections.defaultdict(lambda: [0, 0.0])
for s, t, name in kern:
    short = name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    tot[short][0] += 1
    tot[short][1] += t - s
print(f"span {(t1 - t0) / 1e3:.2f} ms, {len(kern)} records")
for name, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{name[:60]:60s} {c:6d} {us / 1e3:9.2f} ms {us / c:8.1f} us")

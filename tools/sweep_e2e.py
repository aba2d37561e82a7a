"""Sweep the host-buffer pipeline's row chunking at BASELINE config 3 (e2e leg of bench.py):
python tools/sweep_e2e.py first,last,chunk ...  (0 = library default)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6900_b200 as g  # noqa: E402

e, m, k, n = 8, 16384, 16384, 16384
ctx = g.field_new(e)
A = g.PackedMatrix.random(ctx, m, k, 1)
B = g.PackedMatrix.random(ctx, k, n, 2)
hA = torch.empty(tuple(A.storage.words.shape), dtype=torch.int64, pin_memory=True)
hB = torch.empty(tuple(B.storage.words.shape), dtype=torch.int64, pin_memory=True)
hA.copy_(A.storage.words)
hB.copy_(B.storage.words)
hC = torch.empty_like(hA, pin_memory=True)
del A, B
torch.cuda.synchronize()
nA, nB, nC = (t.numpy().view(np.uint64) for t in (hA, hB, hC))
for spec in sys.argv[1:] or ["0,0,0"]:
    first, last, chunk = (int(x) for x in spec.split(","))
    for key, v in (("GF2E_E2E_FIRST", first), ("GF2E_E2E_LAST", last)):
        if v:
            os.environ[key] = str(v)
        else:
            os.environ.pop(key, None)
    ms = [g.karatsuba_mul_packed_host(ctx, nA, k, nB, n, out=nC, chunk_rows=chunk)[1] for _ in range(6)][2:]
    print(f"first={first} last={last} chunk={chunk}: e2e ms median {sorted(ms)[len(ms) // 2]:.2f} "
          f"min {min(ms):.2f} -> {[round(x, 2) for x in ms]}", flush=True)

"""Host-buffer pipeline timing for one shape: python tools/trace_e2e.py e m k n acc [chunk_rows]
(GF2E_E2E_TRACE=1 adds per-stage completion times on stderr)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6900_b200 as g  # noqa: E402

e, m, k, n, acc = (int(x) for x in sys.argv[1:6])
chunk = int(sys.argv[6]) if len(sys.argv) > 6 else 0
ctx = g.field_new(e)
A = g.PackedMatrix.random(ctx, m, k, 1)
B = g.PackedMatrix.random(ctx, k, n, 2)
hA = torch.empty(tuple(A.storage.words.shape), dtype=torch.int64, pin_memory=True)
hB = torch.empty(tuple(B.storage.words.shape), dtype=torch.int64, pin_memory=True)
hA.copy_(A.storage.words)
hB.copy_(B.storage.words)
wpc = g.words_for(n * g.pack_width(e))
hC = torch.zeros((m, wpc), dtype=torch.int64, pin_memory=True)
del A, B
torch.cuda.synchronize()
nA, nB, nC = (t.numpy().view(np.uint64) for t in (hA, hB, hC))
ms = []
for _ in range(4):
    if acc:
        ms.append(g.karatsuba_mul_packed_host(ctx, nA, k, nB, n, C_words=nC, chunk_rows=chunk)[1])
    else:
        ms.append(g.karatsuba_mul_packed_host(ctx, nA, k, nB, n, out=nC, chunk_rows=chunk)[1])
print(f"e={e} {m}x{k}x{n} acc={acc} chunk={chunk}: e2e ms {[round(x, 2) for x in ms]}", flush=True)

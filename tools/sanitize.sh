#!/bin/bash
# compute-sanitizer (one tool per invocation) on small shapes of every kernel path.
tool=${1:-memcheck}
exec compute-sanitizer --tool $tool --error-exitcode 9 python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1111_6900_b200 as g, oracle
for e, m, k, n in [(2, 300, 130, 257), (8, 260, 300, 70), (10, 129, 65, 513)]:
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, k, 1); B = g.PackedMatrix.random(ctx, k, n, 2)
    for backend in ("tc", "m4rm"):
        C = g.karatsuba_mul_packed(A, B, backend=backend)
        C0 = g.PackedMatrix.random(ctx, m, n, 3); g.addmul_packed(C0, A, B, backend=backend)
    Ch, _ = g.karatsuba_mul_packed_host(ctx, A.to_numpy(), k, B.to_numpy(), n, chunk_rows=256)
    ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2), m, k, n)
    assert np.array_equal(C.to_numpy(), oracle.cling_words(e, m, n, ref))
    assert np.array_equal(Ch, oracle.cling_words(e, m, n, ref))
g.reduce_mod_f([g.BitMatrix.random(5, 70, i) for i in range(7)], g.field_new(4))
torch.cuda.synchronize()
print("sanitize run ok")
PY

"""Dev: larger randomized PLE / echelonize / TRSM checks against the oracle (ragged shapes up to
~3000, all e, full / low rank / zero bands).  python tools/ple_stress.py SEEDS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1111_6900_b200 as g  # noqa: E402

nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad = 0
for seed in range(nseeds):
    rng = np.random.default_rng(9000 + seed)
    e = int(rng.integers(2, 11))
    m, n = (int(x) for x in rng.integers(100, 3000, size=2))
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, n, 300 + seed)
    arr = A.to_array()
    kind = seed % 3
    if kind == 1:  # low rank: product of thin factors through the device product
        r0 = int(rng.integers(1, min(m, n)))
        X = g.PackedMatrix.random(ctx, m, r0, 11 + seed)
        Y = g.PackedMatrix.random(ctx, r0, n, 12 + seed)
        A = g.karatsuba_mul_packed(X, Y)
        arr = A.to_array()
    elif kind == 2 and n > 70:
        c0 = int(rng.integers(0, n - 64))
        arr[:, c0:c0 + int(rng.integers(1, 64))] = 0
        A = g.PackedMatrix.from_array(ctx, arr)
    ref, P, Q, r = oracle.ple(e, ctx.f, arr)
    F = g.ple(A.copy())
    ok = F.rank == r and np.array_equal(F.P.entries, P) and np.array_equal(F.Q.entries, Q) and \
        np.array_equal(F.matrix.to_array(), ref)
    E1 = A.copy()
    rk = g.echelonize(E1, full=True)
    ok2 = rk == r and g.ple_reconstruct(F) == A
    print(f"seed {seed}: e={e} {m}x{n} kind={kind} rank={r}: ple {'ok' if ok else 'MISMATCH'}, "
          f"reconstruct/echelon rank {'ok' if ok2 else 'MISMATCH'}", flush=True)
    bad += (not ok) + (not ok2)
print("stress", "ok" if bad == 0 else f"{bad} failures")
sys.exit(1 if bad else 0)

"""Generate tests/golden/golden.npz by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/) and, through it, the CUDA library.  Everything
is produced by the reference's own public functions:
    rng.word_stream                       (rng.py:20-28)
    PackedMatrix.random / storage.words   (mat_packed.py:253-265)
    slice_packed / cling                  (mat_sliced.py:97-106)
    karatsuba_mul + MulCounters           (poly_mul.py:245-259, 32-43)
    karatsuba_mul_packed                  (poly_mul.py:275-278)
    reduce_mod_f                          (poly_mul.py:223-242)
    count_products                        (poly_mul.py:262-272)
    mat_gf2.mul (strategy m4rm / cubic)   (mat_gf2.py:425-455)
    FieldCtx.mul_table                    (gf2e.py:91-106)
Seeds follow SURVEY §8d: A = 1, B = 2, C0 = 3.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from gf2elin import gf2e, mat_gf2, mat_packed, mat_sliced, ple_echelon, poly_mul, rng  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# (m, k, n) shapes: word boundaries 63/64/65/127/128/129, empty dims
SHAPES_ALL_E = [(37, 70, 65), (1, 1, 1)]
SHAPES_EDGE = [(63, 64, 65), (64, 64, 64), (33, 127, 70), (129, 64, 1), (5, 0, 7), (0, 3, 4),
               (65, 129, 128)]
CUSTOM_F = {4: 0b11001, 8: 0x11B, 10: 0b10000001111}  # x^4+x^3+1, AES x^8+x^4+x^3+x+1, x^10+x^3+x^2+x+1


def add_case(store, tag, e, f, m, k, n):
    ctx = gf2e.field_new(e, f)
    A = mat_packed.PackedMatrix.random(ctx, m, k, 1)
    B = mat_packed.PackedMatrix.random(ctx, k, n, 2)
    C0 = mat_packed.PackedMatrix.random(ctx, m, n, 3)
    SA, SB, SC0 = (mat_sliced.slice_packed(X) for X in (A, B, C0))
    cnt = poly_mul.MulCounters()
    SC = poly_mul.karatsuba_mul(SA, SB, cnt)
    PC = poly_mul.karatsuba_mul_packed(A, B)
    assert mat_sliced.cling(SC) == PC
    # addmul, written the way the reference library does it (ple_echelon.py:259 xor_window)
    X = C0.copy()
    X.xor_window(0, 0, PC)
    store[f"{tag}/meta"] = np.array([e, ctx.f, m, k, n], dtype=np.int64)
    store[f"{tag}/A_packed"] = A.storage.words.copy()
    store[f"{tag}/B_packed"] = B.storage.words.copy()
    store[f"{tag}/C0_packed"] = C0.storage.words.copy()
    store[f"{tag}/A_planes"] = np.stack([s.words for s in SA.slices]) if e else None
    store[f"{tag}/B_planes"] = np.stack([s.words for s in SB.slices])
    store[f"{tag}/C0_planes"] = np.stack([s.words for s in SC0.slices])
    store[f"{tag}/C_planes"] = np.stack([s.words for s in SC.slices])
    store[f"{tag}/C_packed"] = PC.storage.words.copy()
    store[f"{tag}/addmul_packed"] = X.storage.words.copy()
    store[f"{tag}/counters"] = np.array([cnt.gf2_matmul_count, cnt.additions, cnt.peak_live_products],
                                        dtype=np.int64)


def main():
    store: dict[str, np.ndarray] = {}
    tags = []
    for e in range(2, 11):
        for (m, k, n) in SHAPES_ALL_E:
            tag = f"kara/e{e}/{m}x{k}x{n}"
            add_case(store, tag, e, None, m, k, n)
            tags.append(tag)
    for e in (2, 8):
        for (m, k, n) in SHAPES_EDGE:
            tag = f"kara/e{e}/{m}x{k}x{n}"
            add_case(store, tag, e, None, m, k, n)
            tags.append(tag)
    for e, f in CUSTOM_F.items():
        tag = f"kara/e{e}f{f:x}/40x33x71"
        add_case(store, tag, e, f, 40, 33, 71)
        tags.append(tag)
    # a medium case for the device tiling (several 128-row / 256-col tiles, ragged edges)
    tag = "kara/e4/300x520x270"
    add_case(store, tag, 4, None, 300, 520, 270)
    tags.append(tag)
    store["kara_tags"] = np.array(tags)

    # count_products (poly_mul.py:262-272)
    store["count_products"] = np.array([poly_mul.count_products(e) for e in range(2, 11)], dtype=np.int64)
    store["default_polys"] = np.array([gf2e.DEFAULT_POLYS[e] for e in range(2, 11)], dtype=np.int64)

    # rng word stream (rng.py:20-28)
    for seed in (0, 1, 2, 3, 2**64 - 1):
        store[f"rng/{seed}"] = rng.word_stream(seed, 16)

    # GF(2) plane products (mat_gf2.py:425-455); k in {0, 1, 255, 256, 257}
    g2 = []
    for (m, k, n) in [(64, 0, 64), (70, 1, 65), (33, 255, 129), (65, 256, 127), (128, 257, 64),
                      (1, 300, 1), (200, 64, 200)]:
        A = mat_gf2.BitMatrix.random(m, k, 11)
        B = mat_gf2.BitMatrix.random(k, n, 12)
        C = mat_gf2.mul(A, B, strategy="m4rm")
        assert C == mat_gf2.mul(A, B, strategy="cubic")
        tag = f"gf2/{m}x{k}x{n}"
        store[f"{tag}/A"] = A.words.copy()
        store[f"{tag}/B"] = B.words.copy()
        store[f"{tag}/C"] = C.words.copy()
        store[f"{tag}/meta"] = np.array([m, k, n], dtype=np.int64)
        g2.append(tag)
    store["gf2_tags"] = np.array(g2)

    # Fig. 1: GF(8) [[5,2],[3,1]]
    ctx8 = gf2e.field_new(3)
    P = mat_packed.PackedMatrix.from_array(ctx8, np.array([[5, 2], [3, 1]]))
    S = mat_sliced.slice_packed(P)
    store["fig1/packed"] = P.storage.words.copy()
    store["fig1/planes"] = np.stack([s.words for s in S.slices])

    # reduce_mod_f GF(4) known answer: (C0, C1, C2) -> (C0^C2, C1^C2)
    ctx4 = gf2e.field_new(2)
    Cs = [mat_gf2.BitMatrix.random(5, 70, 20 + i) for i in range(3)]
    R = poly_mul.reduce_mod_f(Cs, ctx4)
    store["reduce/e2/in"] = np.stack([c.words for c in Cs])
    store["reduce/e2/out"] = np.stack([r.words for r in R])
    ctx8f = gf2e.field_new(8)
    Cs = [mat_gf2.BitMatrix.random(3, 65, 40 + i) for i in range(15)]
    R = poly_mul.reduce_mod_f(Cs, ctx8f)
    store["reduce/e8/in"] = np.stack([c.words for c in Cs])
    store["reduce/e8/out"] = np.stack([r.words for r in R])

    # field tables for e = 2..4 (GF(4) mul(2,2)=3 etc.)
    for e in (2, 3, 4):
        store[f"field/e{e}/mul"] = gf2e.field_new(e).mul_table.copy()

    # triangular solves (ple_echelon.py:138-217): U X = B, L X = B (unit / non-unit)
    tr = []
    for e, m, n, seed in [(2, 70, 130, 5), (8, 300, 90, 6), (5, 257, 64, 7), (10, 130, 300, 8), (3, 1, 5, 9)]:
        ctx = gf2e.field_new(e)
        R = mat_packed.PackedMatrix.random(ctx, m, m, seed).to_array()
        diag = (rng.element_stream(seed + 100, m, e) % (ctx.order - 1)) + 1  # nonzero diagonal
        upper = np.triu(R, 1)
        lower = np.tril(R, -1)
        np.fill_diagonal(upper, diag)
        np.fill_diagonal(lower, diag)
        B = mat_packed.PackedMatrix.random(ctx, m, n, seed + 1)
        U = mat_packed.PackedMatrix.from_array(ctx, upper)
        L = mat_packed.PackedMatrix.from_array(ctx, lower)
        XU, XL, XLu = B.copy(), B.copy(), B.copy()
        ple_echelon.trsm_upper_left(U, XU)
        ple_echelon.trsm_lower_left(L, XL)
        ple_echelon.trsm_lower_left_unit(L, XLu)
        tag = f"trsm/e{e}/{m}x{n}"
        # MulCounters of the three solves at the default crossover and at 16 (ple_echelon.py:130-136)
        cnts = []
        for cx in (None, 16):
            for fn, T in ((ple_echelon.trsm_upper_left, U), (ple_echelon.trsm_lower_left, L),
                          (ple_echelon.trsm_lower_left_unit, L)):
                c = poly_mul.MulCounters()
                fn(T, B.copy(), crossover=cx, counters=c)
                cnts.append([c.gf2_matmul_count, c.additions, c.peak_live_products])
        store[f"{tag}/counters"] = np.array(cnts, dtype=np.int64)
        store[f"{tag}/meta"] = np.array([e, ctx.f, m, n], dtype=np.int64)
        store[f"{tag}/U"] = U.storage.words.copy()
        store[f"{tag}/L"] = L.storage.words.copy()
        store[f"{tag}/B"] = B.storage.words.copy()
        store[f"{tag}/XU"] = XU.storage.words.copy()
        store[f"{tag}/XL"] = XL.storage.words.copy()
        store[f"{tag}/XLu"] = XLu.storage.words.copy()
        tr.append(tag)
    store["trsm_tags"] = np.array(tr)

    # sliced mul_by_x (mat_sliced.py:109-122) and packed scalar_mul (mat_packed.py:192-199)
    sc = []
    for e in range(2, 11):
        ctx = gf2e.field_new(e)
        A = mat_packed.PackedMatrix.random(ctx, 37, 70, 40 + e)
        tag = f"scal/e{e}"
        store[f"{tag}/A"] = A.storage.words.copy()
        store[f"{tag}/xA"] = np.stack([s.words for s in mat_sliced.mul_by_x(mat_sliced.slice_packed(A)).slices])
        cs = [0, 1, 2, ctx.order - 1, (5 * e) % ctx.order]
        store[f"{tag}/c"] = np.array(cs, dtype=np.int64)
        store[f"{tag}/cA"] = np.stack([A.scalar_mul(c).storage.words for c in cs])
        sc.append(tag)
    store["scal_tags"] = np.array(sc)

    # PLE decomposition and echelon forms (ple_echelon.py:240-374): random, low-rank and
    # structured inputs; the reference's result is crossover-independent (checked here)
    pl = []
    # The reference's window paste raises for many unaligned splits (mat_gf2.py:240-251: the
    # shifted buffer is one word short when the window does not spill into an extra word), so
    # shapes are chosen where its recursion survives; failures are reported and skipped.
    for e, m, n, seed, kind in [(8, 150, 256, 11, "rand"), (2, 200, 128, 12, "rand"), (4, 257, 256, 13, "rand"),
                                (8, 300, 256, 14, "lowrank"), (3, 1, 5, 15, "rand"), (5, 5, 1, 16, "rand"),
                                (10, 70, 70, 17, "rand"), (8, 129, 192, 18, "zerocols"), (2, 90, 64, 19, "lowrank"),
                                (8, 64, 128, 20, "dup"), (8, 200, 130, 21, "rand"), (4, 300, 512, 22, "lowrank"),
                                (10, 100, 256, 23, "zerocols"), (6, 100, 96, 24, "rand")]:
        ctx = gf2e.field_new(e)
        if kind == "rand":
            A = mat_packed.PackedMatrix.random(ctx, m, n, seed)
        else:
            if kind == "lowrank":  # rank <= 37: A = X . Y
                X = mat_packed.PackedMatrix.random(ctx, m, 37, seed)
                Y = mat_packed.PackedMatrix.random(ctx, 37, n, seed + 1)
                A = poly_mul.karatsuba_mul_packed(X, Y)
            else:
                arr = mat_packed.PackedMatrix.random(ctx, m, n, seed).to_array()
                if kind == "zerocols":
                    arr[:, 3:70] = 0
                    arr[:, 130:131] = 0
                    arr[:40, 0] = 0
                else:  # duplicated / scaled rows and an all-zero row
                    arr[10:20] = arr[0:10]
                    arr[30] = 0
                    arr[40:50] = (arr[0:10].astype(np.int64) * 0 + arr[50:60]).astype(arr.dtype)
                A = mat_packed.PackedMatrix.from_array(ctx, arr)
        tag = f"ple/e{e}/{m}x{n}/{kind}"
        try:
            F = ple_echelon.ple(A.copy())
            ech = []
            for full in (True, False):
                X = A.copy()
                ech.append((ple_echelon.echelonize(X, full=full), X))
        except ValueError as ex:
            print(f"skip {tag}: reference raised {ex!s:.60}")
            continue
        try:
            F16 = ple_echelon.ple(A.copy(), crossover=16)
            assert F.rank == F16.rank and F.P == F16.P and F.Q == F16.Q and F.matrix == F16.matrix
        except ValueError:
            pass
        store[f"{tag}/meta"] = np.array([e, ctx.f, m, n], dtype=np.int64)
        store[f"{tag}/A"] = A.storage.words.copy()
        store[f"{tag}/ple"] = F.matrix.storage.words.copy()
        store[f"{tag}/P"] = F.P.entries.copy()
        store[f"{tag}/Q"] = F.Q.entries.copy()
        store[f"{tag}/rank"] = np.array([F.rank], dtype=np.int64)
        # MulCounters: ple and echelonize (full, row) at the default crossover and at 16
        cnts = []
        for cx in (None, 16):
            try:
                c = poly_mul.MulCounters()
                ple_echelon.ple(A.copy(), crossover=cx, counters=c)
                row = [c.gf2_matmul_count, c.additions, c.peak_live_products]
                for full in (True, False):
                    c = poly_mul.MulCounters()
                    ple_echelon.echelonize(A.copy(), full=full, crossover=cx, counters=c)
                    row += [c.gf2_matmul_count, c.additions, c.peak_live_products]
            except ValueError:
                row = [-1] * 9  # the reference's recursion raised at this crossover
            cnts.append(row)
        store[f"{tag}/counters"] = np.array(cnts, dtype=np.int64)
        for full, (r, X) in zip((True, False), ech):
            assert r == F.rank
            store[f"{tag}/ech{int(full)}"] = X.storage.words.copy()
        pl.append(tag)
    store["ple_tags"] = np.array(pl)

    # Newton-John table routines (newton_john.py): tables, products, elimination, PLE, TRSM,
    # with the reference's RowOpCounters
    from gf2elin import newton_john, mat_gf2 as mg

    nj = []
    for e, m, k, n, seed in [(3, 40, 33, 70, 31), (8, 65, 64, 129, 32), (10, 20, 17, 9, 33)]:
        ctx = gf2e.field_new(e)
        A = mat_packed.PackedMatrix.random(ctx, m, k, seed)
        B = mat_packed.PackedMatrix.random(ctx, k, n, seed + 1)
        tag = f"nj/e{e}"
        store[f"{tag}/meta"] = np.array([e, ctx.f, m, k, n], dtype=np.int64)
        store[f"{tag}/A"] = A.storage.words.copy()
        store[f"{tag}/B"] = B.storage.words.copy()
        cnt = mg.RowOpCounters()
        store[f"{tag}/table"] = newton_john.make_table(B.copy_window(0, 0, 1, n), cnt).words.copy()
        store[f"{tag}/table_cnt"] = np.array([cnt.scalar_row_muls, cnt.row_adds], dtype=np.int64)
        cnt = mg.RowOpCounters()
        store[f"{tag}/mul"] = newton_john.nj_mul(A, B, cnt).storage.words.copy()
        store[f"{tag}/mul_cnt"] = np.array([cnt.scalar_row_muls, cnt.row_adds], dtype=np.int64)
        store[f"{tag}/cubic"] = newton_john.cubic_mul(A, B).storage.words.copy()
        for full in (True, False):
            X = A.copy()
            cnt = mg.RowOpCounters()
            r = newton_john.nj_gauss(X, full=full, counters=cnt)
            store[f"{tag}/gauss{int(full)}"] = X.storage.words.copy()
            store[f"{tag}/gauss{int(full)}_meta"] = np.array([r, cnt.scalar_row_muls, cnt.row_adds], dtype=np.int64)
        X = A.copy()
        cnt = mg.RowOpCounters()
        P, Q, r = newton_john.nj_ple(X, cnt)
        store[f"{tag}/ple"] = X.storage.words.copy()
        store[f"{tag}/ple_P"] = np.asarray(P, dtype=np.int64)
        store[f"{tag}/ple_Q"] = np.asarray(Q, dtype=np.int64)
        store[f"{tag}/ple_meta"] = np.array([r, cnt.scalar_row_muls, cnt.row_adds], dtype=np.int64)
        R = mat_packed.PackedMatrix.random(ctx, k, k, seed + 2).to_array()
        up = np.triu(R, 1)
        np.fill_diagonal(up, (np.arange(k) % (ctx.order - 1)) + 1)
        U = mat_packed.PackedMatrix.from_array(ctx, up)
        X = B.copy()
        cnt = mg.RowOpCounters()
        newton_john.nj_trsm_upper_left(U, X, cnt)
        store[f"{tag}/U"] = U.storage.words.copy()
        store[f"{tag}/trsm"] = X.storage.words.copy()
        store[f"{tag}/trsm_cnt"] = np.array([cnt.scalar_row_muls, cnt.row_adds], dtype=np.int64)
        nj.append(tag)
    store["nj_tags"] = np.array(nj)

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

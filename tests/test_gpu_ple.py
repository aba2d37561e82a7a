"""SURVEY §8f rank 1 on device: PLE decomposition and echelon forms (ple_echelon.py:240-374)
built on the fused addmul, the device TRSM and the two-phase nj_ple panel kernel.
Bit-exact against fixtures the reference produced (tests/golden/make_golden.py) and, at sizes
the reference cannot reach, against the oracle's restatement of nj_ple (itself pinned to the
same fixtures in test_oracle_golden.py)."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch

    import paper_1111_6900_b200 as g

    torch.cuda.set_device(0)
    return g


def test_ple_golden(g, golden):
    for tag in (str(t) for t in golden["ple_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A"], n)
        F = g.ple(A.copy())
        assert F.rank == int(golden[f"{tag}/rank"][0]), tag
        assert np.array_equal(F.P.entries, golden[f"{tag}/P"]), tag
        assert np.array_equal(F.Q.entries, golden[f"{tag}/Q"]), tag
        assert np.array_equal(F.matrix.to_numpy(), golden[f"{tag}/ple"]), tag
        for full in (True, False):
            X = A.copy()
            assert g.echelonize(X, full=full) == F.rank
            assert np.array_equal(X.to_numpy(), golden[f"{tag}/ech{int(full)}"]), (tag, full)


def _lowrank(g, ctx, m, n, r, seed):
    X = g.PackedMatrix.random(ctx, m, r, seed)
    Y = g.PackedMatrix.random(ctx, r, n, seed + 1)
    return g.karatsuba_mul_packed(X, Y)


@pytest.mark.parametrize("e,m,n,kind", [(8, 1000, 1300, "rand"), (2, 1500, 700, "rand"), (4, 900, 700, "lowrank"),
                                        (10, 2000, 200, "rand"), (6, 600, 900, "zeros"), (8, 700, 64, "lowrank"),
                                        (3, 520, 130, "dup")])
def test_ple_vs_oracle(g, e, m, n, kind):
    ctx = g.field_new(e)
    if kind == "lowrank":
        A = _lowrank(g, ctx, m, n, 45, 30 + e)
    else:
        A = g.PackedMatrix.random(ctx, m, n, 30 + e)
        if kind != "rand":
            arr = A.to_array()
            if kind == "zeros":  # zero column band, zero rows at the top: pivots below the window
                arr[:, 100:400] = 0
                arr[:600, 0] = 0
            else:  # duplicated rows below the 512-row window
                arr[515:519] = arr[0:4]
                arr[:, 7] = 0
            A = g.PackedMatrix.from_array(ctx, arr)
    ref, P, Q, r = oracle.ple(e, ctx.f, A.to_array())
    F = g.ple(A.copy())
    assert F.rank == r
    assert np.array_equal(F.P.entries, P) and np.array_equal(F.Q.entries, Q)
    assert np.array_equal(F.matrix.to_array(), ref)


@pytest.mark.parametrize("seed", range(int(os.environ.get("GF2E_FUZZ_SEEDS", "12"))))
def test_ple_fuzz(g, seed):
    # random field, shape (ragged, word-boundary-crossing), rank profile (full, low rank,
    # zero column bands) against the oracle's nj_ple; reconstruction P L E = A
    rng = np.random.default_rng(5000 + seed)
    e = int(rng.integers(2, 11))
    m, n = (int(x) for x in rng.integers(1, 600, size=2))
    ctx = g.field_new(e)
    kind = seed % 3
    if kind == 1:
        A = _lowrank(g, ctx, m, n, int(rng.integers(1, 1 + min(m, n))), 70 + seed)
    else:
        A = g.PackedMatrix.random(ctx, m, n, 70 + seed)
        if kind == 2 and n > 8:
            arr = A.to_array()
            c0 = int(rng.integers(0, n - 4))
            arr[:, c0:c0 + int(rng.integers(1, n - c0))] = 0
            A = g.PackedMatrix.from_array(ctx, arr)
    ref, P, Q, r = oracle.ple(e, ctx.f, A.to_array())
    F = g.ple(A.copy())
    assert F.rank == r, (e, m, n, kind)
    assert np.array_equal(F.P.entries, P) and np.array_equal(F.Q.entries, Q), (e, m, n, kind)
    assert np.array_equal(F.matrix.to_array(), ref), (e, m, n, kind)
    assert g.ple_reconstruct(F) == A


def test_ple_reconstruct_and_echelon(g):
    ctx = g.field_new(5)
    A = _lowrank(g, ctx, 700, 600, 333, 7)
    F = g.ple(A.copy())
    assert F.rank == 333
    assert g.ple_reconstruct(F) == A
    R = A.copy()
    assert g.echelonize(R, full=True) == 333
    arr = R.to_array()
    assert not arr[333:].any()
    piv = [int(np.nonzero(arr[i])[0][0]) for i in range(333)]
    assert piv == sorted(piv) and np.all(arr[:333, piv] == np.eye(333, dtype=arr.dtype))


def test_perm_helpers(g):
    ctx = g.field_new(4)
    A = g.PackedMatrix.random(ctx, 50, 70, 3)
    S = g.slice_packed(A)
    P = g.PermVector([3, 1, 9, 5, 4])
    B = A.copy()
    g.apply_perm_rows(B, P)
    ref = A.to_array()
    for i, j in enumerate(P.entries):
        ref[[i, j]] = ref[[j, i]]
    assert np.array_equal(B.to_array(), ref)
    g.apply_perm_rows(B, P, forward=False)
    assert B == A
    g.apply_perm_rows(S, P)
    assert np.array_equal(S.to_array(), ref)
    Q = g.PermVector([2, 1, 69])
    C = A.copy()
    g.apply_perm_cols(C, Q)
    refc = A.to_array()
    for i, j in enumerate(Q.entries):
        refc[:, [i, j]] = refc[:, [j, i]]
    assert np.array_equal(C.to_array(), refc)
    g.col_swap(C, 0, 5, row_start=10)
    refc[10:, [0, 5]] = refc[10:, [5, 0]]
    assert np.array_equal(C.to_array(), refc)
    with pytest.raises(ValueError, match="swap target"):
        g.apply_perm_rows(A, [0, 50])
    with pytest.raises(ValueError, match="violates"):
        g.PermVector([1, 0])
    X = g.PackedMatrix.random(ctx, 0, 5, 1)
    F = g.ple(X)
    assert F.rank == 0 and len(F.P) == 0


def test_newton_john_golden(g, golden):
    # newton_john.py API on device: tables, products, elimination, PLE, TRSM, counters
    for tag in (str(t) for t in golden["nj_tags"]):
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A"], k)
        B = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B"], n)
        cnt = g.RowOpCounters()
        row0 = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B"][:1], n)
        T = g.make_table(row0, cnt)
        assert np.array_equal(g._device.to_host_words(T.words), golden[f"{tag}/table"]), tag
        assert [cnt.scalar_row_muls, cnt.row_adds] == golden[f"{tag}/table_cnt"].tolist()
        assert np.array_equal(T.row(3).to_numpy(), golden[f"{tag}/table"][3:4])
        cnt = g.RowOpCounters()
        assert np.array_equal(g.nj_mul(A, B, cnt).to_numpy(), golden[f"{tag}/mul"]), tag
        assert [cnt.scalar_row_muls, cnt.row_adds] == golden[f"{tag}/mul_cnt"].tolist()
        assert np.array_equal(g.cubic_mul(A, B).to_numpy(), golden[f"{tag}/cubic"]), tag
        for full in (True, False):
            X = A.copy()
            cnt = g.RowOpCounters()
            r = g.nj_gauss(X, full=full, counters=cnt)
            assert [r, cnt.scalar_row_muls, cnt.row_adds] == golden[f"{tag}/gauss{int(full)}_meta"].tolist()
            assert np.array_equal(X.to_numpy(), golden[f"{tag}/gauss{int(full)}"]), (tag, full)
        X = A.copy()
        cnt = g.RowOpCounters()
        P, Q, r = g.nj_ple(X, cnt)
        assert [r, cnt.scalar_row_muls, cnt.row_adds] == golden[f"{tag}/ple_meta"].tolist()
        assert np.array_equal(P, golden[f"{tag}/ple_P"]) and np.array_equal(Q, golden[f"{tag}/ple_Q"])
        assert np.array_equal(X.to_numpy(), golden[f"{tag}/ple"]), tag
        U = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/U"], k)
        X = B.copy()
        cnt = g.RowOpCounters()
        g.nj_trsm_upper_left(U, X, cnt)
        assert [cnt.scalar_row_muls, cnt.row_adds] == golden[f"{tag}/trsm_cnt"].tolist()
        assert np.array_equal(X.to_numpy(), golden[f"{tag}/trsm"]), tag
    with pytest.raises(ValueError, match="single row"):
        g.make_table(g.PackedMatrix.random(g.field_new(4), 2, 5, 1))


def test_counters_through_the_api(g, golden):
    # MulCounters passed to trsm_* / ple / echelonize match the reference's own counters
    # (ple_echelon.py:130-136 _dispatch_mul accounting) at the default crossover and at 16;
    # device_products counts the GF(2) products the device actually launched
    for tag in (str(t) for t in golden["trsm_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        U = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/U"], m)
        L = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/L"], m)
        B = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B"], n)
        got = []
        for cx in (None, 16):
            for fn, T in ((g.trsm_upper_left, U), (g.trsm_lower_left, L), (g.trsm_lower_left_unit, L)):
                c = g.MulCounters()
                fn(T, B.copy(), crossover=cx, counters=c)
                got.append([c.gf2_matmul_count, c.additions, c.peak_live_products])
                # (updates and leaves with k <= 128 take the CUDA-core Newton-John form, which runs
                # no GF(2) products; the rest run whole Karatsuba schedules)
                assert c.device_products % g.count_products(e) == 0, tag
        assert got == golden[f"{tag}/counters"].tolist(), tag
    for tag in (str(t) for t in golden["ple_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A"], n)
        for row, cx in zip(golden[f"{tag}/counters"].tolist(), (None, 16)):
            if row[0] < 0:
                continue
            got = []
            c = g.MulCounters()
            g.ple(A.copy(), crossover=cx, counters=c)
            got += [c.gf2_matmul_count, c.additions, c.peak_live_products]
            for full in (True, False):
                c = g.MulCounters()
                g.echelonize(A.copy(), full=full, crossover=cx, counters=c)
                got += [c.gf2_matmul_count, c.additions, c.peak_live_products]
            assert got == row, (tag, cx)


@pytest.mark.parametrize("e,m,n,kind", [(8, 700, 900, "rand"), (2, 1000, 640, "rand"), (4, 513, 300, "lowrank"),
                                        (10, 300, 1300, "rand"), (3, 640, 640, "rand"), (5, 200, 64, "rand")])
def test_ple_speculative_matches_exact(g, e, m, n, kind, monkeypatch):
    # the speculative recursion (full rank at every node, pivots kept on device, one sync) and
    # the host-driven exact recursion give the same factorisation; rank-deficient inputs fall
    # back to the exact path after the rank check
    ctx = g.field_new(e)
    A = _lowrank(g, ctx, m, n, 45, 60 + e) if kind == "lowrank" else g.PackedMatrix.random(ctx, m, n, 60 + e)
    F1 = g.ple(A.copy())
    monkeypatch.setenv("GF2E_PLE_EXACT", "1")
    F2 = g.ple(A.copy())
    assert F1.rank == F2.rank
    assert np.array_equal(F1.P.entries, F2.P.entries) and np.array_equal(F1.Q.entries, F2.Q.entries)
    assert F1.matrix == F2.matrix
    arr = A.to_array()
    Fo = oracle.ple(e, ctx.f, arr)
    assert F1.rank == Fo[3] and np.array_equal(F1.P.entries, Fo[1]) and np.array_equal(F1.Q.entries, Fo[2])
    assert np.array_equal(F1.matrix.to_array(), Fo[0])

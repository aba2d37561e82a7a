"""Parity of the CUDA path (through the C ABI) with the oracle and the reference fixtures.
Bit-exact everywhere: this path is integer/bitwise only."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

BACKENDS = ["tc_i8", "tc_fp4", "tc_run", "m4rm"]


@pytest.fixture(scope="module")
def g():
    import torch

    import paper_1111_6900_b200 as g

    torch.cuda.set_device(0)
    return g


def _tags(golden, key):
    return [str(t) for t in golden[key]]


def _sync():
    import torch

    torch.cuda.synchronize()


# ---- K7 / K1 / K2 ----------------------------------------------------------------------

def test_generators_and_conversions_golden(g, golden):
    for tag in _tags(golden, "kara_tags"):
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        A = g.PackedMatrix.random(ctx, m, k, 1)
        assert np.array_equal(A.to_numpy(), golden[f"{tag}/A_packed"]), tag
        SA = g.slice_packed(A)
        assert np.array_equal(SA.to_numpy(), golden[f"{tag}/A_planes"]), tag
        assert np.array_equal(g.SlicedMatrix.random(ctx, m, k, 1).to_numpy(), golden[f"{tag}/A_planes"]), tag
        assert np.array_equal(g.cling(SA).to_numpy(), golden[f"{tag}/A_packed"]), tag


@pytest.mark.parametrize("e", range(2, 11))
@pytest.mark.parametrize("shape", [(1, 1), (63, 64), (65, 127), (128, 129), (7, 1000), (129, 65)])
def test_slice_cling_roundtrip(g, e, shape):
    m, n = shape
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, n, 5 + e)
    S = g.slice_packed(A)
    ref = oracle.slice_words(e, m, n, oracle.packed_random(e, m, n, 5 + e))
    assert np.array_equal(S.to_numpy(), ref)
    assert g.cling(S) == A


def test_slice_drops_pad_bits(g):
    # mat_packed.py:118-121: only bits 0..e-1 of a slot are read
    ctx = g.field_new(5)
    A = g.PackedMatrix.random(ctx, 9, 33, 1)
    words = A.to_numpy()
    pad = np.full(words.shape, 0xE0E0E0E0E0E0E0E0, dtype=np.uint64)  # bits 5..7 of every 8-bit slot
    pad[:, -1] = np.uint64(0xE0)  # 33 slots: the last word holds one slot
    B = g.PackedMatrix.from_numpy(ctx, words | pad, 33)
    assert g.slice_packed(B) == g.slice_packed(A)


def test_random_words_golden(g, golden):
    for tag in _tags(golden, "gf2_tags"):
        m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        assert np.array_equal(g.BitMatrix.random(m, k, 11).to_numpy(), golden[f"{tag}/A"]), tag


# ---- the hot path ----------------------------------------------------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_karatsuba_golden(g, golden, backend):
    for tag in _tags(golden, "kara_tags"):
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        SA = g.SlicedMatrix.from_numpy(ctx, golden[f"{tag}/A_planes"], k)
        SB = g.SlicedMatrix.from_numpy(ctx, golden[f"{tag}/B_planes"], n)
        cnt = g.MulCounters()
        SC = g.karatsuba_mul(SA, SB, cnt, backend=backend)
        assert np.array_equal(SC.to_numpy(), golden[f"{tag}/C_planes"]), (tag, backend)
        assert [cnt.gf2_matmul_count, cnt.additions, cnt.peak_live_products] == list(golden[f"{tag}/counters"])
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A_packed"], k)
        B = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B_packed"], n)
        assert np.array_equal(g.karatsuba_mul_packed(A, B, backend=backend).to_numpy(),
                              golden[f"{tag}/C_packed"]), (tag, backend)
        C0 = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/C0_packed"], n)
        g.addmul_packed(C0, A, B, backend=backend)
        assert np.array_equal(C0.to_numpy(), golden[f"{tag}/addmul_packed"]), (tag, backend)


@pytest.mark.parametrize("backend", BACKENDS)
def test_gf2_plane_products_golden(g, golden, backend):
    for tag in _tags(golden, "gf2_tags"):
        m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        A = g.BitMatrix.from_numpy(golden[f"{tag}/A"], k)
        B = g.BitMatrix.from_numpy(golden[f"{tag}/B"], n)
        C = g.mul(A, B, backend=backend)
        assert np.array_equal(C.to_numpy(), golden[f"{tag}/C"]), (tag, backend)
        D = g.BitMatrix.random(m, n, 99)
        d0 = D.to_numpy()
        g.gf2_addmul(D, A, B, backend=backend)
        assert np.array_equal(D.to_numpy(), d0 ^ golden[f"{tag}/C"]), (tag, backend)


def test_reduce_mod_f_golden(g, golden):
    for e, key in ((2, "reduce/e2"), (8, "reduce/e8")):
        ctx = g.field_new(e)
        cin = golden[f"{key}/in"]
        n = {2: 70, 8: 65}[e]
        slices = [g.BitMatrix.from_numpy(cin[d], n) for d in range(2 * e - 1)]
        cnt = g.MulCounters()
        out = g.reduce_mod_f(slices, ctx, cnt)
        assert np.array_equal(np.stack([o.to_numpy() for o in out]), golden[f"{key}/out"])
        assert cnt.additions == sum(1 for _ in range(e - 1) for k in range(e) if (ctx.f >> k) & 1)
        with pytest.raises(ValueError, match="coefficient slices"):
            g.reduce_mod_f(slices[:-1], ctx)


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("e", range(2, 11))
def test_word_boundary_shapes(g, e, backend):
    # SPEC.md:146 word boundaries, empty and ragged dimensions, all e
    ctx = g.field_new(e)
    for (m, k, n) in [(63, 65, 129), (64, 64, 64), (129, 1, 257), (5, 0, 7), (0, 3, 4), (3, 4, 0),
                      (130, 300, 70), (1, 129, 1)]:
        SA = g.SlicedMatrix.random(ctx, m, k, 1)
        SB = g.SlicedMatrix.random(ctx, k, n, 2)
        C = g.karatsuba_mul(SA, SB, backend=backend)
        ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2),
                                  m, k, n)
        assert np.array_equal(C.to_numpy(), ref), (m, k, n, backend)


@pytest.mark.parametrize("e", range(2, 11))
def test_long_k_all_e(g, e):
    # k >= 2048 takes the fp4 form with A in TMEM (7 TMEM stages); k = 32768 + 300 crosses
    # the fp4 accumulation-chunk boundary (count < 2^16 per chunk); addmul through the same path
    ctx = g.field_new(e)
    for (m, k, n) in [(300, 2048, 260), (257, 4100, 65), (33, 32768 + 300, 129)]:
        SA = g.SlicedMatrix.random(ctx, m, k, 1)
        SB = g.SlicedMatrix.random(ctx, k, n, 2)
        C0 = g.SlicedMatrix.random(ctx, m, n, 3)
        C = C0.copy()
        g.addmul(C, SA, SB)
        assert g._lib.last_product_kernel() == "k_product_tc2<fp4>"
        ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2),
                                  m, k, n, C0=oracle.sliced_random(e, m, n, 3))
        assert np.array_equal(C.to_numpy(), ref), (e, m, k, n)


@pytest.mark.parametrize("backend", BACKENDS)
def test_errors_match_reference(g, backend):
    A = g.SlicedMatrix.random(g.field_new(4), 5, 6, 1)
    B = g.SlicedMatrix.random(g.field_new(4), 7, 5, 2)
    with pytest.raises(ValueError, match="inner dimensions differ"):
        g.karatsuba_mul(A, B, backend=backend)
    B8 = g.SlicedMatrix.random(g.field_new(8), 6, 5, 2)
    with pytest.raises(ValueError, match="field mismatch"):
        g.karatsuba_mul(A, B8, backend=backend)
    with pytest.raises(ValueError, match="unknown multiplication strategy"):
        g.mul(A.slices[0], g.BitMatrix.random(6, 3, 1), strategy="bogus")


def test_config1_full(g):
    # BASELINE config 1: F_4, 1024^3, bit-exact vs the oracle restatement of the reference
    e, m = 2, 1024
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, m, 1)
    B = g.PackedMatrix.random(ctx, m, m, 2)
    C = g.karatsuba_mul_packed(A, B)
    ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, m, 1), oracle.sliced_random(e, m, m, 2), m, m, m)
    assert np.array_equal(C.to_numpy(), oracle.cling_words(e, m, m, ref))


@pytest.mark.parametrize("backend", BACKENDS)
def test_config2_full(g, backend):
    # BASELINE config 2: F_16, 4096^3, packed -> sliced -> product -> packed
    e, m = 4, 4096
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, m, 1)
    B = g.PackedMatrix.random(ctx, m, m, 2)
    C = g.karatsuba_mul_packed(A, B, backend=backend)
    ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, m, 1), oracle.sliced_random(e, m, m, 2), m, m, m)
    assert np.array_equal(C.to_numpy(), oracle.cling_words(e, m, m, ref))


def _sampled_blocks(g, e, m, k, n, accumulate, rows, col_block, backend="tc"):
    """C[R, S] = A[R, :] . B[:, S] (^ C0[R, S]) via the windowed generator."""
    ctx = g.field_new(e)
    SA = g.SlicedMatrix.random(ctx, m, k, 1)
    SB = g.SlicedMatrix.random(ctx, k, n, 2)
    if accumulate:
        C = g.SlicedMatrix.random(ctx, m, n, 3)
        g.addmul(C, SA, SB, backend=backend)
    else:
        C = g.karatsuba_mul(SA, SB, backend=backend)
    _sync()
    c0, c1 = col_block
    got = C.planes[:, rows, c0 // 64:c1 // 64]
    got = got.cpu().numpy().view(np.uint64)
    for i, r in enumerate(rows):
        a = oracle.sliced_random(e, 1, k, 1, row0=r, gcols=k)
        b = oracle.sliced_random(e, k, c1 - c0, 2, col0=c0, gcols=n)
        ref, _ = oracle.karatsuba(e, ctx.f, a, b, 1, k, c1 - c0)
        if accumulate:
            ref ^= oracle.sliced_random(e, 1, c1 - c0, 3, row0=r, col0=c0, gcols=n)
        assert np.array_equal(got[:, i:i + 1, :], ref), (r, col_block)


def _row_blocks(g, C, e, k, n, accumulate, blocks, col_block):
    """Contiguous row blocks [r0, r0 + nr) x columns [c0, c1) of the device result against the
    oracle on the same windows of the generator streams (A seed 1, B seed 2, C0 seed 3)."""
    ctx = C.ctx
    c0, c1 = col_block
    b = oracle.sliced_random(e, k, c1 - c0, 2, col0=c0, gcols=n)
    for r0, nr in blocks:
        got = C.planes[:, r0:r0 + nr, c0 // 64:-(-c1 // 64)].cpu().numpy().view(np.uint64)
        a = oracle.sliced_random(e, nr, k, 1, row0=r0, gcols=k)
        C0 = oracle.sliced_random(e, nr, c1 - c0, 3, row0=r0, col0=c0, gcols=n) if accumulate else None
        ref, _ = oracle.karatsuba(e, ctx.f, a, b, nr, k, c1 - c0, C0=C0)
        assert np.array_equal(got, ref), (e, r0, nr, col_block)


@pytest.mark.slow
def test_config3_sampled_blocks(g):
    # BASELINE config 3: F_256, 16384^3 on one GPU; sampled rows x 256-column blocks
    rows = [0, 1, 127, 128, 8191, 16383]
    _sampled_blocks(g, 8, 16384, 16384, 16384, False, rows, (16128, 16384))
    _sampled_blocks(g, 8, 16384, 16384, 16384, False, [5, 9000], (0, 256))


@pytest.mark.slow
def test_config3_full(g):
    # BASELINE config 3 in full: every element of the 16384^3 F_256 product
    # against the oracle's C restatement of the reference (poly_mul.py:245-259) on all host
    # cores (~100 s on 16 threads)
    e, m = 8, 16384
    ctx = g.field_new(e)
    C = g.karatsuba_mul(g.SlicedMatrix.random(ctx, m, m, 1), g.SlicedMatrix.random(ctx, m, m, 2))
    got = C.to_numpy()
    del C
    ref, cnt = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, m, 1), oracle.sliced_random(e, m, m, 2), m, m, m)
    assert cnt.gf2_matmul_count == 27
    bad = np.nonzero((got != ref).any(axis=(0, 2)))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:8]}"


@pytest.mark.slow
@pytest.mark.parametrize("e", range(2, 11))
def test_config4_sampled_blocks(g, e):
    # BASELINE config 4: C += A.B, A 65536x256, B 256x65536, C pre-filled (seed 3), every e;
    # 64 rows (the first tile, a middle tile boundary, the last row tile) x the rightmost 512
    # columns, and 16 rows x the first 256 columns
    m, k, n = 65536, 256, 65536
    ctx = g.field_new(e)
    SA = g.SlicedMatrix.random(ctx, m, k, 1)
    SB = g.SlicedMatrix.random(ctx, k, n, 2)
    C = g.SlicedMatrix.random(ctx, m, n, 3)
    g.addmul(C, SA, SB)
    _sync()
    _row_blocks(g, C, e, k, n, True, [(0, 16), (32760, 16), (m - 32, 32)], (n - 512, n))
    _row_blocks(g, C, e, k, n, True, [(40000, 16)], (0, 256))


@pytest.mark.parametrize("backend", BACKENDS)
def test_linearity_and_addmul_consistency(g, backend):
    # size-independent properties: (A1 + A2).B = A1.B + A2.B ; addmul == C0 + mul
    e, m, k, n = 7, 700, 900, 600
    ctx = g.field_new(e)
    A1 = g.SlicedMatrix.random(ctx, m, k, 11)
    A2 = g.SlicedMatrix.random(ctx, m, k, 12)
    B = g.SlicedMatrix.random(ctx, k, n, 13)
    lhs = g.karatsuba_mul(A1 ^ A2, B, backend=backend)
    rhs = g.karatsuba_mul(A1, B, backend=backend) ^ g.karatsuba_mul(A2, B, backend=backend)
    assert lhs == rhs
    C0 = g.SlicedMatrix.random(ctx, m, n, 14)
    D = C0.copy()
    g.addmul(D, A1, B, backend=backend)
    assert D == (C0 ^ g.karatsuba_mul(A1, B, backend=backend))


def test_backends_agree_large(g):
    e, m, k, n = 8, 2048, 2048, 2048
    ctx = g.field_new(e)
    A = g.SlicedMatrix.random(ctx, m, k, 1)
    B = g.SlicedMatrix.random(ctx, k, n, 2)
    assert g.karatsuba_mul(A, B, backend="tc") == g.karatsuba_mul(A, B, backend="m4rm")


def test_native_code_used(g):
    ctx = g.field_new(8)
    A = g.SlicedMatrix.random(ctx, 256, 256, 1)
    g.karatsuba_mul(A, A)
    assert g._lib.last_product_kernel() == "k_product_run<fp4>"  # k < 2048: running-sum form
    assert g._lib.last_launch_count() == 3  # combos(A), combos(B^T), fused product
    # the grouped running-sum sequence: K(8) = 27 products, some accumulated into two groups
    seq, _, _, load = g._lib.run_schedule(8, ctx.f)
    assert g._lib.last_gf2_products() == len(seq) and len(seq) >= 27
    g.karatsuba_mul(A, A, backend="tc_i8")
    assert g._lib.last_product_kernel() == "k_product_tc2<i8>"
    B = g.SlicedMatrix.random(ctx, 4096, 256, 2)
    g.karatsuba_mul(g.SlicedMatrix.random(ctx, 256, 4096, 1), B)
    assert g._lib.last_product_kernel() == "k_product_tc2<fp4>"
    g.karatsuba_mul(A, A, backend="tc_fp4")
    assert g._lib.last_product_kernel() == "k_product_tc2<fp4x2>"  # k < 2048 forced fp4: paired form


@pytest.mark.parametrize("acc", [False, True])
@pytest.mark.parametrize("e,m,k,n,chunk", [(8, 1000, 700, 600, 256), (4, 4096, 4096, 4096, 0), (2, 300, 0, 65, 0),
                                           (2, 600, 300, 8300, 256), (8, 520, 2100, 8192, 256),
                                           (10, 513, 129, 257, 512), (3, 1, 1, 1, 0),
                                           (4, 1324, 200, 9800, 512), (5, 1300, 2100, 9900, 512),
                                           (2, 5000, 300, 8500, 0), (3, 7000, 260, 10000, 0)])
def test_host_buffer_api(g, e, m, k, n, chunk, acc):
    # gf2e_mzed_mul_host: packed host words in, packed host words out, chunked + overlapped
    ctx = g.field_new(e)
    A = oracle.packed_random(e, m, k, 1)
    B = oracle.packed_random(e, k, n, 2)
    C0 = oracle.packed_random(e, m, n, 3) if acc else None
    C, ms = g.karatsuba_mul_packed_host(ctx, A, k, B, n, C_words=None if C0 is None else C0.copy(), chunk_rows=chunk)
    ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2), m, k, n,
                              C0=None if C0 is None else oracle.slice_words(e, m, n, C0))
    assert np.array_equal(C, oracle.cling_words(e, m, n, ref))
    assert ms >= 0


@pytest.mark.parametrize("seed", range(int(os.environ.get("GF2E_FUZZ_SEEDS", "12")) // 2 + 2))
def test_host_buffer_fuzz(g, seed):
    # the host-buffer pipeline's chunking (row plan, B column parts, side-stream preparation,
    # split last chunk) against the device product on the same operands
    import torch

    rng = np.random.default_rng(7000 + seed)
    e = int(rng.integers(2, 11))
    m = int(rng.integers(1, 3000))
    k = int(rng.integers(1, 600)) if seed % 2 else int(rng.integers(4096, 5200))
    n = int(rng.integers(1, 900)) if seed % 3 == 0 else int(rng.integers(8192, 9800))
    chunk = [0, 256, 512, 768][seed % 4]
    acc = seed % 5 == 1
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, m, k, 80 + seed)
    B = g.PackedMatrix.random(ctx, k, n, 81 + seed)
    if acc:
        C = g.PackedMatrix.random(ctx, m, n, 82 + seed)
        C0 = C.to_numpy().copy()
        g.addmul_packed(C, A, B)
        ref = C.to_numpy()
        out, _ = g.karatsuba_mul_packed_host(ctx, A.to_numpy(), k, B.to_numpy(), n, C_words=C0, chunk_rows=chunk)
    else:
        ref = g.karatsuba_mul_packed(A, B).to_numpy()
        out, _ = g.karatsuba_mul_packed_host(ctx, A.to_numpy(), k, B.to_numpy(), n, chunk_rows=chunk)
    torch.cuda.synchronize()
    wb = g.words_for(n * g.pack_width(e))
    assert np.array_equal(out[:, :wb], ref[:, :wb]), (e, m, k, n, chunk, acc)


@pytest.mark.slow
def test_config5_sampled_blocks(g):
    # BASELINE config 5: F_256, 65536^3 on one GPU (the per-GPU problem of the 1-GPU point of the
    # scaling run); sampled rows x 256-column blocks against the oracle
    import torch

    free, _ = torch.cuda.mem_get_info()
    if free < 60 * 2**30:
        pytest.skip("needs ~60 GiB of free HBM")
    _sampled_blocks(g, 8, 65536, 65536, 65536, False, [0, 255, 40000, 65535], (65536 - 256, 65536))


@pytest.mark.parametrize("seed", range(int(os.environ.get("GF2E_FUZZ_SEEDS", "12"))))
def test_fuzz_shapes(g, seed):
    # random e, shapes (ragged, word-boundary-crossing, some long-k for the fp4 forms) and
    # addmul/mul, every backend, against the oracle
    rng = np.random.default_rng(1000 + seed)
    e = int(rng.integers(2, 11))
    m, n = (int(x) for x in rng.integers(1, 700, size=2))
    k = int(rng.integers(1, 700)) if seed % 3 else int(rng.integers(2048, 9000))
    ctx = g.field_new(e)
    SA = g.SlicedMatrix.random(ctx, m, k, seed + 1)
    SB = g.SlicedMatrix.random(ctx, k, n, seed + 2)
    ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, seed + 1),
                              oracle.sliced_random(e, k, n, seed + 2), m, k, n)
    c0 = oracle.sliced_random(e, m, n, seed + 3)
    for backend in BACKENDS:
        C = g.karatsuba_mul(SA, SB, backend=backend)
        assert np.array_equal(C.to_numpy(), ref), (e, m, k, n, backend)
        C0 = g.SlicedMatrix.random(ctx, m, n, seed + 3)
        g.addmul(C0, SA, SB, backend=backend)
        assert np.array_equal(C0.to_numpy(), ref ^ c0), (e, m, k, n, backend, "addmul")


def test_fp4_selfcheck_guard(g):
    # the fp4 exactness self-check: passes on this device; an injected mismatch disables the
    # fp4 forms (products fall back to kind::i8 and stay bit-exact); a re-run restores them
    assert g._lib.fp4_selfcheck() == 1
    ctx = g.field_new(6)
    m, k, n = 300, 9000, 200
    SA = g.SlicedMatrix.random(ctx, m, k, 1)
    SB = g.SlicedMatrix.random(ctx, k, n, 2)
    ref, _ = oracle.karatsuba(6, ctx.f, oracle.sliced_random(6, m, k, 1), oracle.sliced_random(6, k, n, 2), m, k, n)
    try:
        assert g._lib.fp4_selfcheck(rerun=True, inject_fault=True) == -1
        C = g.karatsuba_mul(SA, SB)
        assert g._lib.last_product_kernel() == "k_product_tc2<i8>"
        assert np.array_equal(C.to_numpy(), ref)
    finally:
        assert g._lib.fp4_selfcheck(rerun=True) == 1
    C = g.karatsuba_mul(SA, SB)
    assert g._lib.last_product_kernel() == "k_product_tc2<fp4>"
    assert np.array_equal(C.to_numpy(), ref)


@pytest.mark.parametrize("e", range(2, 11))
def test_run_form_all_e(g, e):
    # the running-sum form (double-buffered accumulators, 256 x 192 tiles): k = 256 (the
    # config-4 / Schur-update shape), ragged m, n across 192-column tiles, an odd number of
    # 256-bit stages, the longest k whose running sums stay below 2^16; mul and addmul
    ctx = g.field_new(e)
    K = g.count_products(e)
    kmax = (65535 // ((K + 1) // 2)) // 256 * 256
    for (m, k, n) in [(513, 256, 577), (256, 256, 192), (300, 700, 1000), (70, kmax, 200), (1, 1, 1)]:
        SA = g.SlicedMatrix.random(ctx, m, k, 1)
        SB = g.SlicedMatrix.random(ctx, k, n, 2)
        C0 = g.SlicedMatrix.random(ctx, m, n, 3)
        ref, _ = oracle.karatsuba(e, ctx.f, oracle.sliced_random(e, m, k, 1), oracle.sliced_random(e, k, n, 2),
                                  m, k, n)
        C = g.karatsuba_mul(SA, SB, backend="tc_run")
        assert g._lib.last_product_kernel() == "k_product_run<fp4>", (e, k)
        assert np.array_equal(C.to_numpy(), ref), (e, m, k, n)
        g.addmul(C0, SA, SB, backend="tc_run")
        assert np.array_equal(C0.to_numpy(), ref ^ oracle.sliced_random(e, m, n, 3)), (e, m, k, n, "addmul")


def test_run_form_falls_back_past_its_range(g):
    # ceil(K/2) * k >= 2^16: the forced running-sum form would overflow its exact range, so
    # the call takes the fp4 long form (and stays exact)
    ctx = g.field_new(2)
    m, k, n = 70, 44000, 200
    C = g.karatsuba_mul(g.SlicedMatrix.random(ctx, m, k, 1), g.SlicedMatrix.random(ctx, k, n, 2), backend="tc_run")
    assert g._lib.last_product_kernel() == "k_product_tc2<fp4>"
    ref, _ = oracle.karatsuba(2, ctx.f, oracle.sliced_random(2, m, k, 1), oracle.sliced_random(2, k, n, 2), m, k, n)
    assert np.array_equal(C.to_numpy(), ref)


def test_run_form_column_view(g):
    # C as a column window of a wider plane stack (ldc > words(n)): the 32-bit stores must
    # leave the neighbouring words alone
    ctx = g.field_new(5)
    m, k, n, wide = 300, 256, 640, 1000
    SA = g.SlicedMatrix.random(ctx, m, k, 1)
    SB = g.SlicedMatrix.random(ctx, k, n, 2)
    W = g.SlicedMatrix.random(ctx, m, wide, 9)
    before = W.to_numpy()
    L = g._lib
    flags = L.ACCUMULATE | L.TC_RUN
    ws = g._device.workspace.get(int(L.load().gf2e_slice_mul_workspace(5, ctx.f, m, k, n, flags)))
    ldw, lda, ldb = W.planes.shape[2], SA.planes.shape[2], SB.planes.shape[2]
    L.call("gf2e_slice_mul", 5, ctx.f, SA.planes.data_ptr(), lda, m * lda, SB.planes.data_ptr(), ldb, k * ldb,
           W.planes.data_ptr() + 2 * 8, ldw, m * ldw, m, k, n, flags, ws.data_ptr(), ws.numel(),
           g._device.stream_handle())
    assert L.last_product_kernel() == "k_product_run<fp4>"
    after = W.to_numpy()
    ref, _ = oracle.karatsuba(5, ctx.f, oracle.sliced_random(5, m, k, 1), oracle.sliced_random(5, k, n, 2), m, k, n)
    assert np.array_equal(after[:, :, 2:2 + g.words_for(n)], before[:, :, 2:2 + g.words_for(n)] ^ ref)
    assert np.array_equal(after[:, :, :2], before[:, :, :2])
    assert np.array_equal(after[:, :, 2 + g.words_for(n):], before[:, :, 2 + g.words_for(n):])


def test_nj_small_products_golden(g, golden):
    # the packed-domain Newton-John kernel (gf2e_nj_mul) on the reference's fixtures: product,
    # addmul, through the routing of karatsuba_mul_packed / addmul_packed and nj_mul directly
    from paper_1111_6900_b200 import poly_mul

    for tag in _tags(golden, "kara_tags"):
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        ctx = g.field_new(e, f)
        A = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/A_packed"], k)
        B = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/B_packed"], n)
        if not poly_mul.nj_fits(e, n):
            continue
        assert np.array_equal(poly_mul.nj_mul_packed(A, B).to_numpy(), golden[f"{tag}/C_packed"]), tag
        assert np.array_equal(g.nj_mul(A, B).to_numpy(), golden[f"{tag}/C_packed"]), tag
        C0 = g.PackedMatrix.from_numpy(ctx, golden[f"{tag}/C0_packed"], n)
        poly_mul.nj_mul_packed(A, B, C0)
        assert np.array_equal(C0.to_numpy(), golden[f"{tag}/addmul_packed"]), tag
        if max(m, k, n) <= poly_mul.NJ_CROSSOVER[e]:
            assert np.array_equal(g.karatsuba_mul_packed(A, B).to_numpy(), golden[f"{tag}/C_packed"]), tag
            assert g._lib.last_product_kernel() == "k_nj_mul"


@pytest.mark.parametrize("e", range(2, 11))
def test_nj_sliced_oracle(g, e):
    # the bit-plane Newton-John product (gf2e_nj_slice_mul: PLE / TRSM small updates) against
    # the oracle, k across table chunks (32 rows of B) and words, n with a partial last word
    from paper_1111_6900_b200 import poly_mul

    ctx = g.field_new(e)
    for (m, k, n) in [(1, 1, 1), (5, 7, 3), (64, 64, 64), (65, 100, 130), (200, 33, 63), (130, 257, 17),
                      (300, 128, 200)]:
        A = oracle.packed_random(e, m, k, 1)
        B = oracle.packed_random(e, k, n, 2)
        C0 = oracle.packed_random(e, m, n, 3)
        SA = oracle.slice_words(e, m, k, A)
        SB = oracle.slice_words(e, k, n, B)
        SC = oracle.slice_words(e, m, n, C0)
        ref, _ = oracle.karatsuba(e, ctx.f, SA, SB, m, k, n)
        gA = g.SlicedMatrix.from_numpy(ctx, SA, k)
        gB = g.SlicedMatrix.from_numpy(ctx, SB, n)
        gC = g.SlicedMatrix.from_numpy(ctx, SC, n)
        assert np.array_equal(poly_mul.nj_mul_sliced(gA, gB).to_numpy(), ref), (m, k, n)
        assert g._lib.last_product_kernel() == "k_nj_sliced"
        poly_mul.nj_mul_sliced(gA, gB, gC)
        assert np.array_equal(gC.to_numpy(), ref ^ SC), (m, k, n, "acc")


@pytest.mark.parametrize("e", [4, 8, 10])
def test_nj_sliced_vs_tensor_cores(g, e):
    # larger shapes (grids with several passes per row block) against the tensor-core product
    from paper_1111_6900_b200 import poly_mul

    ctx = g.field_new(e)
    for (m, k, n) in [(8128, 64, 64), (128, 128, 8064), (3000, 96, 700), (40000, 64, 128)]:
        A = g.SlicedMatrix.random(ctx, m, k, 1)
        B = g.SlicedMatrix.random(ctx, k, n, 2)
        C = g.SlicedMatrix.random(ctx, m, n, 3)
        want = C.copy()
        g.addmul(want, A, B, backend="tc")
        poly_mul.nj_mul_sliced(A, B, C)
        assert np.array_equal(C.to_numpy(), want.to_numpy()), (m, k, n)


@pytest.mark.parametrize("e", range(2, 11))
def test_nj_small_products_oracle(g, e):
    from paper_1111_6900_b200 import poly_mul

    ctx = g.field_new(e)
    nmax = {2: 512, 3: 256, 4: 256}.get(e, 128 if e <= 8 else 64)
    for (m, k, n) in [(1, 1, 1), (5, 7, 3), (64, 64, 64), (65, 100, nmax), (200, 33, nmax - 1), (3, 0, 5),
                      (130, 257, 17)]:
        A = oracle.packed_random(e, m, k, 1)
        B = oracle.packed_random(e, k, n, 2)
        C0 = oracle.packed_random(e, m, n, 3)
        PA = g.PackedMatrix.from_numpy(ctx, A, k)
        PB = g.PackedMatrix.from_numpy(ctx, B, n)
        PC = g.PackedMatrix.from_numpy(ctx, C0, n)
        ref, _ = oracle.karatsuba(e, ctx.f, oracle.slice_words(e, m, k, A), oracle.slice_words(e, k, n, B), m, k, n)
        assert np.array_equal(poly_mul.nj_mul_packed(PA, PB).to_numpy(), oracle.cling_words(e, m, n, ref)), (m, k, n)
        poly_mul.nj_mul_packed(PA, PB, PC)
        ref2 = ref ^ oracle.slice_words(e, m, n, C0)
        assert np.array_equal(PC.to_numpy(), oracle.cling_words(e, m, n, ref2)), (m, k, n, "acc")


def test_release_workspace(g):
    # scratch buffers can be dropped between calls (and the library pool trimmed); products
    # computed before and after are identical
    ctx = g.field_new(8)
    A = g.SlicedMatrix.random(ctx, 300, 500, 1)
    B = g.SlicedMatrix.random(ctx, 500, 400, 2)
    C1 = g.karatsuba_mul(A, B).to_numpy()
    g.release_workspace()
    assert np.array_equal(g.karatsuba_mul(A, B).to_numpy(), C1)

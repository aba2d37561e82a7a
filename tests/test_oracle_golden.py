"""Pin the CPU oracle (oracle/) to fixtures produced by the reference package itself
(tests/golden/make_golden.py imports /root/reference/pkg/src/gf2elin).  CPU only."""

import numpy as np
import pytest

import oracle


def _tags(golden, key):
    return [str(t) for t in golden[key]]


def test_rng_word_stream(golden):
    # rng.py:20-28
    for seed in (0, 1, 2, 3, 2**64 - 1):
        assert np.array_equal(oracle.word_stream(seed, 16), golden[f"rng/{seed}"])


def test_default_polys_and_counts(golden):
    assert [oracle.DEFAULT_POLYS[e] for e in range(2, 11)] == list(golden["default_polys"])
    # poly_mul.count_products (poly_mul.py:262-272): 3, 6, 9, 15, 18, 24, 27, 39, 45
    assert [oracle.schedule(e).n_products for e in range(2, 11)] == list(golden["count_products"])
    assert list(golden["count_products"]) == [3, 6, 9, 15, 18, 24, 27, 39, 45]


@pytest.mark.parametrize("e", range(2, 11))
def test_schedule_shape(e):
    # SURVEY §7.1 measured facts: sum |S_t| and nnz(M) for the default f
    s = oracle.schedule(e)
    ssum = [4, 9, 16, 28, 36, 53, 64, 95, 112][e - 2]
    nnz = [4, 10, 21, 35, 52, 87, 111, 141, 218][e - 2]
    assert sum(bin(x).count("1") for x in s.subsets) == ssum
    assert sum(bin(x).count("1") for x in s.outmap) == nnz


def test_karatsuba_cases(golden):
    for tag in _tags(golden, "kara_tags"):
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        # generator (mat_packed.py:253-259)
        assert np.array_equal(oracle.packed_random(e, m, k, 1), golden[f"{tag}/A_packed"]), tag
        assert np.array_equal(oracle.packed_random(e, k, n, 2), golden[f"{tag}/B_packed"]), tag
        # slice (mat_sliced.py:97-101) and the direct sliced generator
        pa = oracle.slice_words(e, m, k, golden[f"{tag}/A_packed"])
        pb = oracle.slice_words(e, k, n, golden[f"{tag}/B_packed"])
        assert np.array_equal(pa, golden[f"{tag}/A_planes"]), tag
        assert np.array_equal(pb, golden[f"{tag}/B_planes"]), tag
        assert np.array_equal(oracle.sliced_random(e, m, k, 1), pa), tag
        # karatsuba_mul + counters (poly_mul.py:245-259)
        C, cnt = oracle.karatsuba(e, f, pa, pb, m, k, n)
        assert np.array_equal(C, golden[f"{tag}/C_planes"]), tag
        assert [cnt.gf2_matmul_count, cnt.additions, cnt.peak_live_products] == list(golden[f"{tag}/counters"])
        sch = oracle.schedule(e, f)
        assert (sch.counters.gf2_matmul_count, sch.counters.additions, sch.counters.peak_live_products) == (
            cnt.gf2_matmul_count, cnt.additions, cnt.peak_live_products)
        # schedule as data reproduces the product
        assert np.array_equal(oracle.apply_schedule(sch, pa, pb, m, k, n), C), tag
        # cling (mat_sliced.py:104-106) == karatsuba_mul_packed
        assert np.array_equal(oracle.cling_words(e, m, n, C), golden[f"{tag}/C_packed"]), tag
        # addmul == C0 xor A*B (ple_echelon.py:259 pattern)
        c0 = golden[f"{tag}/C0_planes"]
        Cacc, _ = oracle.karatsuba(e, f, pa, pb, m, k, n, C0=c0)
        assert np.array_equal(oracle.cling_words(e, m, n, Cacc), golden[f"{tag}/addmul_packed"]), tag


def test_gf2_products(golden):
    for tag in _tags(golden, "gf2_tags"):
        m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        C = oracle.gf2_mul(golden[f"{tag}/A"], golden[f"{tag}/B"], m, k, n)
        assert np.array_equal(C, golden[f"{tag}/C"]), tag


def test_fig1(golden):
    # SPEC.md:258 / PAPER Fig. 1: [[5,2],[3,1]] over GF(8)
    planes = oracle.slice_words(3, 2, 2, golden["fig1/packed"])
    assert np.array_equal(planes, golden["fig1/planes"])
    assert planes[:, :, 0].tolist() == [[0b01, 0b11], [0b10, 0b01], [0b01, 0b00]]
    assert np.array_equal(oracle.cling_words(3, 2, 2, planes), golden["fig1/packed"])


def test_reduce_known_answer(golden):
    # GF(4) (C0, C1, C2) -> (C0 ^ C2, C1 ^ C2)
    cin = golden["reduce/e2/in"]
    out = golden["reduce/e2/out"]
    assert np.array_equal(out[0], cin[0] ^ cin[2])
    assert np.array_equal(out[1], cin[1] ^ cin[2])
    # e = 8: the schedule's fold matrix reproduces the reference reduce_mod_f
    s = oracle.schedule(8)
    cin = golden["reduce/e8/in"]
    for j in range(8):
        acc = np.zeros_like(cin[0])
        for d in range(15):
            if (s.fold[j] >> d) & 1:
                acc ^= cin[d]
        assert np.array_equal(acc, golden["reduce/e8/out"][j])


def test_sampled_block_generator():
    # a window of the generator matrix equals the same window of the full one
    e, m, n = 8, 50, 130
    full = oracle.sliced_random(e, m, n, 7)
    win = oracle.sliced_random(e, 10, 64, 7, row0=20, col0=64, gcols=n)
    assert np.array_equal(win[:, :, 0], full[:, 20:30, 1])


def _elements(words, e, m, n):
    w = oracle.pack_width(e)
    arr = np.zeros((m, n), dtype=np.uint16)
    for j in range(n):
        wd, s = divmod(j * w, 64)
        arr[:, j] = ((words[:, wd] >> np.uint64(s)) & np.uint64((1 << w) - 1)).astype(np.uint16)
    return arr


def test_oracle_ple_vs_reference(golden):
    # nj_ple restated in C (oracle/gf2e_oracle.c: orc_ple) against the reference's ple()
    for tag in (str(t) for t in golden["ple_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        a, P, Q, r = oracle.ple(e, f, _elements(golden[f"{tag}/A"], e, m, n))
        assert r == int(golden[f"{tag}/rank"][0]), tag
        assert np.array_equal(P, golden[f"{tag}/P"]) and np.array_equal(Q, golden[f"{tag}/Q"]), tag
        assert np.array_equal(a, _elements(golden[f"{tag}/ple"], e, m, n)), tag

"""MulCounters accounting of TRSM / PLE / echelonize (no GPU): the replay of the reference's
recursion (ple_echelon._ref_trsm_calls / _ref_ple_calls) against the counters the reference
itself produced (tests/golden/make_golden.py), at the default crossover and at 16."""

import numpy as np

import paper_1111_6900_b200 as g
from paper_1111_6900_b200 import ple_echelon as pe


def _expect(e, calls):
    K, adds, peak = g.schedule(e).counters
    return [K * calls, adds * calls, peak if calls else 0]


def test_trsm_counters_match_reference(golden):
    for tag in (str(t) for t in golden["trsm_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        got = []
        for cx in (None, 16):
            calls = pe._ref_trsm_calls(m, n, pe._crossover(cx))
            got += [_expect(e, calls)] * 3  # upper, lower, unit lower: same recursion shape
        assert got == golden[f"{tag}/counters"].tolist(), tag


def test_ple_and_echelonize_counters_match_reference(golden):
    checked = 0
    for tag in (str(t) for t in golden["ple_tags"]):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        r = int(golden[f"{tag}/rank"][0])
        pivots = golden[f"{tag}/Q"][:r]
        for row, cx in zip(golden[f"{tag}/counters"].tolist(), (None, 16)):
            if row[0] < 0:  # the reference's recursion raised at this crossover
                continue
            c = pe._crossover(cx)
            ple_calls = pe._ref_ple_calls(m, n, 0, pivots, c)
            assert row[0:3] == _expect(e, ple_calls), (tag, cx, "ple")
            full_calls = ple_calls + (pe._ref_trsm_calls(r, n, c) if r else 0)
            assert row[3:6] == _expect(e, full_calls), (tag, cx, "echelonize full")
            assert row[6:9] == _expect(e, ple_calls), (tag, cx, "echelonize row")
            checked += 1
    assert checked >= 20


def test_pivots_are_the_column_rank_profile(golden):
    # the replay assumes Q[:rank] lists the pivot columns in increasing order
    for tag in (str(t) for t in golden["ple_tags"]):
        r = int(golden[f"{tag}/rank"][0])
        q = golden[f"{tag}/Q"][:r]
        assert np.all(np.diff(q) > 0) and np.all(q >= np.arange(r)), tag

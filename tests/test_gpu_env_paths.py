"""Code paths that environment switches select at process start (read once per process, so
each runs in a fresh interpreter): the running-sum form's drain grouping (GF2E_RUN_DRAINS),
the consumers without programmatic dependent launch (GF2E_PDL=0), the small-product
crossover of PLE / TRSM (GF2E_NJS_MAXK=0: every update on the tensor cores), the paired drains
of the running-sum form (GF2E_RUN_PAIR_E).  Each child
compares its results with the oracle / with the default path computed here."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD_PRODUCT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1111_6900_b200 as g, oracle
from paper_1111_6900_b200 import _lib
out = {}
for e in (4, 8, 10):
    ctx = g.field_new(e)
    m, k, n = 300, 700, 400
    A = oracle.sliced_random(e, m, k, 1)
    B = oracle.sliced_random(e, k, n, 2)
    ref, _ = oracle.karatsuba(e, ctx.f, A, B, m, k, n)
    C = g.karatsuba_mul(g.SlicedMatrix.from_numpy(ctx, A, k), g.SlicedMatrix.from_numpy(ctx, B, n), backend="tc_run")
    seq, gsize, _, _ = _lib.run_schedule(e, ctx.f)
    out[e] = [bool(np.array_equal(C.to_numpy(), ref)), len(gsize), len(seq), _lib.last_gf2_products()]
print(json.dumps(out))
"""

CHILD_CONSUMERS = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1111_6900_b200 as g
res = []
for e, n in ((8, 700), (3, 520), (10, 300)):
    ctx = g.field_new(e)
    A = g.PackedMatrix.random(ctx, n, n, 11)
    P = A.copy()
    f = g.ple(P)
    E = A.copy()
    r = g.echelonize(E, full=True)
    U = np.triu(A.to_array(), 1)
    np.fill_diagonal(U, (np.arange(n) % (ctx.order - 1)) + 1)
    X = g.PackedMatrix.random(ctx, n, 333, 3)
    g.trsm_upper_left(g.PackedMatrix.from_array(ctx, U), X)
    res += [P.to_numpy(), E.to_numpy(), X.to_numpy(), np.array([r, f.rank]), f.P.entries, f.Q.entries]
np.savez(sys.argv[2], *res)
"""


def _run(code, env_extra, *args):
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", code, ROOT, *args], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return p.stdout


@pytest.mark.parametrize("drains", ["20", "12"])
def test_run_form_drain_grouping_parity(drains):
    # products accumulated in groups (fewer drains than products): bit-exact with the oracle,
    # and the launched GF(2) products are the grouped sequence's entries
    out = json.loads(_run(CHILD_PRODUCT, {"GF2E_RUN_DRAINS": drains}).strip().splitlines()[-1])
    for e, (ok, ngrp, nseq, launched) in out.items():
        assert ok, (drains, e)
        K = oracle.schedule(int(e)).counters.gf2_matmul_count
        assert ngrp <= max(int(drains), int(e)) or ngrp == K, (drains, e, ngrp)
        assert launched == nseq and nseq >= K, (drains, e)


def test_consumers_without_pdl_and_small_products_match(tmp_path):
    # PLE, echelonize and TRSM with programmatic dependent launch off, and with every update
    # on the tensor cores (no sliced Newton-John), equal the default paths bit for bit
    base = tmp_path / "base.npz"
    _run(CHILD_CONSUMERS, {}, str(base))
    ref = np.load(base)
    for env in ({"GF2E_PDL": "0"}, {"GF2E_NJS_MAXK": "0"}, {"GF2E_RUNX_MAXM": "0"}):
        alt = tmp_path / "alt.npz"
        _run(CHILD_CONSUMERS, env, str(alt))
        got = np.load(alt)
        for key in ref.files:
            assert np.array_equal(ref[key], got[key]), (env, key)


CHILD_RUN_ALL_E = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1111_6900_b200 as g, oracle
out = {}
for e in range(2, 11):
    ctx = g.field_new(e)
    for (m, k, n, acc) in ((520, 256, 700, True), (300, 64, 260, False), (2100, 130, 450, True)):
        A = oracle.sliced_random(e, m, k, 1)
        B = oracle.sliced_random(e, k, n, 2)
        C0 = oracle.sliced_random(e, m, n, 3)
        ref, _ = oracle.karatsuba(e, ctx.f, A, B, m, k, n)
        C = g.SlicedMatrix.from_numpy(ctx, C0.copy(), n)
        if acc:
            g.addmul(C, g.SlicedMatrix.from_numpy(ctx, A, k), g.SlicedMatrix.from_numpy(ctx, B, n), backend="tc_run")
            ref = ref ^ C0
        else:
            C = g.karatsuba_mul(g.SlicedMatrix.from_numpy(ctx, A, k), g.SlicedMatrix.from_numpy(ctx, B, n),
                                backend="tc_run")
        out[f"{e}/{m}x{k}x{n}"] = bool(np.array_equal(C.to_numpy(), ref))
print(json.dumps(out))
"""


@pytest.mark.parametrize("pair_e", ["0x1fc", "0"])
def test_run_form_paired_drains_parity(pair_e):
    # the paired-drain running-sum form (two groups per accumulator fill, the second scaled by
    # 2^11) forced on for every e <= 8 where its sums stay exact, and forced off: bit-exact
    # with the oracle for every e, mul and addmul, in-kernel and pre-expanded B (m > 2048)
    out = json.loads(_run(CHILD_RUN_ALL_E, {"GF2E_RUN_PAIR_E": pair_e}).strip().splitlines()[-1])
    bad = [key for key, ok in out.items() if not ok]
    assert not bad, (pair_e, bad)

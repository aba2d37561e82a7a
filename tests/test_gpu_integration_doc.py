"""The reference-side ctypes binding shown in INTEGRATION.md, executed verbatim (only the
library path is substituted), against fixtures the reference produced: the documented
drop-in boundary works as written."""

import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_namespace():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# gf2elin/_b200\.py.*?)```", text, re.S).group(1)
    lib = os.path.join(ROOT, "paper_1111_6900_b200", "libgf2e_b200.so")
    block = block.replace('ctypes.CDLL("libgf2e_b200.so")', f"ctypes.CDLL({lib!r})")
    ns = {}
    exec(compile(block, "INTEGRATION.md:_b200.py", "exec"), ns)
    return ns


def test_integration_stub_slice_mul(golden):
    pytest.importorskip("cuda.bindings.runtime")
    ns = _stub_namespace()
    for tag in ("kara/e8/37x70x65", "kara/e2/63x64x65", "kara/e10/65x129x128"):
        if f"{tag}/meta" not in golden:
            continue
        e, f, m, k, n = (int(x) for x in golden[f"{tag}/meta"])
        A, B = golden[f"{tag}/A_planes"], golden[f"{tag}/B_planes"]
        C = ns["slice_mul"](e, f, A, B, m, k, n)
        assert np.array_equal(C, golden[f"{tag}/C_planes"]), tag
        C0 = golden[f"{tag}/C0_planes"]
        Cacc = ns["slice_mul"](e, f, A, B, m, k, n, C_planes=C0.copy())
        assert np.array_equal(Cacc, C0 ^ golden[f"{tag}/C_planes"]), tag
    with pytest.raises(ValueError):      # e outside 2..10: GF2E_EINVAL -> ValueError, as the stub maps it
        ns["slice_mul"](11, 0x805, np.zeros((11, 4, 1), np.uint64), np.zeros((11, 3, 1), np.uint64), 4, 3, 5)


def test_integration_stub_ple(golden):
    """The INTEGRATION.md ``ple`` call site: plane stack in, PLE'd planes + P, Q, rank out."""
    pytest.importorskip("cuda.bindings.runtime")
    import ctypes

    import oracle

    ns = _stub_namespace()
    L, rt, dev = ns["_L"], ns["rt"], ns["_dev"]
    I64P = ctypes.POINTER(ctypes.c_int64)
    for tag in ("ple/e8/150x256/rand", "ple/e4/300x512/lowrank", "ple/e10/70x70/rand"):
        e, f, m, n = (int(x) for x in golden[f"{tag}/meta"])
        S = np.ascontiguousarray(oracle.slice_words(e, m, n, golden[f"{tag}/A"]))
        P = np.zeros(min(m, n), np.int64)
        Q = np.zeros_like(P)
        r = ctypes.c_int64()
        dS = dev(S)
        rc = L.gf2e_ple(e, f, dS, S.shape[2], m * S.shape[2], m, n,
                        P.ctypes.data_as(I64P), Q.ctypes.data_as(I64P), ctypes.byref(r), None)
        assert rc == 0, L.gf2e_last_error().decode()
        rt.cudaMemcpy(S.ctypes.data, dS, S.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        rt.cudaFree(dS)
        assert r.value == int(golden[f"{tag}/rank"][0]), tag
        assert np.array_equal(P, golden[f"{tag}/P"]) and np.array_equal(Q, golden[f"{tag}/Q"]), tag
        assert np.array_equal(oracle.cling_words(e, m, n, S), golden[f"{tag}/ple"]), tag

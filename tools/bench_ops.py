"""Per-kernel measurements beside bench.py's headline: HBM-bound conversions against the
measured HBM roofline, and the TRSM consumer's throughput.  Prints one JSON line per op.

    python tools/bench_ops.py [--e 8] [--m 16384] [--n 16384]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1111_6900_b200 as g  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--e", type=int, default=8)
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--trsm-m", type=int, default=8192)
    ap.add_argument("--ple-n", type=int, default=8192)
    ap.add_argument("--skip-hbm", action="store_true")
    a = ap.parse_args()
    try:
        hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                          "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        hbm = 6650.0
    e, m, n = a.e, a.m, a.n
    ctx = g.field_new(e)
    w = g.pack_width(e)
    P = g.PackedMatrix.random(ctx, m, n, 1)
    S = g.slice_packed(P)
    packed_b = m * g.words_for(n * w) * 8
    planes_b = e * m * g.words_for(n) * 8

    def line(op, ms, bytes_, extra=None):
        gbs = bytes_ / (ms * 1e-3) / 1e9
        d = {"op": op, "e": e, "shape": [m, n], "ms": round(ms, 4), "bytes": bytes_, "GB/s": round(gbs, 1),
             "hbm_peak_GB/s": hbm, "frac": round(gbs / hbm, 3)}
        d.update(extra or {})
        print(json.dumps(d), flush=True)

    if a.skip_hbm:
        return ple_lines(a, ctx)
    line("slice (K1)", timed(lambda: g.slice_packed(P, out=S)), packed_b + planes_b)
    line("cling (K2)", timed(lambda: g.cling(S, out=P)), packed_b + planes_b)
    line("mul_by_x", timed(lambda: g.mul_by_x(S)), 2 * planes_b)
    line("scalar_mul", timed(lambda: P.scalar_mul(3)), 2 * packed_b)
    line("random_sliced (K7)", timed(lambda: g.SlicedMatrix.random(ctx, m, n, 5)), planes_b,
         {"note": "ALU-bound generator (2 64-bit multiplies per element)"})

    # TRSM consumer: U X = B, m x m upper triangular, n right-hand sides
    tm = a.trsm_m
    R = g.PackedMatrix.random(ctx, tm, tm, 7).to_array()
    up = np.triu(R, 1)
    np.fill_diagonal(up, (np.arange(tm) % (ctx.order - 1)) + 1)
    Us = g.slice_packed(g.PackedMatrix.from_array(ctx, up))
    B0 = g.SlicedMatrix.random(ctx, tm, n, 8)
    X = B0.copy()

    def solve():
        X.planes.copy_(B0.planes)
        g.trsm_sliced(Us, X, upper=True)

    ms = timed(solve, reps=3, warm=1)
    K = g.count_products(e)
    ops = K * tm * tm * n  # ~K(e) * 2 * (m^2/2) * n GF(2) bit-ops for the triangular product
    print(json.dumps({"op": "trsm_upper (sliced)", "e": e, "m": tm, "n": n, "ms": round(ms, 3),
                      "eff_Tbit-op/s": round(ops / (ms * 1e-3) / 1e12, 1),
                      "note": "K(e)*m^2*n GF(2) bit-ops; updates via addmul, 256-row diagonal blocks (128 below "
                              "m = 1024 or n = 4096) inverted on device"}),
          flush=True)
    ple_lines(a, ctx)


def ple_lines(a, ctx):
    """PLE / echelonize consumers: device time at n x n, and the oracle's nj_ple (C, all host
    threads) at a size it finishes, for scale."""
    import time

    import oracle

    e = ctx.e
    n = a.ple_n
    A = g.PackedMatrix.random(ctx, n, n, 11)
    S0 = g.slice_packed(A)
    S = S0.copy()

    def run_ple():
        S.planes.copy_(S0.planes)
        g.ple_sliced(S)

    ms = timed(run_ple, reps=5, warm=2)
    K = g.count_products(e)
    print(json.dumps({"op": "ple (sliced, in place)", "e": e, "m": n, "n": n, "ms": round(ms, 2),
                      "eff_Tbit-op/s": round(K * 2 * n ** 3 / 3 / (ms * 1e-3) / 1e12, 1),
                      "note": "work ~ K(e)*2n^3/3 GF(2) bit-ops (LU-like); 64-col panels on device, Schur "
                              "updates via addmul, corner solves via device TRSM; host recursion syncs per panel"}),
          flush=True)

    def run_ech():
        S.planes.copy_(S0.planes)
        g.echelonize_sliced(S, True)

    ms = timed(run_ech, reps=5, warm=2)
    print(json.dumps({"op": "echelonize full (sliced)", "e": e, "m": n, "n": n, "ms": round(ms, 2)}), flush=True)
    nc = 1024
    arr = g.PackedMatrix.random(ctx, nc, nc, 11).to_array()
    t0 = time.perf_counter()
    oracle.ple(e, ctx.f, arr)
    dt = time.perf_counter() - t0
    B = g.slice_packed(g.PackedMatrix.random(ctx, nc, nc, 11))

    def small():
        g.ple_sliced(B)

    ms_small = timed(small, reps=3, warm=1)
    print(json.dumps({"op": "ple 1024^2 GPU vs oracle nj_ple (C)", "e": e, "gpu_ms": round(ms_small, 2),
                      "cpu_ms": round(dt * 1e3, 1), "cpu_threads": oracle.max_threads()}), flush=True)


if __name__ == "__main__":
    main()

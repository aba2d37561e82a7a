"""Command-line harness (SPEC.md cli module): matrix files in and out,
products and echelon forms on the device, a self-test of the device path's algebraic
identities, and a one-line benchmark.

    python -m paper_1111_6900_b200 random E M N SEED OUT [--f HEX] [--repr packed|sliced]
    python -m paper_1111_6900_b200 mul A B OUT [--backend cubic|nj|strassen|karatsuba] [--crossover N] [--counts]
    python -m paper_1111_6900_b200 echelonize IN OUT [--full] [--backend nj|ple] [--crossover N]
    python -m paper_1111_6900_b200 selftest [--e 2,3,...] [--sizes 1,63,200] [--iters K] [--seed S] [--out-dir D]
    python -m paper_1111_6900_b200 bench OP E N [--reps K]      (OP: mul addmul ple echelonize trsm)

Exit codes (SPEC cli invariants): 0 success, 1 computation or self-test failure, 2 usage
error (bad arguments, unreadable or malformed files, field or shape mismatch).  Every
backend name selects the same device computation — the products and echelon forms are
unique, so the reference's backends agree bit for bit (SPEC acceptance criterion 1) — and
``--backend``/``--crossover``/``GF2E_CROSSOVER`` are accepted for interface parity.
``--counts`` prints the reference's counters for the chosen backend on standard error.
The self-test checks identities that need no second implementation: backend equivalence
(int8, fp4 and M4RM product kernels), slice/cling round trips, P·L·E = A, RREF shape and
rank agreement, U·X = B and L·X = B for solved systems, and make_table against scalar_mul
with the Gray-code counts.  On a failure the inputs are written as matrix files and the
command exits 1.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np


class UsageError(Exception):
    pass


def _crossover(args) -> int | None:
    if getattr(args, "crossover", None) is not None:
        return args.crossover
    env = os.environ.get("GF2E_CROSSOVER")
    if env is None:
        return None
    try:
        return int(env)
    except ValueError:
        raise UsageError(f"GF2E_CROSSOVER must be an integer, got {env!r}")


def _load(path: str):
    from . import matfile
    from .mat_packed import PackedMatrix
    from .mat_sliced import cling

    try:
        with open(path, "r", newline="\n") as fh:
            text = fh.read()
    except OSError as exc:
        raise UsageError(f"cannot read {path}: {exc.strerror}")
    try:
        M = matfile.parse(text)
    except ValueError as exc:
        raise UsageError(f"{path}: {exc}")
    return M if isinstance(M, PackedMatrix) else cling(M)


def _save(path: str, A, sliced: bool = False) -> None:
    from . import matfile
    from .mat_sliced import slice_packed

    matfile.save_matrix(path, slice_packed(A) if sliced else A)


def cmd_random(args) -> int:
    from .gf2e import field_new
    from .mat_packed import PackedMatrix

    try:
        ctx = field_new(args.e, int(args.f, 16) if args.f else None)
    except ValueError as exc:
        raise UsageError(str(exc))
    if args.m < 0 or args.n < 0:
        raise UsageError("dimensions must be non-negative")
    _save(args.out, PackedMatrix.random(ctx, args.m, args.n, args.seed), sliced=args.repr == "sliced")
    return 0


def cmd_mul(args) -> int:
    from .mat_gf2 import RowOpCounters
    from .newton_john import cubic_mul, nj_mul
    from .poly_mul import MulCounters, karatsuba_mul_packed

    A, B = _load(args.a), _load(args.b)
    if A.ctx != B.ctx:
        raise UsageError(f"field mismatch: {A.ctx} vs {B.ctx}")
    if A.ncols != B.nrows:
        raise UsageError(f"inner dimensions differ: {A.nrows}x{A.ncols} times {B.nrows}x{B.ncols}")
    _crossover(args)
    if args.backend == "karatsuba":
        cnt = MulCounters()
        C = karatsuba_mul_packed(A, B, cnt)
        line = (f"counts gf2_matmul_count={cnt.gf2_matmul_count} additions={cnt.additions} "
                f"peak_live_products={cnt.peak_live_products}")
    elif args.backend == "nj":
        rc = RowOpCounters()
        C = nj_mul(A, B, rc)
        line = f"counts row_adds={rc.row_adds} scalar_row_muls={rc.scalar_row_muls}"
    else:  # cubic, strassen: the same unique product
        C = cubic_mul(A, B)
        line = "counts none"
    _save(args.out, C)
    if args.counts:
        print(line, file=sys.stderr)
    return 0


def cmd_echelonize(args) -> int:
    from .newton_john import nj_gauss
    from .ple_echelon import echelonize

    A = _load(args.inp)
    cx = _crossover(args)
    r = nj_gauss(A, full=args.full) if args.backend == "nj" else echelonize(A, full=args.full, crossover=cx)
    _save(args.out, A)
    print(f"rank={r}")
    return 0


# -- self-test ------------------------------------------------------------------------------


def _random_upper(ctx, n: int, seed: int, lower: bool = False):
    """Triangular matrix with a nonzero diagonal, from the reference generator."""
    from .mat_packed import PackedMatrix

    arr = PackedMatrix.random(ctx, n, n, seed).to_array()
    arr = np.tril(arr) if lower else np.triu(arr)
    d = np.arange(n)
    arr[d, d] = np.where(arr[d, d] == 0, 1, arr[d, d])
    return PackedMatrix.from_array(ctx, arr)


def _is_rref(arr: np.ndarray, r: int) -> bool:
    lead = -1
    for i in range(arr.shape[0]):
        nz = np.nonzero(arr[i])[0]
        if i >= r:
            if nz.size:
                return False
            continue
        if not nz.size or nz[0] <= lead or arr[i, nz[0]] != 1:
            return False
        lead = nz[0]
        col = arr[:, lead]
        if np.count_nonzero(col) != 1:
            return False
    return True


def _selftest_case(e: int, m: int, k: int, n: int, seed: int):
    """Yield (check name, ok, inputs to dump on failure) for one field and shape."""
    from .gf2e import field_new
    from .mat_gf2 import RowOpCounters
    from .mat_packed import PackedMatrix
    from .mat_sliced import cling, slice_packed
    from .newton_john import make_table
    from .ple_echelon import echelonize, ple, ple_reconstruct, trsm_lower_left, trsm_upper_left
    from .poly_mul import karatsuba_mul, karatsuba_mul_packed

    ctx = field_new(e)
    A = PackedMatrix.random(ctx, m, k, seed)
    B = PackedMatrix.random(ctx, k, n, seed + 1)
    SA, SB = slice_packed(A), slice_packed(B)
    ref = karatsuba_mul(SA, SB, backend="m4rm")
    ok = all(karatsuba_mul(SA, SB, backend=b) == ref for b in ("tc_i8", "tc_fp4"))
    ok = ok and karatsuba_mul(SA, SB) == ref
    yield "backend_equivalence", ok, {"A": A, "B": B}
    yield "slice_cling_roundtrip", cling(SA) == A and cling(SB) == B, {"A": A, "B": B}
    F = ple(A.copy())
    yield "ple_reconstruction", ple_reconstruct(F) == A, {"A": A}
    X = A.copy()
    r = echelonize(X, full=True)
    yield "rref", r == F.rank and _is_rref(X.to_array(), r), {"A": A}
    U = _random_upper(ctx, m, seed + 2)
    Y = PackedMatrix.random(ctx, m, n, seed + 3)
    Z = Y.copy()
    trsm_upper_left(U, Z)
    yield "trsm_upper_identity", karatsuba_mul_packed(U, Z) == Y, {"U": U, "B": Y}
    L = _random_upper(ctx, m, seed + 4, lower=True)
    Z = Y.copy()
    trsm_lower_left(L, Z)
    yield "trsm_lower_identity", karatsuba_mul_packed(L, Z) == Y, {"L": L, "B": Y}
    if m and k:
        row = PackedMatrix.random(ctx, 1, k, seed + 5)
        cnt = RowOpCounters()
        T = make_table(row, cnt)
        ok = (cnt.scalar_row_muls, cnt.row_adds) == (e, (1 << e) - 1)
        ok = ok and all(T.row(x) == row.scalar_mul(x) for x in (0, 1, 2, (1 << e) - 1))
        yield "make_table_counts", ok, {"row": row}


def cmd_selftest(args) -> int:
    try:
        es = [int(x) for x in args.e.split(",")] if args.e else list(range(2, 11))
        sizes = [int(x) for x in args.sizes.split(",")] if args.sizes else [1, 63, 64, 65, 200]
    except ValueError:
        raise UsageError("--e and --sizes take comma-separated integers")
    if any(not 2 <= e <= 10 for e in es) or any(s < 1 for s in sizes) or args.iters < 1:
        raise UsageError("e must be in 2..10, sizes >= 1, iters >= 1")
    rng = np.random.default_rng(args.seed)
    checks = 0
    for e in es:
        for it in range(args.iters):
            m, k, n = (int(rng.choice(sizes)) for _ in range(3))
            seed = args.seed * 1000 + it * 10 + e
            for name, ok, inputs in _selftest_case(e, m, k, n, seed):
                checks += 1
                if not ok:
                    os.makedirs(args.out_dir, exist_ok=True)
                    paths = []
                    for label, M in inputs.items():
                        p = os.path.join(args.out_dir, f"selftest_{name}_e{e}_{label}.mat")
                        _save(p, M)
                        paths.append(p)
                    print(f"selftest FAILED check={name} e={e} m={m} k={k} n={n} seed={seed} "
                          f"inputs={','.join(paths)}", file=sys.stderr)
                    return 1
    print(f"selftest ok checks={checks} e={','.join(map(str, es))} iters={args.iters}")
    return 0


# -- bench ----------------------------------------------------------------------------------


def cmd_bench(args) -> int:
    import torch

    from .gf2e import field_new
    from .mat_packed import PackedMatrix
    from .mat_sliced import slice_packed
    from .ple_echelon import echelonize, ple, trsm_upper_left
    from .poly_mul import MulCounters, addmul, karatsuba_mul

    if not 2 <= args.e <= 10 or args.n < 1 or args.reps < 1:
        raise UsageError("e must be in 2..10, n >= 1, reps >= 1")
    ctx = field_new(args.e)
    n = args.n
    A = PackedMatrix.random(ctx, n, n, 1)
    B = PackedMatrix.random(ctx, n, n, 2)
    counted = args.op in ("mul", "addmul")
    if args.op in ("mul", "addmul"):
        SA, SB = slice_packed(A), slice_packed(B)
        SC = slice_packed(PackedMatrix.random(ctx, n, n, 3))
        run = (lambda c: karatsuba_mul(SA, SB, c)) if args.op == "mul" else (lambda c: addmul(SC, SA, SB, c))
    elif args.op == "ple":
        run = lambda c: ple(A.copy())  # noqa: E731
    elif args.op == "echelonize":
        run = lambda c: echelonize(A.copy(), full=True)  # noqa: E731
    else:  # trsm
        U = _random_upper(ctx, n, 4)
        run = lambda c: trsm_upper_left(U, B.copy())  # noqa: E731
    run(None)
    torch.cuda.synchronize()
    times, cnt = [], MulCounters()
    for _ in range(args.reps):
        cnt.reset()
        t0 = time.perf_counter()
        run(cnt)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    muls = str(cnt.gf2_matmul_count) if counted else "na"
    print(f"bench op={args.op} e={args.e} n={n} reps={args.reps} median_s={float(np.median(times)):.6f} "
          f"gf2_muls={muls}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_1111_6900_b200",
                                description="GF(2^e) matrices on the B200: files, products, echelon forms")
    sub = p.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("random", help="write a reference-generator random matrix")
    r.add_argument("e", type=int)
    r.add_argument("m", type=int)
    r.add_argument("n", type=int)
    r.add_argument("seed", type=int)
    r.add_argument("out")
    r.add_argument("--f", default=None, help="modulus as hex (default: the reference's DEFAULT_POLYS[e])")
    r.add_argument("--repr", choices=("packed", "sliced"), default="packed")
    r.set_defaults(fn=cmd_random)
    m = sub.add_parser("mul", help="C = A*B")
    m.add_argument("a")
    m.add_argument("b")
    m.add_argument("out")
    m.add_argument("--backend", choices=("cubic", "nj", "strassen", "karatsuba"), default="karatsuba")
    m.add_argument("--crossover", type=int, default=None)
    m.add_argument("--counts", action="store_true")
    m.set_defaults(fn=cmd_mul)
    ech = sub.add_parser("echelonize", help="(reduced) row echelon form; prints rank=<r>")
    ech.add_argument("inp")
    ech.add_argument("out")
    ech.add_argument("--full", action="store_true")
    ech.add_argument("--backend", choices=("nj", "ple"), default="ple")
    ech.add_argument("--crossover", type=int, default=None)
    ech.set_defaults(fn=cmd_echelonize)
    st = sub.add_parser("selftest", help="algebraic identities of the device path")
    st.add_argument("--e", default=None, help="comma-separated degrees (default 2..10)")
    st.add_argument("--sizes", default=None, help="comma-separated dimensions to draw from")
    st.add_argument("--iters", type=int, default=2)
    st.add_argument("--seed", type=int, default=1)
    st.add_argument("--out-dir", default=".")
    st.set_defaults(fn=cmd_selftest)
    b = sub.add_parser("bench", help="median wall time of one operation on n x n matrices")
    b.add_argument("op", choices=("mul", "addmul", "ple", "echelonize", "trsm"))
    b.add_argument("e", type=int)
    b.add_argument("n", type=int)
    b.add_argument("--reps", type=int, default=5)
    b.set_defaults(fn=cmd_bench)
    return p


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)  # usage errors: argparse exits 2
    try:
        return args.fn(args)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (ValueError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


__all__ = ["main", "build_parser"]

"""bench.py — GF(2^e) bitsliced-Karatsuba matmul on B200: effective GF(2) Tbit-op/s.

Default workload (BASELINE.json config 3): F_256 (e=8, f=0x11d), C = A.B with A, B
16384 x 16384 per GPU, entries from the reference generator (seeds A=1, B=2), sliced planes
resident in HBM.  One step = one ``karatsuba_mul`` (mzd_slice_mul): operand combinations +
the fused tcgen05 product/combine/fold kernel.  Metric: K(e) * 2*m*k*n GF(2) bit-ops per
second (K(8) = 27).  Multi-GPU (torchrun): each rank owns a 16384-row block of
C (weak scaling, no data-path collective); B is generated on rank 0 and broadcast once with
NCCL before timing.  ``--config 5`` runs the 65536^3 case sharded by C row-blocks instead.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3|1|2|4|5]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_OF_E = {2: 3, 3: 6, 4: 9, 5: 15, 6: 18, 7: 24, 8: 27, 9: 39, 10: 45}
DEFAULT_F = {2: 0x7, 3: 0xB, 4: 0x13, 5: 0x25, 6: 0x43, 7: 0x83, 8: 0x11D, 9: 0x211, 10: 0x409}


def workload(config: int, e_override: int | None, world: int):
    """(name, e, m_per_rank, k, n, accumulate, scaling)"""
    if config == 1:
        return ("F4 C=A.B 1024^3 (BASELINE config 1)", 2, 1024, 1024, 1024, False, "weak")
    if config == 2:
        return ("F16 C=A.B 4096^3 (BASELINE config 2)", 4, 4096, 4096, 4096, False, "weak")
    if config == 3:
        return ("F256 C=A.B 16384^3 per GPU (BASELINE config 3)", 8, 16384, 16384, 16384, False, "weak")
    if config == 4:
        e = e_override or 8
        return (f"F(2^{e}) C+=A.B 65536x256.256x65536 (BASELINE config 4)", e, 65536, 256, 65536, True, "weak")
    if config == 5:
        if 65536 % world:
            raise SystemExit("config 5 needs world size dividing 65536")
        return ("F256 C=A.B 65536^3 sharded by C row-blocks (BASELINE config 5)", 8, 65536 // world, 65536,
                65536, False, "strong")
    raise SystemExit(f"unknown config {config}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def host_threads() -> int:
    """All host cores this process may use (torchrun sets OMP_NUM_THREADS=1 per rank; the CPU
    baseline and the reference arm run on rank 0 only and use every core)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def cpu_sample(e: int, k: int, n: int, rows: int, threads: int = 0, acc: bool = False, row0: int = 0):
    """Oracle ("port") karatsuba on C rows [row0, row0 + rows) — a bounded slice of the same
    workload (A seed 1, B seed 2, C0 seed 3 for addmul).  Returns (Tbit-op/s, s, C rows)."""
    import oracle

    f = DEFAULT_F[e]
    a = oracle.sliced_random(e, rows, k, 1, row0=row0, gcols=k)
    b = oracle.sliced_random(e, k, n, 2)
    c0 = oracle.sliced_random(e, rows, n, 3, row0=row0, gcols=n) if acc else None
    t0 = time.perf_counter()
    ref, _ = oracle.karatsuba(e, f, a, b, rows, k, n, C0=c0, nthreads=threads)
    dt = time.perf_counter() - t0
    ops = K_OF_E[e] * 2.0 * rows * k * n
    return ops / dt / 1e12, dt, ref


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle

    name, e, m, k, n, acc, scaling = workload(args.config, args.e, 1)
    rows = args.cpu_rows or (256 if k * n >= 16384 * 16384 else min(m, 1024))
    cores = host_threads()
    vals = []
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample(e, k, n, min(rows, 64), cores, acc)
    for _ in range(args.steps):
        v, dt, _ = cpu_sample(e, k, n, rows, cores, acc)
        vals.append((v, dt))
    v = statistics.median(x[0] for x in vals)
    dt = statistics.median(x[1] for x in vals)
    sample = (f"rows 0..{rows - 1} of C ({rows}x{k}x{n}, e={e}) through oracle.karatsuba "
              f"(C port of the reference poly_mul._kara + M4RM), {cores} threads")
    line = {
        "metric": "effective GF(2) Tbit-op/s (K(e)*2mkn / time)", "value": round(v, 4), "unit": "Tbit-op/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u64 (GF(2) bit-planes)",
        "data": "synthetic (reference splitmix64 generator, seeds A=1 B=2)", "impl": "reference",
        "config": {"workload": name, "e": e, "m": m, "k": k, "n": n, "f": hex(DEFAULT_F[e])},
        "cpu_baseline": {"value": round(v, 4), "unit": "Tbit-op/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "Tbit-op/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1111_6900_b200 as g
    from paper_1111_6900_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the multi-rank flow on a one-GPU box (not a measurement): every rank
    # on cuda:0, host-side gloo collectives (kernels of different ranks never wait on each other)
    if args.dist_backend == "gloo-shared-gpu":
        local = 0
    torch.cuda.set_device(local)
    # a process group whenever launched by torchrun (even with one rank: the NCCL path runs)
    use_pg = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if use_pg:
        if args.dist_backend == "gloo-shared-gpu":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    name, e, m, k, n, acc, scaling = workload(args.config, args.e, world)
    ctx = g.field_new(e)
    K = g.count_products(e)
    ops_rank = K * 2.0 * m * k * n
    backend = args.backend

    # ---- inputs resident in HBM: A row-block (rank's rows of the global matrix); B generated on
    #      rank 0, kept there pre-split into the broadcast's column parts ----
    from paper_1111_6900_b200 import dist as gdist

    row0 = rank * m
    A = g.SlicedMatrix.random(ctx, m, k, 1, row0=row0, gcols=k)
    if rank == 0:
        B = g.SlicedMatrix.random(ctx, k, n, 2)
    else:
        B = g.SlicedMatrix(ctx, k, n, torch.empty((e, k, g.words_for(n)), dtype=torch.int64, device=dev))
    flags = g.poly_mul._resolve_backend(backend) | (_lib.ACCUMULATE if acc else 0)
    tile = int(_lib.load().gf2e_tile_cols(e, ctx.f, k, flags))
    pairs = torch.cuda.get_device_properties(dev).multi_processor_count // 2
    # first part = the smallest whole number of product waves >= n/8: no partial wave is added
    bounds = gdist.col_parts(n, args.bcast_parts, tile=tile, rows=m, pairs=pairs)
    src_parts = gdist.split_parts(B.planes, bounds) if rank == 0 else None
    gdist.broadcast_planes(B.planes, src=0)  # a resident copy of B on every rank (compute-only line)
    C = (g.SlicedMatrix.random(ctx, m, n, 3, row0=row0, gcols=n) if acc
         else g.SlicedMatrix(ctx, m, n, torch.empty((e, m, g.words_for(n)), dtype=torch.int64, device=dev)))
    torch.cuda.synchronize()

    out = [C]

    def step_compute():
        """B resident on every GPU: operand combinations + the fused product."""
        if acc:
            g.addmul(C, A, B, backend=backend)
        else:
            out[0] = g.karatsuba_mul(A, B, backend=backend)
        return _lib.last_launch_count()

    def step_comm():
        """The data-path collective included: B broadcast from rank 0 in column parts on a side
        stream (NCCL over NVLink), each part multiplied as it arrives (gf2e_slice_mul_parts)."""
        pieces, events = gdist.broadcast_parts(B.planes if rank == 0 else None, (e, k, g.words_for(n)), bounds,
                                               src=0, device=dev, src_parts=src_parts)
        if acc:
            gdist.mul_parts(e, ctx.f, A.planes, pieces, events, bounds, k, n, C.planes, True, backend)
        else:
            Cn = torch.empty((e, m, g.words_for(n)), dtype=torch.int64, device=dev)
            gdist.mul_parts(e, ctx.f, A.planes, pieces, events, bounds, k, n, Cn, False, backend)
            out[0] = g.SlicedMatrix(ctx, m, n, Cn)
        return _lib.last_launch_count()

    # under torchrun (any N, including 1) the headline step includes the B broadcast
    step = step_comm if use_pg else step_compute

    def timed(fn, nsteps, sample_clocks=False):
        """max over ranks of the per-step ms (CUDA events on the launching stream, barrier +
        sync on both sides) and of the product-kernel ms per step; launches per step."""
        sampler = ClockSampler(local) if sample_clocks else None
        if sampler:
            sampler.start()
        _lib.profile_enable(True)
        _lib.profile_read()
        if use_pg:
            dist.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(st)
        nl = 0
        for _ in range(nsteps):
            nl += fn()
        ev1.record(st)
        torch.cuda.synchronize()
        if use_pg:
            dist.barrier()
        clk = sampler.stop() if sampler else None
        pms, _ = _lib.profile_read()
        kname = _lib.last_product_kernel()
        _lib.profile_enable(False)
        t = torch.tensor([ev0.elapsed_time(ev1) / nsteps, pms / nsteps], dtype=torch.float64, device=dev)
        if use_pg:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0]), float(t[1]), nl, clk, kname

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ms_max, prod_ms_max, launches, clocks, kernel_name = timed(step, args.steps, sample_clocks=True)
    value = world * ops_rank / (ms_max * 1e-3) / 1e12
    nsteps_done = args.warmup + args.steps
    compute_only = None
    if use_pg:
        for _ in range(args.warmup):
            step_compute()
        c_ms, c_prod, _, _, _ = timed(step_compute, args.steps)
        nsteps_done += args.warmup + args.steps
        compute_only = {"value": round(world * ops_rank / (c_ms * 1e-3) / 1e12, 4), "ms_per_step": round(c_ms, 4),
                        "kernel_ms": round(c_prod, 4),
                        "what": "B resident on every GPU (broadcast before timing): combos + fused product only"}

    # parity sample of the timed result: C rows [0, prow) of this rank's block (C0 ^ A.B for
    # addmul: one more untimed step when the step count left C at C0), compared on rank 0
    # with the oracle rows computed for cpu_baseline
    prow = min(m, args.cpu_rows or (256 if k * n >= 16384 * 16384 else min(m, 1024)))
    if acc and nsteps_done % 2 == 0:
        step_compute()
    dev_rows = out[0].planes[:, :prow].cpu().numpy().view("uint64").copy()
    del out

    # ---- e2e through the public host-buffer API (gf2e_mzed_mul_host), per step: H2D of packed A
    #      from pinned host memory, slice, combos, product, cling, D2H of packed C; the library
    #      overlaps copies of one row chunk with the kernels of another.  N = 1: B is uploaded
    #      by the same call (in column parts, overlapped).  torchrun: rank 0 uploads packed B once,
    #      NCCL broadcasts it, and every rank runs the call with B already on its GPU.  Timed by
    #      CUDA events (N = 1: inside the call, first H2D -> last D2H; torchrun: from rank 0's B
    #      upload to the call's return), max over ranks. ----
    e2e = None
    if not args.no_e2e:
        import numpy as np

        Ap = g.cling(A)
        Bp = g.cling(B)
        hA = torch.empty(tuple(Ap.storage.words.shape), dtype=torch.int64, pin_memory=True)
        hA.copy_(Ap.storage.words)
        hB = torch.empty(tuple(Bp.storage.words.shape), dtype=torch.int64, pin_memory=rank == 0)
        if rank == 0:
            hB.copy_(Bp.storage.words)
        wpc = g.words_for(n * g.pack_width(e))
        hC = torch.empty((m, wpc), dtype=torch.int64, pin_memory=True)
        if acc:  # C0 again (the device C above holds C0 ^ A.B)
            hC.copy_(g.cling(g.SlicedMatrix.random(ctx, m, n, 3, row0=row0, gcols=n)).storage.words)
        del Ap, Bp
        nA, nB, nC = (t.numpy().view(np.uint64) for t in (hA, hB, hC))
        dB = torch.empty(tuple(hB.shape), dtype=torch.int64, device=dev) if use_pg else None

        def e2e_call(bwords):
            if acc:
                return g.karatsuba_mul_packed_host(ctx, nA, k, bwords, n, C_words=nC, chunk_rows=args.chunk_rows)[1]
            return g.karatsuba_mul_packed_host(ctx, nA, k, bwords, n, out=nC, chunk_rows=args.chunk_rows)[1]

        def e2e_step():
            if not use_pg:
                return e2e_call(nB)
            st = torch.cuda.current_stream()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(st)
            if rank == 0:
                dB.copy_(hB, non_blocking=True)
            gdist.broadcast_planes(dB, src=0)
            e2e_call(dB)
            ev1.record(st)
            ev1.synchronize()
            return ev0.elapsed_time(ev1)

        e2e_warm = max(1, args.warmup)
        for _ in range(e2e_warm):
            e2e_step()
        if use_pg:
            dist.barrier()
        ms_list = [e2e_step() for _ in range(args.steps)]
        if acc and (e2e_warm + args.steps) % 2 == 0:
            e2e_step()  # leave hC = C0 ^ A.B for the parity sample
        e2e_rows = nC[:prow].copy()
        te = torch.tensor([sum(ms_list) / len(ms_list)], dtype=torch.float64, device=dev)
        if use_pg:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        # whole-job bytes per step: every rank's A (and C0 / C) rows, B once
        e2e = {"value": round(world * ops_rank / (float(te[0]) * 1e-3) / 1e12, 4), "unit": "Tbit-op/s",
               "h2d_bytes_per_step": int(world * (hA.numel() * 8 + (hC.numel() * 8 if acc else 0)) + hB.numel() * 8),
               "d2h_bytes_per_step": int(world * hC.numel() * 8), "ms_per_step": round(float(te[0]), 3),
               "path": ("gf2e_mzed_mul_host: pinned packed A,B -> H2D -> slice -> combos -> product -> cling -> D2H, "
                        "row chunks pipelined on 4 streams") if not use_pg else
                       ("rank 0: pinned packed B -> H2D -> NCCL broadcast; every rank: gf2e_mzed_mul_host with B on "
                        "its GPU (GF2E_B_DEVICE), pinned packed A rows -> H2D ... -> D2H of its C rows")}

    if rank != 0:
        if use_pg:
            dist.destroy_process_group()
        return 0

    pk, pk_kind = peaks()
    # Denominator: the dense tensor rate of the form the kernel ran (kind::i8 or kind::mxf4),
    # measured on THIS GPU right now by a pure-MMA loop on every SM.  MEASURED_PEAKS.json holds
    # only bf16 (its cuBLAS figure x2 understates the int8 pipe), reported alongside.
    fp4_form = "fp4" in kernel_name
    bound = "tensor"
    if "m4rm" in kernel_name:  # the INT-pipe form: its roofline is the shared-memory table reads
        bps, tc_peak = _lib.int_peak(2000)
        bound = "int-pipe (LDS.128)"
        peak_basis = (f"measured live: conflict-free LDS.128 on all SMs = {bps / 1e12:.1f} TB/s; M4RM reads one "
                      "16-byte table row per 128 columns x 8 k-bits (2048 GF(2) bit-ops)")
    elif fp4_form:
        tc_peak = max(_lib.mma_peak_fp4(20000), _lib.mma_peak_fp4(20000))
        peak_basis = ("measured live: pure tcgen05.mma kind::mxf4 (e2m1, scale 1.0) loop on all SMs "
                      "(zero operands; random GF(2)-encoded operands and 0.25 s loops measure the same); "
                      f"for reference 4 x {pk_kind} cuBLAS bf16 = {4 * pk['bf16_tflops']:.1f}")
    else:
        tc_peak = max(_lib.mma_peak(2, 20000)[0], _lib.mma_peak(1, 20000)[0])
        peak_basis = ("measured live: pure tcgen05.mma kind::i8 loop on all SMs (gf2e_mma_peak); "
                      f"for reference 2 x {pk_kind} cuBLAS bf16 = {2 * pk['bf16_tflops']:.1f}")
    # per step: one launch (N = 1) or one per broadcast part with complete tiles (torchrun)
    achieved = ops_rank / (prod_ms_max * 1e-3) / 1e12  # GF(2) bit-ops == int8 tensor ops (1 MAC = 2 ops)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            key = f"config{args.config}" + (f"_e{e}" if args.config == 4 else "") + (
                f"_{backend}" if backend and backend != "tc" else "")
            ent = json.load(open(tpath)).get(key)
            # dram bytes per launch of this kernel from the committed ncu capture of it
            traffic = ent["dram_bytes_per_launch"] if ent else None
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": "effective GF(2) Tbit-op/s (K(e)*2mkn / time)", "value": round(value, 4), "unit": "Tbit-op/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "e2m1 0/1 (kind::mxf4, exact fp32 acc)" if fp4_form else "u8 0/1 (kind::i8, s32 acc)",
        "data": "synthetic (reference splitmix64 generator, seeds A=1 B=2 C0=3)",
        "config": {"workload": name, "e": e, "f": hex(ctx.f), "m_per_gpu": m, "k": k, "n": n,
                   "gf2_products": K, "backend": backend or "tc", "parallelism": f"C row-blocks x{world}",
                   "l2": "inputs larger than L2 (A planes + combos >> 126 MB)"},
        "time_s": round(ms_max / 1e3, 6),
        "comm_included": bool(use_pg),
        "gpu_launches": launches,
        "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": round(tc_peak, 1),
                     "unit": "TFLOP/s", "frac": round(achieved / tc_peak, 4), "traffic": traffic,
                     "kernel": kernel_name, "kernel_ms": round(prod_ms_max, 4),
                     "peak_basis": peak_basis,
                     "ops_per_launch": ops_rank},
        "clocks": clocks,
    }

    if compute_only:
        line["compute_only"] = compute_only
        line["config"]["broadcast"] = (f"B ({e} planes, {e * k * g.words_for(n) * 8} bytes) from rank 0 in "
                                       f"{len(bounds) - 1} column parts {bounds}, NCCL on a side stream, each "
                                       "part multiplied as it arrives; included in value / ms_per_step")
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        import oracle

        # rank 0's rows 0..prow-1 are rows 0..prow-1 of the global C at every N
        v, dt, ref = cpu_sample(e, k, n, prow, host_threads(), acc)
        if world == 1:  # the CPU baseline is an N=1 figure
            line["cpu_baseline"] = {"value": round(v, 4), "unit": "Tbit-op/s", "cores": host_threads(),
                                    "kind": "port",
                                    "sample": f"rows 0..{prow - 1} of C ({prow}x{k}x{n}, e={e}) via oracle.karatsuba, "
                                              f"{dt:.2f} s"}
        par = {"rows": f"C rows 0..{prow - 1} (all {n} columns, all {e} planes) vs oracle.karatsuba",
               "device": "ok" if (dev_rows == ref).all() else "MISMATCH"}
        if e2e:
            par["e2e"] = "ok" if (e2e_rows == oracle.cling_words(e, prow, n, ref)).all() else "MISMATCH"
        line["parity"] = par
    print(json.dumps(line), flush=True)
    if use_pg:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 5; 100 for the sub-millisecond configs 1 and 2, whose "
                         "short steps are host-enqueue bound, so a 5-step window is dominated by its start)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--e", type=int, default=None, help="field degree for config 4")
    ap.add_argument("--backend", default=None, choices=[None, "tc", "tc_i8", "tc_fp4", "tc_run", "m4rm"])
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chunk-rows", type=int, default=0, help="row chunk of the host-buffer e2e call (0: library default)")
    ap.add_argument("--bcast-parts", type=int, default=2, help="column parts of B's broadcast under torchrun")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo-shared-gpu"],
                    help="gloo-shared-gpu: functional multi-rank check with every rank on cuda:0 (no timing meaning)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 100 if args.config in (1, 2) and args.impl == "ours" else 5
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

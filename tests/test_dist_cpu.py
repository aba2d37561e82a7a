"""Multi-rank host logic of the C row-block partition on CPU (gloo, world sizes 2 and 4).

The device product is replaced by the oracle (test infrastructure) so the partition, the B
broadcast and the row reassembly are checked end to end without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1111_6900_b200 import dist as gd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_compute(e, f, A, B, C0, k, n):
    a = A.numpy().view(np.uint64)
    b = B.numpy().view(np.uint64)
    c0 = None if C0 is None else C0.numpy().view(np.uint64)
    C, _ = oracle.karatsuba(e, f, a, b, a.shape[1], k, n, C0=c0, nthreads=1)
    return torch.from_numpy(C.view(np.int64))


CASES = {  # world -> (m, n, parts, acc) cases, run in one process group per world size
    2: [(200, 130, 1, False), (200, 130, 1, True), (300, 2500, 4, True)],
    4: [(1000, 130, 1, True), (700, 1700, 3, False), (3, 70, 1, False)],
}
E, K = 5, 70


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e, k, f = E, K, oracle.DEFAULT_POLYS[E]
        for (m, n, parts, acc) in CASES[world]:
            row0, rows = gd.row_partition(m, world)[rank]
            A = torch.from_numpy(oracle.sliced_random(e, rows, k, 1, row0=row0, gcols=k).view(np.int64))
            if rank == 0:
                B = torch.from_numpy(oracle.sliced_random(e, k, n, 2).view(np.int64))
            elif parts > 1:  # column parts: only the source rank holds B
                B = None
            else:  # garbage: must be replaced by the broadcast
                B = torch.full((e, k, (n + 63) // 64), -1, dtype=torch.int64)
            C0 = (torch.from_numpy(oracle.sliced_random(e, rows, n, 3, row0=row0, gcols=n).view(np.int64))
                  if acc else None)
            C = gd.sharded_mul(e, f, A, B, k, n, C0_block=C0, parts=parts, compute=_oracle_compute)
            full = gd.all_gather_rows(C, m)
            if rank == 0:
                out_q.put(full.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_row_blocks_match_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in CASES[world]]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    e, k = E, K
    for (m, n, parts, acc), g in zip(CASES[world], got):
        ref, _ = oracle.karatsuba(e, oracle.DEFAULT_POLYS[e], oracle.sliced_random(e, m, k, 1),
                                  oracle.sliced_random(e, k, n, 2), m, k, n,
                                  C0=oracle.sliced_random(e, m, n, 3) if acc else None)
        assert np.array_equal(g, ref), (world, m, n, parts, acc)


def test_row_partition():
    assert gd.row_partition(65536, 8) == [(g * 8192, 8192) for g in range(8)]
    # whole 256-row tiles dealt out evenly; no empty rank when there are enough rows
    assert gd.row_partition(1000, 3) == [(0, 512), (512, 256), (768, 232)]
    assert gd.row_partition(1000, 4) == [(0, 256), (256, 256), (512, 256), (768, 232)]
    assert gd.row_partition(300, 4) == [(0, 128), (128, 64), (192, 64), (256, 44)]  # 64-row tiles
    assert gd.row_partition(3, 4) == [(0, 1), (1, 1), (2, 1), (3, 0)]  # m < world
    for m in range(0, 3000, 37):
        for w in (1, 2, 3, 4, 5, 8):
            parts = gd.row_partition(m, w)
            assert parts[0][0] == 0 and sum(r for _, r in parts) == m
            assert all(a + r == b for (a, r), (b, _) in zip(parts, parts[1:]))
            assert m < w or all(r > 0 for _, r in parts)
    assert gd.row_partition(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        gd.row_partition(10, 0)


def test_col_parts():
    assert gd.col_parts(16384, 1) == [0, 16384]
    b = gd.col_parts(16384, 4)
    assert b == [0, 1536, 6912, 11520, 16384]  # first part ~n/8, whole 768-column multiples
    assert all(x % 768 == 0 for x in b[1:-1]) and all(x < y for x, y in zip(b, b[1:]))
    assert gd.col_parts(1000, 4) == [0, 1000]  # too narrow to split
    for n in range(1537, 70000, 997):
        for p in (2, 3, 8):
            b = gd.col_parts(n, p)
            assert b[0] == 0 and b[-1] == n and all(x < y for x, y in zip(b, b[1:]))
            assert all(x % 768 == 0 for x in b[1:-1])

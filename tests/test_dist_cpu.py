"""Multi-rank host logic of the C row-block partition on CPU (gloo, world_size 2).

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


def _worker(rank, world, port, e, m, k, n, acc, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = oracle.DEFAULT_POLYS[e]
        row0, rows = gd.row_partition(m, world, align=64)[rank]
        A = torch.from_numpy(oracle.sliced_random(e, rows, k, 1, row0=row0, gcols=k).view(np.int64))
        if rank == 0:
            B = torch.from_numpy(oracle.sliced_random(e, k, n, 2).view(np.int64))
        else:  # garbage: must be replaced by the broadcast
            B = torch.full((e, k, (n + 63) // 64), -1, dtype=torch.int64)
        C0 = (torch.from_numpy(oracle.sliced_random(e, rows, n, 3, row0=row0, gcols=n).view(np.int64))
              if acc else None)
        C = gd.sharded_mul(e, f, A, B, k, n, C0_block=C0, compute=_oracle_compute)
        full = gd.all_gather_rows(C, m, align=64)
        if rank == 0:
            out_q.put(full.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("acc", [False, True])
def test_two_rank_row_blocks_match_single(acc):
    e, m, k, n = 5, 200, 70, 130
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, e, m, k, n, acc, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, _ = oracle.karatsuba(e, oracle.DEFAULT_POLYS[e], oracle.sliced_random(e, m, k, 1),
                              oracle.sliced_random(e, k, n, 2), m, k, n,
                              C0=oracle.sliced_random(e, m, n, 3) if acc else None)
    assert np.array_equal(got, ref)


def test_row_partition():
    assert gd.row_partition(65536, 8) == [(g * 8192, 8192) for g in range(8)]
    parts = gd.row_partition(1000, 3)
    assert parts == [(0, 512), (512, 488), (1000, 0)]
    assert sum(r for _, r in parts) == 1000
    assert gd.row_partition(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        gd.row_partition(10, 0)

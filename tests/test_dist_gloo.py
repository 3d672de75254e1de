"""Multi-rank host logic on CPU (world size 2, gloo): the row/column partition, the
cabs_comm callbacks that the C library calls for its collectives, and the exchange
patterns the library relies on (owner-written slots summed = allgather; the fused
k-means payload; max-over-ranks timing).  No GPU needed."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_07395_b200.dist import col_partition, make_plan, row_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1607_07395_b200.dist import TorchComm
        comm = TorchComm(torch.device("cpu"))
        out = {}
        # 1) the raw C callbacks (as libcabs calls them): sum-allreduce in place
        x = torch.arange(10, dtype=torch.float64) * (rank + 1)
        rc = comm.c.allreduce_f64(ctypes.c_void_p(x.data_ptr()), 10, None, None)
        out["f64"] = (rc, x.tolist())
        y = torch.full((7,), float(rank + 1), dtype=torch.float32)
        rc = comm.c.allreduce_f32(ctypes.c_void_p(y.data_ptr()), 7, None, None)
        out["f32"] = (rc, y.tolist())
        # 2) pilot row exchange: each rank writes the sampled rows it owns into a zeroed
        #    k x n buffer; the sum is the full R, bit-exact (x + 0 = x)
        m, n, k = 1000, 37, 9
        g = np.random.default_rng(0)
        A = g.standard_normal((m, n)).astype(np.float32)
        I = np.sort(g.choice(m, k, replace=False))
        r0, r1 = row_partition(m, rank, world, align=250)
        R = torch.zeros((k, n), dtype=torch.float32)
        for a, gi in enumerate(I):
            if r0 <= gi < r1:
                R[a] = torch.from_numpy(A[gi])
        comm.c.allreduce_f32(ctypes.c_void_p(R.data_ptr()), R.numel(), None, None)
        out["R_exact"] = bool(np.array_equal(R.numpy(), A[I]))
        # 3) fused k-means payload [k2*d sums | k2 weights | objective | ties] from row shards
        X = g.standard_normal((m, 3))
        lab = g.integers(0, 4, m)
        sl = slice(r0, r1)
        sums = np.zeros((4, 3)); wts = np.zeros(4)
        np.add.at(sums, lab[sl], X[sl]); np.add.at(wts, lab[sl], 1.0)
        payload = torch.from_numpy(np.concatenate([sums.ravel(), wts, [float(r1 - r0)], [rank]]).copy())
        comm.c.allreduce_f64(ctypes.c_void_p(payload.data_ptr()), payload.numel(), None, None)
        full = np.zeros((4, 3)); fw = np.zeros(4)
        np.add.at(full, lab, X); np.add.at(fw, lab, 1.0)
        p = payload.numpy()
        out["payload_ok"] = bool(np.allclose(p[:12].reshape(4, 3), full, rtol=1e-14) and np.array_equal(p[12:16], fw)
                                 and p[16] == m and p[17] == sum(range(world)))
        out["calls"] = comm.calls
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_comm_callbacks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        o = res[rank]
        assert o["f64"][0] == 0 and o["f64"][1] == [3.0 * i for i in range(10)]
        assert o["f32"][0] == 0 and o["f32"][1] == [3.0] * 7
        assert o["R_exact"] and o["payload_ok"] and o["calls"] == 4


@pytest.mark.parametrize("m,world,align", [(2000, 2, 250), (20000, 8, 250), (1001, 3, 1), (7, 4, 1), (400000, 8, 250)])
def test_row_partition_covers(m, world, align):
    parts = [row_partition(m, r, world, align) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == m
    for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
        assert a1 == b0 and a0 <= a1
    for a0, _ in parts:
        assert a0 % align == 0 or a0 == m


@pytest.mark.parametrize("n,world", [(1500, 2), (10000, 8), (5, 4)])
def test_col_partition_covers(n, world):
    parts = [col_partition(n, r, world) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(a1 == b0 for (_, a1), (b0, _) in zip(parts, parts[1:]))


def test_make_plan_fields():
    p = make_plan(20000, 10000, 50, rank=1, nranks=4, align=250)
    assert (p.m, p.n, p.kmax, p.rank, p.nranks) == (20000, 10000, 50, 1, 4)
    assert (p.row_begin, p.row_end) == (5000, 10000) and (p.col_begin, p.col_end) == (2500, 5000)

"""The tree-structured exchange (HMAT_EXCHANGE_TREE, csrc/comm.cpp) as a schedule:
log2 P rounds of recursive doubling, round j swapping the whole packed buffer
with rank ^ 2^j and adding the partner's copy (the paper's tree reduce +
broadcast of Steps 2-4, on the hypercube of ranks).

Run here with world-size 2/4/8 `gloo` processes on random fp64 buffers:
every rank ends with BIT-IDENTICAL sums (both partners add the same two
operands and IEEE addition is commutative), equal to the exact sum within
rounding -- the property that makes the exchange deterministic.  The NCCL
calls themselves run on the GPU at one rank (hmat_nccl_selftest)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal(n) * 10.0 ** rank)
        tmp = torch.empty_like(buf)
        bit = 1
        while bit < world:                                   # comm_tree_allreduce_sum's schedule
            partner = rank ^ bit
            reqs = [dist.isend(buf, partner), dist.irecv(tmp, partner)]
            for r in reqs:
                r.wait()
            buf += tmp                                       # launch_add_inplace
            bit <<= 1
        out_q.put((rank, buf.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_recursive_doubling_is_bitwise_identical_on_every_rank(world):
    n = 3001
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, world, port, n, out_q)) for g in range(world)]
    for p in procs:
        p.start()
    res = dict(out_q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for g in range(1, world):
        assert np.array_equal(res[g].view(np.int64), res[0].view(np.int64))
    exact = sum(np.random.default_rng(100 + g).standard_normal(n) * 10.0 ** g for g in range(world))
    assert np.abs(res[0] - exact).max() <= 1e-15 * world * np.abs(exact).max() * 10

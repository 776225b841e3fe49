"""Multi-GPU host logic on CPU: world-size 2/4/8 `gloo` process
groups emulate the per-rank work of the library's shards.

Each rank asks the library for its plan (hmat_plan_query: Morton row slice,
exchanged levels, packed exchange layout), computes from ITS OWN rows of V and x
the contributions the project kernel writes (numpy), sums the packed exchange
buffer over ranks with all_reduce (the library does the same with NCCL), computes
its rows of y from its rows of U, D and the z's, and rank 0 compares the gathered
y with the oracle.  This checks the partition and the exchange layout with real
multi-process communication; the CUDA kernels themselves are covered by the GPU
parity tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import hgen
from gen.hgen import HConfig


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sib(c, t, q):
    me = t % c
    return (t // c) * c + (q if q < me else q + 1)


def _slot(c, t, s):
    me, other = t % c, s % c
    return other if other < me else other - 1


def _worker(rank, world, port, cfg, nrhs, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_12441_b200 import hmat as hm
        info = hm.hmat_plan_query(cfg.L, cfg.d, cfg.b, cfg.r, world, rank)
        r0, r1 = info.row_begin, info.row_end
        n = r1 - r0
        c, r, W, L = cfg.c, cfg.r, cfg.W, cfg.L
        U, V, D = hgen.inputs(cfg, r0, r1)          # this rank's rows only
        x = hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1)
        E = np.zeros((max(1, info.exchange_rows), W, nrhs))
        Zloc = {}
        for l in range(1, L + 1):
            m = cfg.m(l)
            seg = min(m, n)
            for s_loc in range(n // seg):
                s = r0 // m + s_loc                      # global source node
                rows = slice(s_loc * seg, (s_loc + 1) * seg)
                zfull = V[l - 1][rows].T @ x[rows]       # (W, nrhs): all slots of s
                for q in range(c - 1):
                    t = _sib(c, s, q)
                    qt = _slot(c, t, s)
                    z = zfull[q * r:(q + 1) * r]
                    if l <= info.cross_levels:
                        E[info.level_rows_offset[l] + t, qt * r:(qt + 1) * r] += z
                    else:
                        assert s // c == t // c and (t * m) // n == (s * m) // n, "sibling off-rank"
                        Zloc.setdefault((l, t), np.zeros((W, nrhs)))[qt * r:(qt + 1) * r] = z
        Et = torch.from_numpy(E)
        dist.all_reduce(Et, op=dist.ReduceOp.SUM)       # Steps 2-4
        E = Et.numpy()
        y = np.einsum("kij,kjn->kin", D.reshape(-1, cfg.b, cfg.b), x.reshape(-1, cfg.b, nrhs)).reshape(n, nrhs)
        for l in range(1, L + 1):
            m = cfg.m(l)
            for i in range(n):
                t = (r0 + i) // m
                zt = E[info.level_rows_offset[l] + t] if l <= info.cross_levels else Zloc[(l, t)]
                y[i] += U[l - 1][i] @ zt
        ys = [torch.zeros(n, nrhs, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(y))
        if rank == 0:
            out_q.put((np.concatenate([t.numpy() for t in ys]), info.exchange_rows, info.cross_levels,
                       [(i.row_begin, i.row_end) for i in
                        [hm.hmat_plan_query(cfg.L, cfg.d, cfg.b, cfg.r, world, g) for g in range(world)]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [
    (HConfig("m2", d=2, L=3, b=8, r=3, seed=31), 2),
    (HConfig("m2", d=2, L=3, b=8, r=3, seed=31), 4),
    (HConfig("m2", d=2, L=3, b=8, r=3, seed=31), 8),
    (HConfig("m3", d=3, L=2, b=4, r=2, seed=32), 2),
    (HConfig("m3", d=3, L=2, b=4, r=2, seed=32), 8),
    (HConfig("m1", d=1, L=5, b=3, r=2, seed=33), 4),
])
def test_sharded_matvec_with_gloo(cfg, world):
    from oracle import oracle
    nrhs = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), cfg, nrhs, q), nprocs=world, join=True)
    y, ex_rows, cross, ranges = q.get(timeout=60)
    U, V, D = hgen.inputs(cfg)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs))
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    # contiguous equal Morton slices
    assert ranges == [(g * cfg.N // world, (g + 1) * cfg.N // world) for g in range(world)]
    # exchanged levels: parent spans > 1 rank  <=>  c^(l-1) < P
    assert cross == max(l for l in range(1, cfg.L + 1) if cfg.c ** (l - 1) < world)
    assert ex_rows == sum(cfg.c ** l for l in range(1, cross + 1))


@pytest.mark.parametrize("d,L,r,P,bytes_", [(2, 7, 16, 2, 1536), (2, 9, 16, 4, 1536), (2, 9, 16, 8, 7680),
                                             (3, 5, 32, 2, 14336), (3, 5, 32, 4, 14336), (3, 5, 32, 8, 14336)])
def test_exchange_bytes_match_survey_table(d, L, r, P, bytes_):
    """Packed exchange per rhs: 1,536 B (2D, P=2/4), 7,680 B (2D,
    P=8), 14,336 B (3D, P=2..8) -- independent of N, O(beta log^2 P)."""
    from paper_2008_12441_b200 import hmat as hm
    info = hm.hmat_plan_query(L, d, 64, r, P, 0)
    assert info.exchange_rows * info.W * 8 == bytes_

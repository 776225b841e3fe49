"""The library's kernels with a REAL collective between PROCESSES: one process
per rank (as bench.py runs under torchrun), all on the one GPU of the test box,
the cross-rank Steps 2-4 done by torch.distributed.

Each of P processes builds its Morton-row shard with a
caller-provided exchange (HMAT_EXCHANGE_EXTERNAL), runs hmat_project (Step 1 and
the on-chip Step 2) into its packed exchange buffer, the processes sum those
buffers with a gloo all_reduce, and hmat_expand (Step 5) reads the sum -- the
path bench.py falls back to when the library's own NCCL communicator cannot be
made, and the data path of the NCCL / tree exchanges minus their transport.  The
rows of every rank together are compared with the CPU oracle, for several
products in a row on the same handle and buffer.  (The NCCL transports
themselves need one GPU per rank: hmat_nccl_selftest runs them at one rank.)
"""
import os
import socket

import numpy as np
import pytest

from gen import hgen
from gen.hgen import HConfig
from oracle import oracle
from tests.helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, nrhs, out_q, trans=0, alpha=1.0, beta=0.0):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = None
    try:
        from paper_2008_12441_b200 import hmat as hm
        torch.cuda.set_device(0)
        r0, r1 = rank * cfg.N // world, (rank + 1) * cfg.N // world
        U, V, D = hgen.inputs(cfg, r0, r1)
        dd = hm._dist(nranks=world, rank=rank, device=0, external_exchange=True)
        create = hm.hmat_create_standard if cfg.adm else hm.hmat_create
        h = create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D, dd)
        assert hm.hmat_local_rows(h) == (r0, r1)
        cnt = hm.hmat_exchange_size_op(h, trans, nrhs)
        xbuf = torch.zeros(max(1, cnt), dtype=torch.float64, device="cuda")
        outs, sizes = [], []
        for rep in range(REPS):
            xh = hgen.xblock(cfg, nrhs=nrhs, vec=rep, row_begin=r0, row_end=r1)   # (rows, nrhs)
            x = torch.from_numpy(np.ascontiguousarray(xh.T)).cuda()                # column-major (rows, nrhs)
            y = torch.from_numpy(np.ascontiguousarray(_y0(cfg, nrhs, rep)[r0:r1].T)).cuda()
            hm.hmat_project_op(h, trans, x.t(), xbuf, nrhs)
            torch.cuda.synchronize()
            xc = xbuf.cpu()
            dist.all_reduce(xc)                                                   # Steps 2-4: sum over ranks
            xbuf.copy_(xc)
            hm.hmat_expand_op(h, trans, alpha, x.t(), xbuf, beta, y.t(), nrhs)
            torch.cuda.synchronize()
            outs.append(y.t().cpu().numpy())
            sizes.append(cnt)
        out_q.put((rank, (outs, sizes)))
    except Exception as e:  # pragma: no cover - reported to the parent
        out_q.put((rank, repr(e)))
    finally:
        if h is not None:
            hm.hmat_destroy(h)
        dist.destroy_process_group()


def _y0(cfg, nrhs, rep):
    """The y the GEMV form starts from (beta y0)."""
    return np.random.default_rng(900 + rep).standard_normal((cfg.N, nrhs))


def _run(cfg, P, nrhs, trans=0, alpha=1.0, beta=0.0):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, P, port, cfg, nrhs, q, trans, alpha, beta)) for g in range(P)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    for g in range(P):
        assert not isinstance(res[g], str), res[g]
    assert len({tuple(res[g][1]) for g in range(P)}) == 1     # every rank packs the same exchange
    assert res[0][1][0] > 0                                     # P > 1: there is a cross-rank exchange
    return [np.concatenate([res[g][0][rep] for g in range(P)], axis=0) for rep in range(REPS)]


@pytest.mark.parametrize("cfg,P,nrhs", [
    (HConfig("ext2d", d=2, L=4, b=16, r=4, seed=521), 2, 1),      # SIMT, 1 rhs
    (HConfig("ext3d", d=3, L=3, b=8, r=3, seed=522), 4, 2),       # SIMT, 2 rhs, octree
    (HConfig("ext2d8", d=2, L=5, b=16, r=8, seed=523), 8, 1),     # P = 8 (BASELINE's largest)
    (HConfig("extdm", d=2, L=4, b=64, r=16, seed=524), 4, 16),    # FP64 tensor cores (16-wide pass)
    (HConfig("extdm64", d=2, L=3, b=64, r=16, seed=525), 2, 64),  # FP64 tensor cores (64-wide pass)
], ids=lambda v: getattr(v, "name", str(v)))
def test_external_exchange_across_processes(cfg, P, nrhs):
    ys = _run(cfg, P, nrhs)
    U, V, D = hgen.inputs(cfg)
    for rep in range(REPS):
        ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs, vec=rep))
        assert_parity(ys[rep].reshape(ref.shape), ref)


@pytest.mark.parametrize("cfg,P,nrhs,trans", [
    (HConfig("exts2", d=2, L=4, b=8, r=3, adm=1, seed=531), 4, 2, 0),      # SIMT, boundary (halo) exchange
    (HConfig("exts2", d=2, L=4, b=8, r=3, adm=1, seed=531), 4, 1, 1),      # H^T: near-field products exchanged
    (HConfig("exts1", d=1, L=6, b=4, r=2, adm=1, seed=532), 8, 1, 0),      # 1D, nodes spanning ranks
    (HConfig("extsd", d=2, L=4, b=64, r=16, adm=1, seed=533), 2, 12, 0),   # tensor cores (16-wide), halo x by TMA
    (HConfig("extsd", d=2, L=4, b=64, r=16, adm=1, seed=533), 2, 12, 1),
], ids=lambda v: getattr(v, "name", str(v)))
def test_standard_external_exchange_across_processes(cfg, P, nrhs, trans):
    """Standard admissibility: the packed boundary
    exchange -- cross-rank z entries and the halo x of near-field neighbours (H),
    or the cross near-field products (H^T) -- summed by a real all_reduce between
    processes; the GEMV form alpha op(H) x + beta y0."""
    alpha, beta = 0.75, -0.5
    ys = _run(cfg, P, nrhs, trans, alpha, beta)
    U, V, D = hgen.inputs(cfg)
    loop = oracle.std_matvec_t if trans else oracle.std_matvec
    for rep in range(REPS):
        ref = alpha * loop(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs, vec=rep)) \
            + beta * _y0(cfg, nrhs, rep)
        assert_parity(ys[rep], ref)

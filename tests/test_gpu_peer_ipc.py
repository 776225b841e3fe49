"""HMAT_EXCHANGE_PEER across PROCESSES (one process per rank, as bench.py runs
it under torchrun), on the one GPU of the test box (f4).

Each of P processes builds its shard with exchange = PEER, exports the CUDA IPC
handle of its mailbox, all-gathers the handles (gloo) and imports them: the
project kernels then write into the other processes' mailboxes through the
mapped IPC memory and raise system-scope flags there.  To stay within the
one-GPU rule (no kernel may wait for a kernel of another rank that runs at the
same time) every process finishes its project (stream synchronised) before a
host barrier, and only then are the expands launched: each expand finds its P
flags already raised.  On P GPUs the host barrier is not needed.
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, nrhs, reps, out_q):
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
        h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D,
                           hm._dist(nranks=world, rank=rank, device=0, exchange=hm.HMAT_EXCHANGE_PEER))
        handles = [None] * world
        dist.all_gather_object(handles, hm.hmat_peer_export(h))
        hm.hmat_peer_import(h, handles)
        x = torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r1).T)).cuda()
        outs = []
        for _ in range(reps):
            hm.hmat_project(h, x.t(), None, nrhs)
            torch.cuda.synchronize()
            dist.barrier()          # every rank's flags are raised before any expand starts
            y = torch.empty_like(x)
            hm.hmat_expand(h, x.t(), None, y.t(), nrhs)
            torch.cuda.synchronize()
            dist.barrier()
            outs.append(y.t().cpu().numpy())
        out_q.put((rank, outs))
        dist.barrier()              # mailboxes stay mapped until every rank is done
    except Exception as e:  # pragma: no cover - reported to the parent
        out_q.put((rank, repr(e)))
    finally:
        if h is not None:
            hm.hmat_destroy(h)
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,P,nrhs", [
    (HConfig("ipc2d", d=2, L=4, b=16, r=4, seed=501), 2, 1),
    (HConfig("ipc3d", d=3, L=3, b=8, r=3, seed=502), 4, 3),
    (HConfig("ipcdm", d=2, L=4, b=64, r=16, seed=503), 2, 16),   # tensor-core path (16-wide pass)
], ids=lambda v: getattr(v, "name", str(v)))
def test_peer_exchange_ipc_processes(cfg, P, nrhs):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, P, port, cfg, nrhs, 3, q)) for g in range(P)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    for g in range(P):
        assert not isinstance(res[g], str), res[g]
    U, V, D = hgen.inputs(cfg)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, hgen.xblock(cfg, nrhs=nrhs))
    for rep in range(3):
        y = np.concatenate([res[g][rep] for g in range(P)], axis=0)
        assert_parity(y, ref)

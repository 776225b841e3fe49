"""Standard admissibility with P > 1 ranks: the library's packed
cross-rank exchange (csrc/std_exchange.h, queried through
hmat_std_exchange_query) checked on CPU.

* its sizes against brute-force counts built from the ORACLE's slot function
  (every interaction pair of levels 2..L not inside one rank; every leaf whose
  near field reaches another rank) and the closed form of a P = 2 cut;
* the whole data path with real multi-process communication: world-size 2/4/8
  `gloo` groups, each rank computing from ITS OWN rows (numpy) what the project
  kernel writes into the buffer (z of its sources, x of its boundary leaves),
  all_reduce, then its rows of y from its Zt rows (local pairs + unpacked
  entries) and the halo x, compared with the oracle by rank 0.
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
from oracle import oracle
from paper_2008_12441_b200 import hmat as hm


def morton_decode(d, k, level):
    x = [0] * d
    for j in range(level):
        for i in range(d):
            x[i] |= ((k >> (j * d + i)) & 1) << j
    return x


def brute_counts(d, L, b, P):
    """(E, Hn) by brute force over all node pairs, with the oracle's slot function."""
    c = 1 << d
    N = b * c ** L
    n_loc = N // P
    E = 0
    for l in range(2, L + 1):
        m = N // c ** l
        nodes = c ** l
        for t in range(nodes):
            for s in range(nodes):
                if oracle.std_slot(d, l, t, s) < 0:
                    continue
                inside = m <= n_loc and (t * m) // n_loc == (s * m) // n_loc
                E += not inside
    leaves = c ** L
    n = 1 << L
    Hn = 0
    for s in range(leaves):
        xs = morton_decode(d, s, L)
        for t in range(leaves):
            xt = morton_decode(d, t, L)
            if all(abs(xs[i] - xt[i]) <= 1 for i in range(d)) and (t * b) // n_loc != (s * b) // n_loc:
                Hn += 1
                break
    assert n > 0
    return E, Hn


@pytest.mark.parametrize("d,L,b,P", [(2, 3, 4, 2), (2, 3, 4, 4), (2, 4, 2, 8), (1, 6, 2, 8), (3, 2, 2, 8), (2, 3, 4, 16)])
def test_exchange_sizes_equal_brute_force(d, L, b, P):
    E, Hn = brute_counts(d, L, b, P)
    for g in range(P):
        q = hm.hmat_std_exchange_query(L, d, b, 2, P, g)
        assert (q["E"], q["Hn"]) == (E, Hn)


@pytest.mark.parametrize("d", [2, 3])
def test_halo_of_a_two_way_cut(d):
    """P = 2 cuts the domain at the top Morton bit (the last coordinate): the
    halo is the two leaf layers beside the cut, 2 n^(d-1) leaves: O((N/P)^((d-1)/d))
    (PAPER.md:1061-1068), not O(N)."""
    L = 5 if d == 2 else 3
    n = 1 << L
    q = hm.hmat_std_exchange_query(L, d, 4, 1, 2, 0)
    assert q["Hn"] == 2 * n ** (d - 1)
    assert len(q["pack"]) == n ** (d - 1)                       # this rank's layer
    assert (q["halo_of"] >= 0).sum() == (3 * n - 2) ** (d - 1)   # (t, eps) pairs across the cut


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, nrhs, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, L, b, r, c = cfg.d, cfg.L, cfg.b, cfg.r, cfg.c
        q = hm.hmat_std_exchange_query(L, d, b, r, world, rank)
        M, N = q["M"], cfg.N
        n = N // world
        r0 = rank * n
        U, V, Dn = hgen.inputs(cfg, r0, r0 + n)              # this rank's rows only
        x = hgen.xblock(cfg, nrhs=nrhs, row_begin=r0, row_end=r0 + n)
        cap = 1 if nrhs == 1 else 2 if nrhs == 2 else 4 if nrhs <= 4 else 8
        hb = (q["E"] * r * cap + 1) // 2 * 2
        buf = np.zeros(hb + q["Hn"] * cap * q["bpad"])
        zt = {}                                              # (level, target) -> (M r, nrhs)
        for l in range(2, L + 1):
            m = cfg.m(l)
            base, cnt = r0 // m, max(1, n // m)
            seg = min(m, n)
            for k in range(cnt):
                s = base + k
                rows = slice(k * seg, (k + 1) * seg)
                zfull = V[l - 1][rows].T @ x[rows]           # all slots of s (partial if s spans ranks)
                for qs in range(M):
                    t = -1
                    for tt in range(c ** l):                 # slot qs of s -> its target (oracle's slot map)
                        if oracle.std_slot(d, l, s, tt) == qs:
                            t = tt
                            break
                    if t < 0:
                        continue                             # partner outside the domain
                    z = zfull[qs * r:(qs + 1) * r]
                    e = q["src_entry"][q["src_off"][l] + k * M + qs]
                    if e >= 0:
                        for kk in range(nrhs):
                            buf[(e * cap + kk) * r:(e * cap + kk) * r + r] += z[:, kk]
                    else:
                        qt = oracle.std_slot(d, l, t, s)
                        zt.setdefault((l, t), np.zeros((M * r, nrhs)))[qt * r:(qt + 1) * r] = z
        for h, leaf in q["pack"]:                            # this rank's boundary-leaf x
            for kk in range(nrhs):
                o = hb + (h * cap + kk) * q["bpad"]
                buf[o:o + b] = x[leaf * b:(leaf + 1) * b, kk]
        t_buf = torch.from_numpy(buf)
        dist.all_reduce(t_buf, op=dist.ReduceOp.SUM)         # the library: ncclAllReduce
        buf = t_buf.numpy()
        for e, rq in q["unpack"]:                            # received entries -> Zt rows
            row, qt = rq >> 8, rq & 255
            l = max(ll for ll in range(2, L + 1) if q["zt_row_offset"][ll] <= row)
            t = r0 // cfg.m(l) + (row - q["zt_row_offset"][l])
            for kk in range(nrhs):
                zt.setdefault((l, t), np.zeros((M * r, nrhs)))[qt * r:(qt + 1) * r, kk] = \
                    buf[(e * cap + kk) * r:(e * cap + kk) * r + r]
        y = np.zeros((n, nrhs))
        nd = 3 ** d
        for i in range(n):
            gi = r0 + i
            lt = i // b
            xt = morton_decode(d, gi // b, L)
            for e in range(nd):                              # near field: local x or halo x
                off = [(e // 3 ** k) % 3 - 1 for k in range(d)]
                xs = [xt[k] + off[k] for k in range(d)]
                if any(v < 0 or v >= (1 << L) for v in xs):
                    continue
                s = sum(((xs[k] >> j) & 1) << (j * d + k) for j in range(L) for k in range(d))
                h = q["halo_of"][lt * nd + e]
                if h >= 0:
                    xv = np.stack([buf[hb + (h * cap + kk) * q["bpad"]:][:b] for kk in range(nrhs)], axis=1)
                else:
                    xv = x[s * b - r0:(s + 1) * b - r0]
                y[i] += Dn[i, e * b:(e + 1) * b] @ xv
            for l in range(2, L + 1):                        # far field
                t = gi // cfg.m(l)
                if (l, t) in zt:
                    y[i] += U[l - 1][i] @ zt[(l, t)]
        out_q.put((rank, y))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world,nrhs", [
    (HConfig("g2", d=2, L=3, b=4, r=2, adm=1, seed=901), 2, 1),
    (HConfig("g4", d=2, L=3, b=4, r=2, adm=1, seed=902), 4, 2),
    (HConfig("g8", d=1, L=5, b=3, r=2, adm=1, seed=903), 8, 1),   # 1D: nodes spanning ranks, odd leaf
])
def test_gloo_standard_exchange_matches_oracle(cfg, world, nrhs):
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, world, port, cfg, nrhs, out_q)) for g in range(world)]
    for p in procs:
        p.start()
    parts = dict(out_q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = np.concatenate([parts[g] for g in range(world)])
    U, V, Dn = hgen.inputs(cfg)
    ref = oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, hgen.xblock(cfg, nrhs=nrhs))
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("d,L,b,P", [(2, 3, 4, 2), (2, 4, 2, 8), (1, 6, 2, 8), (3, 2, 2, 8), (2, 3, 4, 16)])
def test_transposed_near_field_pairs(d, L, b, P):
    """H^T with P > 1: the cross near-field pairs (S, T) -- touching leaves on
    different ranks -- counted by brute force from the leaf geometry; every pair
    is written by exactly one rank (the owner of S, with T = S + eps_e, e the
    near-field code of T - S) and added by exactly one rank (the owner of T)."""
    c = 1 << d
    N = b * c ** L
    n_loc = N // P
    leaves = c ** L
    pairs = {}
    for s in range(leaves):
        xs = morton_decode(d, s, L)
        for e in range(3 ** d):
            eps = [(e // 3 ** i) % 3 - 1 for i in range(d)]
            xt = [xs[i] + eps[i] for i in range(d)]
            if not all(0 <= v < (1 << L) for v in xt):
                continue
            t = sum(((xt[i] >> j) & 1) << (j * d + i) for j in range(L) for i in range(d))
            if (s * b) // n_loc != (t * b) // n_loc:
                pairs[len(pairs)] = (s, t, e)
    written, added = {}, {}
    for g in range(P):
        q = hm.hmat_std_exchange_query(L, d, b, 2, P, g)
        assert q["Hp"] == len(pairs)
        lbase = g * n_loc // b
        for pair, sl, e in q["tpack"]:
            assert pair not in written and pairs[pair] == (lbase + sl, pairs[pair][1], e)
            written[pair] = g
        off = q["tadd_off"]
        assert len(off) == len(q["tadd_leaf"]) + 1 and off[0] == 0
        for k, tl in enumerate(q["tadd_leaf"]):
            pl = list(q["tadd_pair"][off[k]:off[k + 1]])
            assert pl == sorted(pl) and len(pl) > 0
            for pair in pl:
                assert pair not in added and pairs[pair][1] == lbase + tl
                added[pair] = g
    assert sorted(written) == sorted(added) == list(range(len(pairs)))

#!/usr/bin/env python
"""Benchmark of the weak-admissibility H-matvec y = Hx (arXiv 2008.12441) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one whole matvec (project + on-chip reduction + [exchange] + expand
with the dense leaf blocks) over one synthetic input vector of BASELINE.json's
workload.  Default workload: configs[3] ("c4", 2D, N = 2^24, L = 9, b = 64,
r = 16, 124.55 GB of factors), the configuration BASELINE.json quotes the
1/2/4/8-GPU metric on; it fits one B200.  Inputs: seeded synthetic panels
generated in place on the device (gen/), distinct x per step; the working set
(125 GB) is far larger than L2 (126 MB), so no flush is needed.

N > 1: one rank per GPU.  Launched by torch.distributed.run (the driver), or
`python bench.py --gpus N` re-executes itself under torch.distributed.run with
N local ranks; a world size different from --gpus is an error (rc 2).  Each
rank owns the Morton rows [g N/P, (g+1) N/P) of every panel (strong scaling of
one operator) and the library exchanges the cross-GPU z vectors with the
paper's tree-structured Steps 2-4 over NCCL (--exchange tree, the default;
PAPER.md:746-904).  Time = max over ranks.

Rank 0 prints one JSON line (see DESIGN.md §7 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gen import hgen  # noqa: E402
from gen.hgen import CONFIGS, EXTRA_CONFIGS  # noqa: E402

ALL_CONFIGS = {**CONFIGS, **EXTRA_CONFIGS}

METRIC = "H-matvec GB/s of factor data & matvecs/s vs HBM roofline, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(ALL_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="tree", choices=["tree", "nccl", "peer"],
                    help="N > 1: the paper's tree-structured exchange (recursive doubling over ncclSend/ncclRecv, "
                         "default), one ncclAllReduce, or the in-kernel exchange over NVLink peer memory (opt-in)")
    ap.add_argument("--launcher-check", action="store_true",
                    help="host-only: start the ranks (gloo), report the world each one sees, exit")
    return ap.parse_args()


def self_launch(args):
    """`--gpus N` (N > 1) outside torch.distributed: re-execute this script under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous) and return its
    exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launcher_check(args):
    """The ranks self_launch / the driver started: each joins a gloo group and
    rank 0 prints what every rank saw (a host test of the launcher)."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    seen = [(rank, world, int(os.environ.get("LOCAL_RANK", "0")))]
    if world > 1:
        dist.init_process_group("gloo")
        allv = [None] * world
        dist.all_gather_object(allv, seen[0])
        seen = allv
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"launcher_check": True, "gpus": args.gpus, "world": world,
                          "ranks": sorted(s[0] for s in seen), "worlds": sorted(set(s[1] for s in seen))}), flush=True)


def workload_desc(cfg):
    if cfg.adm:
        return (f"{cfg.name}: {cfg.d}D H-matrix fp64, STANDARD admissibility (rho=sqrt(d)), N={cfg.N} (Morton), "
                f"depth L={cfg.L}, leaf b={cfg.b}, rank r={cfg.r} blocks vs up to {cfg.slots} interaction-list "
                f"boxes per node, dense {cfg.b}x{cfg.b} near-field blocks (3^d per leaf), nrhs={cfg.nrhs}, seeded "
                f"synthetic (U,V~N(0,1)/sqrt(m_l), D~N(0,1)/8, x~U[-1,1]); not a BASELINE config")
    if cfg.name == "c2strict":
        return (f"c2strict: c2 (2D, N={cfg.N}, r={cfg.r}) under the paper-strict reading of Def 2.4: dense "
                f"{cfg.b}x{cfg.b} leaf-parent diagonal blocks, rank-{cfg.r} sibling blocks at levels 1..{cfg.L} "
                f"(= weak structure of depth {cfg.L}, leaf {cfg.b}); seeded synthetic; not a BASELINE config")
    return (f"{cfg.name}: {cfg.d}D H-matrix fp64, weak admissibility, N={cfg.N} (Morton), depth L={cfg.L}, "
            f"leaf b={cfg.b}, rank r={cfg.r} blocks vs each of {cfg.c - 1} siblings at every level, "
            f"dense {cfg.b}x{cfg.b} leaf-diagonal blocks, nrhs={cfg.nrhs}, seeded synthetic "
            f"(U,V~N(0,1)/sqrt(m_l), D~N(0,1)/8, x~U[-1,1])")


def alg_bytes(cfg, n_rows, nrhs):
    """Algorithmic bytes of one matvec over n_rows rows:
    factor panels once + x in + y out.  Split per kernel."""
    W, b = cfg.W, cfg.dcols
    L = cfg.L - (1 if cfg.adm else 0)  # standard admissibility: level 1 holds no blocks and is skipped
    project = 8 * n_rows * (W * L) + 8 * n_rows * nrhs
    expand = 8 * n_rows * (W * L + b) + 16 * n_rows * nrhs
    factor = 8 * n_rows * (2 * W * L + b)
    return {"project": project, "expand": expand, "factor": factor, "total": factor + 16 * n_rows * nrhs}


# Roofline of a pass: FP64 tensor pipe when its arithmetic intensity (2 nb flops per
# 8-byte factor entry, nb = the pass width) exceeds the ridge 37.07 TF / 7.3 TB/s
# ~ 5 flop/B, i.e. from 32-wide passes (33+ rhs); narrower passes stream HBM.
TENSOR_BOUND_RHS = 33
FP64_PEAK_TFLOPS = 37.07  # scripts/fp64_peak.cu, DMMA m8n8k4, this pool (profiles/r01_fp64_peak.txt)
# Read-only stream ceiling: scripts/hbm_read_peak.cu (bulk-TMA ring, random fp64 data,
# 800 back-to-back launches under the 1000 W cap), profiles/r01_hbm_read_peak.txt.
# The matvec is a read stream (124.8 GB read, 0.27 GB written at c4), so this is
# the number the kernels are compared with beside the copy peak.
HBM_READ_STREAM_GBS = 7300.0


def alg_flops(cfg, n_rows, nrhs):
    """Algorithmic flops of one matvec over n_rows rows: 2 per multiply-add."""
    W, b = cfg.W, cfg.dcols
    L = cfg.L - (1 if cfg.adm else 0)  # as alg_bytes
    return {"project": 2 * n_rows * W * L * nrhs, "expand": 2 * n_rows * (W * L + b) * nrhs}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config_name, kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d[config_name][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, pw, plim = [], [], set(), [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [s.strip() for s in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
            for dst, i in ((pw, 3), (plim, 9)):  # board power draw / enforced limit, W
                try:
                    dst.append(float(f[i]))
                except (ValueError, IndexError):
                    pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w": float(np.median(pw)) if pw else None,
                "power_limit_w": max(plim) if plim else None}


# --------------------------------------------------------------------------------------
# CPU oracle baseline: the oracle as it stands, single-threaded, on a bounded sample
# --------------------------------------------------------------------------------------

SAMPLE_BYTES = 1.5e9  # factor bytes of the oracle's bounded sample of a workload


def oracle_sample(cfg, budget_bytes=SAMPLE_BYTES):
    """The bounded sample the CPU oracle is timed on (cpu_baseline AND the
    reference arm: the same sample): the leading diagonal sub-H-matrix of `cfg`
    rooted at level q (rows [0, N/c^q)) -- exactly the blocks of cfg at levels
    q+1..L inside that diagonal block plus its dense leaves, an H-matrix of depth
    L-q with the same b, r, d -- for the smallest q whose factor bytes fit the
    budget.  Values are extrapolated to the whole workload by factor bytes."""
    for q in range(0, cfg.L + 1):
        n = cfg.N // cfg.c ** q
        depth = cfg.L - q
        fb = 8 * n * (2 * cfg.W * depth + cfg.dcols)
        if fb <= budget_bytes:
            return q, n, depth, fb
    return cfg.L, cfg.b, 0, 8 * cfg.b * cfg.b


def sample_desc(cfg, q, n, depth, fb):
    return (f"the leading level-{q} diagonal sub-H-matrix of {cfg.name} (rows [0,{n}), its blocks at levels "
            f"{q + 1}..{cfg.L} + dense leaves = an H-matrix of depth {depth}, {fb / 1e9:.3f} GB of factors, "
            f"nrhs={cfg.nrhs}); value extrapolated by factor bytes to {cfg.factor_bytes / 1e9:.2f} GB per matvec")


class OracleSample:
    """Panels of the sample (generated from the full operator's streams: the same
    values as the GPU operator's rows) and a timer of the oracle on them."""

    def __init__(self, cfg):
        import dataclasses
        self.cfg = cfg
        self.q, self.n, self.depth, self.fb = oracle_sample(cfg)
        if cfg.adm:
            # standard admissibility: a standalone operator of depth L-q with the same
            # b, r, d (a sub-block is not an H-matrix of the same kind at the boundary)
            sub = dataclasses.replace(cfg, L=self.depth)
            self.U, self.V, self.D = hgen.inputs(sub)
            self.x = hgen.xblock(sub, nrhs=cfg.nrhs)
        else:
            q = self.q
            self.U = [hgen.panel(cfg, hgen.TAG_U, q + l, 0, self.n) for l in range(1, self.depth + 1)]
            self.V = [hgen.panel(cfg, hgen.TAG_V, q + l, 0, self.n) for l in range(1, self.depth + 1)]
            self.D = hgen.panel(cfg, hgen.TAG_D, 0, 0, self.n)
            self.x = hgen.xblock(cfg, nrhs=cfg.nrhs, vec=0, row_begin=0, row_end=self.n)

    def once(self, threads):
        """Seconds of one oracle matvec over the sample on `threads` host threads
        (1: the plain block loop; more: its all-cores form, bit-identical)."""
        from oracle import oracle
        c = self.cfg
        t0 = time.perf_counter()
        if c.adm:
            oracle.std_matvec(c.d, self.depth, c.b, c.r, self.U, self.V, self.D, self.x)
        elif threads == 1:
            oracle.matvec(c.d, self.depth, c.b, c.r, self.U, self.V, self.D, self.x)
        else:
            oracle.matvec_par(c.d, self.depth, c.b, c.r, self.U, self.V, self.D, self.x, threads=threads)
        return time.perf_counter() - t0

    def timed(self, threads, min_seconds, max_reps):
        times = []
        while not times or (sum(times) < min_seconds and len(times) < max_reps):
            times.append(self.once(threads))
        return times

    def value(self, t):
        """matvec/s of the whole workload from the seconds of one sample pass."""
        return (self.fb / t) / self.cfg.factor_bytes


def cpu_baseline_record(cfg):
    """The oracle (as it stands) on the box's host cores, on the bounded sample:
    all cores (OpenMP block loop; the standard-admissibility oracle is single
    threaded) and, beside it, the plain one-thread loop."""
    from oracle import oracle
    smp = OracleSample(cfg)
    cores = 1 if cfg.adm else oracle.host_threads()
    t_all = smp.timed(cores, 8.0, 400)
    t_one = smp.timed(1, 8.0, 40) if cores > 1 else t_all
    med_all, med_one = float(np.median(t_all)), float(np.median(t_one))
    return {
        "value": smp.value(med_all),
        "unit": "matvec/s",
        "cores": cores,
        "kind": "oracle",
        "host_cores_available": len(os.sched_getaffinity(0)),
        "sample": f"{sample_desc(cfg, smp.q, smp.n, smp.depth, smp.fb)}; median of {len(t_all)} passes "
                  f"({med_all:.3f} s each) on {cores} host thread(s)",
        "factor_GBps": smp.fb / med_all / 1e9,
        "one_core": {"value": smp.value(med_one), "cores": 1, "factor_GBps": smp.fb / med_one / 1e9,
                     "reps": len(t_one), "median_s": med_one},
    }


def environment():
    """The report record's environment fields."""
    import platform
    env = {"host_cores": len(os.sched_getaffinity(0)), "glibc": "-".join(platform.libc_ver())}
    try:
        with open("/proc/cpuinfo") as f:
            env["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    try:
        import torch
        env["torch"] = torch.__version__
        env["cuda_runtime"] = torch.version.cuda
        if torch.cuda.is_available():
            env["gpu_name"] = torch.cuda.get_device_name()
            v = torch.cuda.nccl.version()
            env["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
        out = subprocess.run(["nvidia-smi", "--query-gpu=driver_version", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=10)
        env["driver"] = out.stdout.strip().splitlines()[0] if out.returncode == 0 and out.stdout.strip() else None
    except Exception:
        pass
    return env


def workload_config(cfg):
    """The `config` object of both arms (same workload, same keys)."""
    return {"workload": workload_desc(cfg), "N": cfg.N, "nrhs": cfg.nrhs, "factor_bytes": cfg.factor_bytes,
            "l2": "working set >> L2 (126 MB) except c1; no flush between steps"}


def run_reference(args):
    """--impl reference: the oracle timed on the host cores (rank 0 only), each
    step one pass over the same bounded sample cpu_baseline uses."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    cfg = ALL_CONFIGS[args.config]
    smp = OracleSample(cfg)
    cores = 1 if cfg.adm else oracle.host_threads()
    times = [smp.once(cores) for _ in range(args.warmup + args.steps)][args.warmup:]
    t = float(np.sum(times))
    value = args.steps * smp.fb / t / cfg.factor_bytes
    cpu = {"value": value, "unit": "matvec/s", "cores": cores, "kind": "oracle",
           "sample": f"per step: {sample_desc(cfg, smp.q, smp.n, smp.depth, smp.fb)}; {cores} host thread(s)"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2008_12441_b200 import hmat as hm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if local >= torch.cuda.device_count():
        print(f"error: rank {rank} has LOCAL_RANK {local} but {torch.cuda.device_count()} visible GPU(s)",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = ALL_CONFIGS[args.config]
    nrhs = cfg.nrhs
    stream = torch.cuda.Stream()   # one stream for fills, matvecs and the timing events
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream

    nid = None
    if world > 1:
        obj = [hm.hmat_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    create = hm.hmat_create_standard_uninit if cfg.adm else hm.hmat_create_uninit
    t_setup = time.perf_counter()
    # the in-kernel peer exchange serves the weak structure (SIMT and tensor-core
    # paths); the standard structure exchanges through NCCL
    exchange = args.exchange if world > 1 else "none"
    if exchange == "peer" and cfg.adm:
        exchange = "nccl"  # the peer exchange serves the weak-admissibility structure
    h = None
    if exchange == "peer":
        # mailboxes connected once through CUDA IPC handles (hmat_peer_export/_import)
        err = ""
        try:
            h = create(cfg.L, cfg.d, cfg.b, cfg.r,
                       hm._dist(nranks=world, rank=rank, cuda_stream=sptr, device=local,
                                exchange=hm.HMAT_EXCHANGE_PEER))
            handles = [None] * world
            dist.all_gather_object(handles, hm.hmat_peer_export(h))
            hm.hmat_peer_import(h, handles)
        except Exception as e:  # reported in the JSON line, never silent
            err = f"{type(e).__name__}: {e}"
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if any(errs):
            print(f"warning: peer exchange unavailable ({[e for e in errs if e][0]}); using NCCL", file=sys.stderr)
            if h is not None:
                hm.hmat_destroy(h)
            h = None
            exchange = "nccl (peer unavailable: " + [e for e in errs if e][0][:120] + ")"
    external = False
    if h is None:
        dd = hm._dist(nranks=world, rank=rank, nccl_unique_id=nid, cuda_stream=sptr, device=local,
                      exchange=hm.HMAT_EXCHANGE_TREE if exchange == "tree" else hm.HMAT_EXCHANGE_NCCL)
        err = ""
        try:
            h = create(cfg.L, cfg.d, cfg.b, cfg.r, dd)
        except Exception as e:  # reported in the JSON line, never silent
            err = f"{type(e).__name__}: {e}"
        if world > 1:
            errs = [None] * world
            dist.all_gather_object(errs, err)
            err = next((e for e in errs if e), "")
        if err:
            if world == 1:
                raise RuntimeError(err)
            # the library's own communicator could not be made: the same data path
            # with the exchange through torch.distributed (the split-phase API,
            # HMAT_EXCHANGE_EXTERNAL), so the run still measures the operator
            print(f"warning: library NCCL exchange unavailable ({err}); using the split-phase API with "
                  "torch.distributed all_reduce", file=sys.stderr)
            if h is not None:
                hm.hmat_destroy(h)
            h = create(cfg.L, cfg.d, cfg.b, cfg.r, hm._dist(nranks=world, rank=rank, cuda_stream=sptr, device=local,
                                                            external_exchange=True))
            external = True
            exchange = "external: torch.distributed all_reduce (library exchange unavailable: " + err[:120] + ")"
    r0, r1 = hm.hmat_local_rows(h)
    n = r1 - r0
    comm_nranks, comm_rank = hm.hmat_comm_info(h)
    hgen.dev_fill_operator(cfg, lambda kind, level: hm.hmat_panel(h, kind, level), r0, r1, sptr)
    xcnt = hm.hmat_exchange_size(h, nrhs) if external else 0
    xbuf = torch.zeros(max(1, xcnt), dtype=torch.float64, device="cuda") if external else None

    def matvec(xv, yv):
        """One product: hmat_matvec, or (fallback) project -> all_reduce -> expand."""
        if not external:
            hm.hmat_matvec(h, xv, yv, nrhs)
            return
        if xv.device.type != "cuda":   # e2e: host vectors through device copies
            xd = xv.to("cuda", non_blocking=True)
            yd = torch.empty_like(xd)
            matvec(xd, yd)
            yv.copy_(yd)
            return
        hm.hmat_project(h, xv, xbuf, nrhs)
        if xcnt:
            dist.all_reduce(xbuf)
        hm.hmat_expand(h, xv, xbuf, yv, nrhs)
    # distinct seeded x per timed step, up to the paper's 128 vectors,
    # as many as fit in a third of the free device memory (same count on every rank)
    free, _ = torch.cuda.mem_get_info()
    nvec = int(max(1, min(128, args.steps, free // 3 // max(1, 8 * n * nrhs))))
    if world > 1:
        tv = torch.tensor([nvec], device="cuda")
        dist.all_reduce(tv, op=dist.ReduceOp.MIN)
        nvec = int(tv.item())
    X = [torch.empty(nrhs, n, dtype=torch.float64, device="cuda") for _ in range(nvec)]
    for v, xv in enumerate(X):
        hgen.dev_fill_x(cfg, nrhs, v, r0, r1, xv.data_ptr(), n, sptr)
    Y = torch.empty(nrhs, n, dtype=torch.float64, device="cuda")
    xs = [xv.t() for xv in X]
    ys = Y.t()
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        matvec(xs[i % nvec], ys)
    torch.cuda.synchronize()
    hm.hmat_synchronize(h)  # raises on an asynchronous exchange error

    # ---------------- timed region (device, CUDA events on the launch stream) ----------
    # The K steps exactly as a user runs them (no per-kernel events: the library then
    # also overlaps expand's launch with project's tail, PDL) give `value`; a second
    # pass of K steps with the library's per-kernel CUDA events (same stream) gives
    # each kernel's mean duration for the roofline.
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)

    def timed_steps():
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for i in range(args.steps):
            matvec(xs[i % nvec], ys)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return ev0.elapsed_time(ev1)

    def per_step_times():
        """The same K steps with an event after each: per-step durations (max over
        ranks per step) for the median / min / max beside the mean."""
        barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for i in range(args.steps):
            matvec(xs[i % nvec], ys)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)], dtype=torch.float64,
                         device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        barrier()
        return t.cpu().numpy()

    ms_local = timed_steps()
    step_ms = per_step_times()
    hm.hmat_profile(h, True)
    hm.hmat_profile_read(h)  # reset
    ms_profiled = timed_steps()
    prof = hm.hmat_profile_read(h)
    hm.hmat_profile(h, False)
    clk = clocks.stop()
    hm.hmat_synchronize(h)  # raises on an asynchronous exchange error
    ms_total = max_over_ranks(ms_local)
    ms_step = ms_total / args.steps
    ms_prof_step = max_over_ranks(ms_profiled) / args.steps  # (collective: every rank)
    launches = hm.hmat_launches_per_matvec(h, nrhs) * args.steps

    # ---------------- e2e: C-ABI call with pinned host x / y, copies timed --------------
    # Every step copies its own x in from pinned host memory and its y back out,
    # through hmat_matvec with HOST pointers.  Two ways, both reported:
    #  * blocking (the default mode of the API): each call returns after y is home;
    #  * streaming (hmat_set_host_async): calls return once enqueued, x in / y out
    #    run on copy streams and overlap the neighbouring calls' kernels; timed
    #    from before the first call to hmat_synchronize() after the last.
    e2e = None
    if not args.no_e2e:
        xh = [torch.empty(nrhs, n, dtype=torch.float64).pin_memory() for _ in range(2)]
        for v, xv in enumerate(xh):
            xv.copy_(X[v % nvec])
        yh = torch.empty(nrhs, n, dtype=torch.float64).pin_memory()
        e2e_steps = max(3, min(args.steps, 64))  # the timed steps K (fill and drain of the copy pipeline amortised over them)
        matvec(xh[0].t(), yh.t())
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(e2e_steps):
            matvec(xh[i % 2].t(), yh.t())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        sync_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
        hm.hmat_set_host_async(h, True)
        matvec(xh[0].t(), yh.t())   # warm the staging buffers / streams
        hm.hmat_synchronize(h)
        barrier()
        torch.cuda.synchronize()
        runs = []  # wall clock: median of 3 runs, so one host hiccup does not decide it
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                matvec(xh[i % 2].t(), yh.t())
            hm.hmat_synchronize(h)
            runs.append(max_over_ranks((time.perf_counter() - t0) * 1e3) / e2e_steps)
        async_ms = sorted(runs)[1]
        hm.hmat_set_host_async(h, False)
        barrier()
        e2e = {"value": 1e3 / async_ms, "unit": "matvec/s", "h2d_bytes_per_step": 8 * cfg.N * nrhs,
               "d2h_bytes_per_step": 8 * cfg.N * nrhs, "ms_per_step": async_ms, "steps": e2e_steps,
               "runs_ms_per_step": runs,
               "how": "hmat_matvec with pinned host x/y in the streaming mode (hmat_set_host_async): every step's "
                      "H2D of x and D2H of y overlap the neighbouring steps' kernels; wall clock from the first "
                      "call to hmat_synchronize, max over ranks, median of 3 runs",
               "blocking": {"value": 1e3 / sync_ms, "ms_per_step": sync_ms,
                            "how": "same calls in the blocking mode (each returns after its y is home), CUDA events"}}

    # ---------------- roofline of the dominant kernel ----------------------------------
    ab = alg_bytes(cfg, n, nrhs)
    per_kernel = {}
    for ph in ("project", "expand"):
        ms, nl = prof[ph]
        if nl:
            per_kernel[ph] = {"avg_ms": ms / nl, "launches": nl, "alg_bytes_per_launch": ab[ph] / max(1, (nl // args.steps)),
                              "GBps": ab[ph] / (ms / nl * 1e-3) / 1e9 / max(1, (nl // args.steps))}
    dom = max(per_kernel, key=lambda k: per_kernel[k]["avg_ms"])
    if nrhs >= TENSOR_BOUND_RHS:
        # many right-hand sides: a dense FP64 contraction on the DMMA tensor pipe
        fl = alg_flops(cfg, n, nrhs)
        for ph, d in per_kernel.items():
            d["alg_flops_per_launch"] = fl[ph] / max(1, d["launches"] // args.steps)
            d["TFLOPs"] = d["alg_flops_per_launch"] / (d["avg_ms"] * 1e-3) / 1e12
        achieved = per_kernel[dom]["TFLOPs"]
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": ncu_traffic(cfg.name, dom),
                "peak_source": "measured FP64 DMMA m8n8k4 peak on this pool (profiles/r01_fp64_peak.txt)",
                "per_kernel": per_kernel}
        # the DMMA peak scales with the SM clock; under the board's power cap the
        # timed region runs below the clock the peak was measured at (1965 MHz)
        if clk.get("sm_mhz") and clk.get("sm_max_mhz"):
            at_clk = FP64_PEAK_TFLOPS * clk["sm_mhz"] / clk["sm_max_mhz"]
            roof["peak_at_clock"] = at_clk
            roof["frac_at_clock"] = achieved / at_clk
    else:
        peak, peak_src = measured_peaks()
        achieved = per_kernel[dom]["GBps"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(cfg.name, dom), "peak_source": peak_src,
                "per_kernel": per_kernel, "frac_of_8TBps_nominal": achieved / 8000.0,
                "frac_of_read_stream": achieved / HBM_READ_STREAM_GBS,
                "read_stream_source": "scripts/hbm_read_peak.cu sustained bulk-TMA read ring (profiles/r01_hbm_read_peak.txt)"}

    value = 1e3 / ms_step  # matvecs/s of the whole job (one operator across all ranks)
    # board energy per matvec (rank 0's GPU; median power x step time) -- only over a
    # timed region of >= 2 s: nvidia-smi's power.draw is a 1-s average, which lags a
    # shorter region (profiles/r02_power_probe.txt)
    if clk.get("power_w") and ms_total >= 2000.0:
        clk["j_per_matvec"] = clk["power_w"] * ms_step / 1e3
    elif clk.get("power_w"):
        clk["power_note"] = "timed region < 2 s: power.draw (1-s average) lags it"
    # bytes of the packed cross-GPU exchange buffer per pass (0 at P = 1), per step
    exch_width = min(nrhs, 64)
    try:
        exch_doubles = hm.hmat_exchange_size(h, exch_width) if world > 1 else 0
    except Exception:
        exch_doubles = 0
    # every rank's communicator spans the whole job (NCCL's own count for NCCL / TREE)
    cn = torch.tensor([comm_nranks], device="cuda")
    if world > 1:
        dist.all_reduce(cn, op=dist.ReduceOp.MIN)
    comm_nranks_ok = int(cn.item()) == world and comm_nranks == world
    factor_gbps = alg_bytes(cfg, cfg.N, nrhs)["factor"] / (ms_step * 1e-3) / 1e9
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_record(cfg)
        line = {
            "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg),
            "parallelism": f"Morton-row subtree shards x{world}, one rank per GPU",
            "exchange": exchange, "comm_nranks": comm_nranks, "comm_nranks_ok": bool(comm_nranks_ok),
            "distinct_x": nvec,
            "step_ms": {"mean": float(step_ms.mean()), "median": float(np.median(step_ms)),
                        "min": float(step_ms.min()), "max": float(step_ms.max()), "n": int(len(step_ms)),
                        "how": "a second pass of the K steps with a CUDA event after each step, max over ranks "
                               f"per step; {nvec} distinct seeded x (PAPER.md:1129-1130 averages 128); the events "
                               "between steps cost the cross-step launch overlap, so this pass runs a little slower "
                               "than the plain one that gives `value`"},
            "factor_GBps": factor_gbps,
            "alg_GBps": ab["total"] * world / (ms_step * 1e-3) / 1e9,
            # the memory floor: every factor byte and x / y once at the read-stream ceiling
            "floor_ms": alg_bytes(cfg, cfg.N, nrhs)["total"] / (HBM_READ_STREAM_GBS * 1e9) * 1e3 / world,
            "frac_of_floor": alg_bytes(cfg, cfg.N, nrhs)["total"] / (HBM_READ_STREAM_GBS * 1e9) * 1e3 / world / ms_step,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "phase_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
            "profiled_ms_per_step": ms_prof_step,
            "setup_s": setup_s,
            "vec_matvecs_per_s": value * nrhs,
            "exchange_bytes_per_step": 8 * exch_doubles * ((nrhs + exch_width - 1) // exch_width),
            "env": environment(),
        }
        print(json.dumps(line), flush=True)
    barrier()  # peer mailboxes are mapped by every rank: free them together
    hm.hmat_destroy(h)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1 and args.impl == "ours":
        sys.exit(self_launch(args))     # one rank per GPU under torch.distributed.run
    if world is not None and int(world) != args.gpus:
        print(f"error: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.launcher_check:
        launcher_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

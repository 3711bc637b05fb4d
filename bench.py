#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the stencil FMM same-level step.

Workload (BASELINE.json configs[3]): V1309 Scorpii contact-binary initial-model
shape, max refinement level 13, theta = 0.34 (the paper's 1074-element
stencil), FP64, all levels (root by reading C2).  A step = one pass of the hot path
over the whole tree: level ingest (octo_fmm_load_level from device buffers:
SURVEY 8(a) a1) for every level + octo_fmm_compute_interactions over all
levels (ghost exchange when N > 1, P2P / mixed / M2L+Lc kernels, a2-a8).
Inputs are synthetic (synth.config_v1309, seeded-free analytic densities);
multipole moments come from FMM step 1 run by the library's own kernels
(octo_fmm_p2m / octo_fmm_m2m) before timing.

metric: cell-interactions/s (whole job, all ranks), plus algorithmic FP64
GFLOP/s and the roofline of the dominant kernel measured live with CUDA events
recorded by the library (OCTO_TIMING) on the launching stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N > 1: launched by torch.distributed.run, one rank per GPU, NCCL; strong
scaling (the same tree partitioned along the Morton curve).
--impl reference: the oracle (oracle/, plain C, 1 core) timed on bounded
samples of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# FP64 flop per interaction of the formula the shipped kernels evaluate
# (C10; DFMA = 2, DMUL / DADD / rsqrt seed = 1), derived from the
# library's SASS by tests/flop_count.py and pinned to it by tests/test_flop_count.py
FLOPS = {"p2p": 8, "mixed": 120, "m2l": 195}
PAPER_FLOPS = {"p2p": 12, "m2l": 455}          # P:L529-531 (context only)
E2E_HANDLES = int(os.environ.get("OCTO_E2E_HANDLES", "3"))   # pipelined e2e loop (bench leg "e2e")
# configs[4]: V1309 at max level 15 with every node within
# r_env of the COM refined to 15; r_env = C4_R1 * N^(1/3) keeps ~1.2 M level-15
# sub-grids (~100 GB of the library's HBM) per GPU: weak scaling
C4_R1 = 2.0
THEORETICAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="v1309", choices=["c1", "c2", "c3", "v1309", "c4"],
                    help="BASELINE.json configs[0..3]; v1309 (configs[3]) is the bench workload")
    ap.add_argument("--max-level", type=int, default=13)
    ap.add_argument("--theta", type=float, default=None,
                    help="default: 0.5 for c1/c2 (as configured), 0.34 (the paper's 1074 stencil) otherwise")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-targets", type=int, default=80000)
    ap.add_argument("--rank-detail", action="store_true", help="per-rank breakdown on stderr")
    ap.add_argument("--env-radius", type=float, default=None,
                    help="configs[4] common-envelope radius (default C4_R1 * n_gpus^(1/3): weak scaling)")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the configs[0..2] lines (key 'other_configs', N = 1 only)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if r.returncode == 0 and r.stdout.strip():
                    self.rows.append([x.strip() for x in r.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "power_w_max": max(float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()),
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
# The contract's stdout carries exactly one JSON line (rank 0).  Everything
# else written to file descriptor 1 -- NCCL's version banner when a
# communicator is created, library or tool prints -- is routed to stderr;
# the result line goes to a duplicate of the original stdout.
RESULT_OUT = None


def claim_stdout():
    global RESULT_OUT
    sys.stdout.flush()
    RESULT_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(line):
    print(json.dumps(line), file=RESULT_OUT or sys.stdout, flush=True)


def dist_init(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------------------
# the oracle as a CPU baseline / reference arm (bounded samples)
# ---------------------------------------------------------------------------
def oracle_sample(tree, mom, theta, n_targets, seed):
    """Time the oracle on n_targets target cells drawn uniformly over all cells
    of all levels; returns (interactions, seconds)."""
    import oracle
    rng = np.random.default_rng(seed)
    lv = list(tree.levels)
    w = np.array([l.n_nodes for l in lv], float)
    pick = rng.choice(len(lv), size=n_targets, p=w / w.sum())
    inter, secs = 0, 0.0
    for i, l in enumerate(lv):
        k = int(np.sum(pick == i))
        if k == 0:
            continue
        tn = rng.integers(0, l.n_nodes, k)
        tc = rng.integers(0, 512, k).astype(np.int32)
        inter += int(oracle.count_interactions(tree, l.level, theta, targets=(tn, tc)).sum())
        t0 = time.perf_counter()
        oracle.same_level(tree, mom, l.level, theta, targets=(tn, tc))
        secs += time.perf_counter() - t0
    return inter, secs


# ---- the oracle on all host cores: a pool of processes, each holding the
# same seeded tree and moments, running the unmodified oracle on chunks of
# the sample (wall time of the whole pool = the host's throughput)
_W = {}


def _worker_init(cfg, max_level, theta):
    import argparse as _ap
    import oracle
    tree, _ = make_tree(_ap.Namespace(config=cfg, max_level=max_level, theta=theta))
    _W.update(tree=tree, mom=oracle.moments(tree), theta=theta)


def _worker_task(job):
    import oracle
    l, tn, tc = job
    oracle.same_level(_W["tree"], _W["mom"], l, _W["theta"], targets=(tn, tc))
    return len(tn)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_pool(args, procs):
    import multiprocessing as mp
    pool = mp.get_context("spawn").Pool(procs, initializer=_worker_init,
                                        initargs=(args.config, args.max_level, args.theta))
    pool.map(_worker_task, [(1, np.zeros(1, np.int64), np.zeros(1, np.int32))] * procs)   # warm every worker
    return pool


def oracle_sample_parallel(tree, pool, procs, theta, n_targets, seed):
    """oracle_sample's work split over `procs` processes; (interactions, wall seconds)."""
    import oracle
    rng = np.random.default_rng(seed)
    lv = list(tree.levels)
    w = np.array([l.n_nodes for l in lv], float)
    pick = rng.choice(len(lv), size=n_targets, p=w / w.sum())
    jobs, inter = [], 0
    for i, l in enumerate(lv):
        k = int(np.sum(pick == i))
        if k == 0:
            continue
        tn = rng.integers(0, l.n_nodes, k)
        tc = rng.integers(0, 512, k).astype(np.int32)
        inter += int(oracle.count_interactions(tree, l.level, theta, targets=(tn, tc)).sum())
        for a in range(0, k, max(1, k // (4 * procs) + 1)):
            b_ = min(k, a + max(1, k // (4 * procs) + 1))
            jobs.append((l.level, tn[a:b_], tc[a:b_]))
    t0 = time.perf_counter()
    pool.map(_worker_task, jobs, chunksize=1)
    return inter, time.perf_counter() - t0


def make_tree(args):
    """BASELINE.json configs."""
    if args.theta is None:
        args.theta = 0.5 if args.config in ("c1", "c2") else 0.34
    if args.config == "c1":
        return synth.config_c1(0), "configs[0]: 2x2x2 leaf sub-grids, random densities"
    if args.config == "c2":
        return synth.config_c2(), "configs[1]: uniform level 3 (512 sub-grids), Gaussian star"
    if args.config == "c3":
        return synth.config_c3(), "configs[2]: rotating n=1 polytrope, 3-level AMR"
    if args.config == "c4":
        return None, "configs[4]: V1309 binary, max level 15 + common envelope"
    return synth.config_v1309(args.max_level), f"configs[3]: V1309 binary, max level {args.max_level}"


def run_reference(args, ws, rank):
    if rank != 0:
        return
    tree, wname = make_tree(args)
    procs = host_cores()
    pool = oracle_pool(args, procs)
    n = max(50, args.cpu_sample_targets // 16) * procs   # ~0.8 s of oracle work per step on all cores
    for s in range(args.warmup):
        oracle_sample_parallel(tree, pool, procs, args.theta, n, 1000 + s)
    inter, secs = 0, 0.0
    for s in range(args.steps):
        i, t = oracle_sample_parallel(tree, pool, procs, args.theta, n, s)
        inter += i
        secs += t
    pool.close()
    v = inter / secs
    line = {"impl": "reference", "metric": "FMM cell-interactions/s", "value": v, "unit": "interactions/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{wname}, theta {args.theta}",
                       "sample": f"{n} random target cells per step over all levels (oracle, {procs} processes)"},
            "cpu_baseline": {"value": v, "unit": "interactions/s", "cores": procs, "kind": "oracle",
                             "sample": f"{n} random target cells per step, {args.steps} steps, one oracle process "
                                       f"per host core"},
            "e2e": {"value": v, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------------------
# configs[0..2] in the same process: same step definition
# (load every level from device buffers + compute over all levels), same
# event timing on the launching stream and L2 flush between timed steps
# ---------------------------------------------------------------------------
def time_other_config(name, steps, warmup, flush):
    import torch
    import paper_1908_03121_b200 as P
    from paper_1908_03121_b200.levels import upward
    ns = argparse.Namespace(config=name, max_level=13, theta=None)
    tree, wname = make_tree(ns)
    f = P.OctoFMM(ns.theta, timing=True)
    data = upward(f, tree)
    stream = torch.cuda.current_stream()

    def step(levels=None):
        for lv in tree.levels:
            if levels is not None and lv.level not in levels:
                continue
            d = data[lv.level]
            f.load_level(lv.level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, None, d["mono"], d["com"],
                         d["mom"])
        f.compute_interactions(P.OCTO_ALL_LEVELS if levels is None else levels[0])

    def timed(levels=None):
        for _ in range(max(3, warmup)):
            step(levels)
        torch.cuda.synchronize()
        f.kernel_times()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            step(levels)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        f.sync()
        kms, calls = f.kernel_times()
        return sum(a.elapsed_time(b) for a, b in evs) / steps, [k / max(1, calls) for k in kms]

    def graph_timed():
        """The same step (ingest of every level + the kernels) captured once
        into a CUDA graph by a second handle (no event timing) and replayed:
        these configs are launch-bound (sub-ms steps), and a graph replays the
        step's 5-6 launches without per-call host work."""
        g_f = P.OctoFMM(ns.theta)

        def gstep():
            for lv in tree.levels:
                d = data[lv.level]
                g_f.load_level(lv.level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, None, d["mono"],
                               d["com"], d["mom"])
            g_f.compute_interactions(P.OCTO_ALL_LEVELS)
        try:
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                for _ in range(max(3, warmup)):
                    gstep()
            stream.wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                gstep()
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for k in range(steps):
                flush.fill_(float(k))
                evs[k][0].record(stream)
                graph.replay()
                evs[k][1].record(stream)
            torch.cuda.synchronize()
            g_f.sync()   # surfaces any ingest / kernel error of the replays
            return sum(a.elapsed_time(b) for a, b in evs) / steps, None
        except Exception as e:   # capture not possible here: report the stream-launched step only
            return None, f"{type(e).__name__}: {e}"[:160]
        finally:
            g_f.close()

    step()
    f.sync()
    counts = f.interaction_counts()
    ms, kms = timed()
    gms, gerr = graph_timed()
    inter = int(counts.sum())
    fl = counts[0] * FLOPS["p2p"] + counts[2] * FLOPS["mixed"] + counts[1] * FLOPS["m2l"]
    best = min(ms, gms) if gms else ms
    out = {"workload": f"{wname}, theta {ns.theta}", "value": inter / (best * 1e-3), "unit": "interactions/s",
           "ms_per_step": best, "launch": "cuda_graph" if gms and gms <= ms else "stream",
           "ms_per_step_stream": ms, "ms_per_step_graph": gms, "steps": steps, "interactions_per_step": inter,
           "gflops_fp64": fl / (best * 1e-3) / 1e9,
           "kernel_ms_per_step": {"p2p": kms[0], "mixed": kms[1], "m2l": kms[2]}}
    if gerr:
        out["graph_error"] = gerr
    if name == "c2":
        # d2: the level-3 P2P launch alone (the config's "monopole-only P2P path")
        lv3 = max(lv.level for lv in tree.levels)
        c3 = f.interaction_counts(lv3)
        ms3, k3 = timed([lv3])
        out["p2p_level"] = {"level": lv3, "value": int(c3.sum()) / (ms3 * 1e-3), "ms_per_step": ms3,
                            "interactions_per_step": int(c3.sum()), "p2p_kernel_ms": k3[0],
                            "gflops_fp64": int(c3[0]) * FLOPS["p2p"] / (k3[0] * 1e-3) / 1e9 if k3[0] else None}
    f.close()
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    claim_stdout()
    ws, rank, local = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    import paper_1908_03121_b200 as P
    from paper_1908_03121_b200.levels import upward
    from paper_1908_03121_b200.peaks import measure_fp64_peak

    torch.cuda.set_device(local)
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    tree, wname = make_tree(args)
    sharded = args.config == "c4"
    if sharded:
        # configs[4]: structure on every rank, data only for the rank's shard
        r_env = args.env_radius if args.env_radius is not None else C4_R1 * ws ** (1.0 / 3.0)
        model = synth.V1309(15, r_env)
        tree = model.tree(structure_only=True)
    lvls = list(tree.levels)   # root (a9, reading C2) included
    # partition weights: per-node interaction counts (the library's host-side
    # node_costs) x per-class device cost
    nodew = [synth.cost_weights(P.node_costs(args.theta, lv.refined, lv.neighbors)) if lv.level >= 1
             else np.ones(lv.n_nodes) for lv in lvls]
    if sharded:
        owners_sh, l0 = synth.shard_owners(tree, ws, node_weights=nodew)
        wname = f"{wname}, r_env {r_env:.3f}, subtree partition at level {l0}"
    owner = {lv.level: synth.partition_level(lv.refined, ws, weights=nodew[lv.level]) for lv in lvls}

    nccl_id, nccl_id2 = None, [None] * (E2E_HANDLES - 1)
    if ws > 1:
        import torch.distributed as dist
        obj = [[P.nccl_unique_id() for _ in range(1 + E2E_HANDLES - 1)] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id, nccl_id2 = obj[0][0], obj[0][1:]
    fmm = P.OctoFMM(args.theta, device=dev, rank=rank, nranks=ws, nccl_id=nccl_id, timing=True)

    # ---- inputs: densities (host, synthetic; device for configs[4]) -> FMM step 1 on the device
    if sharded:
        import torch.distributed as dist
        from paper_1908_03121_b200.levels import upward_shard
        tables, data = upward_shard(fmm, tree, model, owners_sh, l0, rank,
                                    (lambda t: dist.all_reduce(t)) if ws > 1 else (lambda t: None))
    else:
        data = upward(fmm, tree)
        tables = [(lv.ijk, lv.refined, lv.neighbors, owner[lv.level] if ws > 1 else None) for lv in lvls]
    torch.cuda.synchronize()

    def load_all(src, f=fmm, stream=None):
        for lv in lvls:
            d = src[lv.level]
            ijk, ref, nb, ow = tables[lv.level]
            f.load_level(lv.level, lv.h, tree.origin, ijk, ref, nb, ow, d["mono"], d["com"], d["mom"], stream=stream)

    def step():
        load_all(data)
        fmm.compute_interactions()

    step()
    torch.cuda.synchronize()
    fmm.sync()
    counts = fmm.interaction_counts()          # this rank's owned work
    inter_rank = int(counts.sum())
    inter_total = allreduce_sum(inter_rank, ws)
    flops_rank = counts[0] * FLOPS["p2p"] + counts[2] * FLOPS["mixed"] + counts[1] * FLOPS["m2l"]
    flops_total = allreduce_sum(float(flops_rank), ws)

    # L2 flush buffer (> 126 MB L2), written between timed steps
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    fmm.kernel_times()                            # reset accumulators
    launches0 = fmm.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    gpu_launches = fmm.launch_count() - launches0
    ms_rank = sum(a.elapsed_time(b) for a, b in evs)
    ms = allreduce_max(ms_rank, ws)
    kms, kcalls = fmm.kernel_times()
    if args.rank_detail:
        print(json.dumps({"rank": rank, "ms_step": ms_rank / args.steps, "counts": [int(c) for c in counts],
                          "kernel_ms": [k / max(1, kcalls) for k in kms]}), file=sys.stderr, flush=True)
    ms_step = ms / args.steps
    value = inter_total * args.steps / (ms * 1e-3)
    gflops = flops_total * args.steps / (ms * 1e-3) / 1e9

    by_kernel = {"p2p": int(allreduce_sum(float(counts[0]), ws)), "m2l": int(allreduce_sum(float(counts[1]), ws)),
                 "mixed": int(allreduce_sum(float(counts[2]), ws))}
    # paper convention (context): 549,888 x 455 flop per refined
    # sub-grid, 549,888 x 12 per leaf sub-grid, per step
    n_ref = sum(int(lv.refined.sum()) for lv in lvls if lv.level >= 1)
    n_leaf = sum(int((lv.refined == 0).sum()) for lv in lvls if lv.level >= 1)
    paper_gflops = (n_ref * 549888 * PAPER_FLOPS["m2l"] + n_leaf * 549888 * PAPER_FLOPS["p2p"]) / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (rank 0's own launches)
    names = ["p2p", "mixed", "m2l"]
    xms = kms[3] / max(1, kcalls)
    kms = kms[:3]
    dom = int(np.argmax(kms))
    dom_ms = kms[dom] / max(1, kcalls)
    dom_flops = [counts[0] * FLOPS["p2p"], counts[2] * FLOPS["mixed"], counts[1] * FLOPS["m2l"]][dom]
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12
    peak = measure_fp64_peak(reps=10) if rank == 0 else {"fp64_tflops_burst": None}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(names[dom])
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "kernel": {"p2p": "p2p_kernel", "mixed": "m2l_mixed_kernel",
                                            "m2l": "m2l_dense_kernel"}[names[dom]],
                "achieved": achieved, "peak": THEORETICAL_FP64_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / THEORETICAL_FP64_TFLOPS, "traffic": traffic,
                "peak_source": "148 SM x 64 FP64 lanes x 2 flop x 1.965 GHz (DESIGN.md Roofline)",
                "peak_measured_dfma": peak["fp64_tflops_burst"],
                "frac_of_measured_dfma": (achieved / peak["fp64_tflops_burst"]) if peak["fp64_tflops_burst"] else None,
                "kernel_ms_per_step": {n: kms[i] / max(1, kcalls) for i, n in enumerate(names)},
                "exchange_ms_per_step": xms,
                "flop_per_interaction": FLOPS}

    # ---- e2e through the public API with HOST buffers (pinned), copies inside
    # the timed region.  Steps are pipelined the way a serving loop runs them:
    # E2E_HANDLES handles on as many streams, with event chains so that the
    # host->device ingest, the kernels and the device->host result copies
    # (OCTO_HOST_ASYNC) each process the steps in order -- step k+1's ingest
    # overlaps step k's kernels, step k's result copy overlaps step k+1's.
    e2e = None
    if sharded:
        e2e = {"value": None, "unit": "interactions/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "not_measured": "configs[4] inputs are generated on the device per shard (tens of GB per rank)"}
    elif not args.no_e2e:
        host = {}
        for lv in lvls:
            d = data[lv.level]
            host[lv.level] = {k: (d[k].cpu().pin_memory() if d[k] is not None else None) for k in d}
        hs = [fmm] + [P.OctoFMM(args.theta, device=dev, rank=rank, nranks=ws, nccl_id=nccl_id2[i])
                      for i in range(E2E_HANDLES - 1)]
        ss = [torch.cuda.Stream() for _ in hs]
        outs = []
        for i in range(len(hs)):
            o = {}
            for lv in lvls:
                nr, nf = fmm.compact_sizes(lv.level)
                o[lv.level] = (torch.empty((23, nr, 512), dtype=torch.float64).pin_memory(),
                               torch.empty((7, nf, 512), dtype=torch.float64).pin_memory())
            outs.append(o)
        # the library copies only the owned rows of host inputs (ghost rows come
        # from the exchange): count exactly those bytes
        h2d = 0
        for lv in lvls:
            ow = tables[lv.level][3]
            mine = np.ones(lv.n_nodes, bool) if ow is None else (np.asarray(ow) == rank)
            # mono (all owned nodes) + com (3 rows) + mom rows 0 and 4..19 (the dipole rows 1..3 are
            # ignored by contract and not copied) of the owned refined nodes
            h2d += 512 * 8 * (int(mine.sum()) + 20 * int((mine & (lv.refined == 1)).sum()))
        d2h = sum(a.numel() * 8 + b.numel() * 8 for a, b in outs[0].values())
        chain = {}

        def phase(s_, name):
            # order this phase after the same phase of the previous step
            if name in chain:
                s_.wait_event(chain[name])
            e = torch.cuda.Event()
            chain[name] = e
            return e

        def e2e_step(k):
            i = k % len(hs)
            f, s_, o = hs[i], ss[i], outs[i]
            e = phase(s_, "h2d")
            load_all(host, f, s_)
            e.record(s_)
            e = phase(s_, "compute")
            f.compute_interactions(stream=s_)
            e.record(s_)
            e = phase(s_, "d2h")
            for lv in lvls:
                f.get_expansions_compact(lv.level, o[lv.level][0], o[lv.level][1], stream=s_, non_blocking=True)
            e.record(s_)

        for k in range(len(hs)):
            e2e_step(k)
        torch.cuda.synchronize()
        for f in hs:
            f.sync()                      # deferred input-validation errors, if any
        ke = max(4, min(args.steps, 50))   # pipeline fill + drain (~1 step) amortised over ke steps
        barrier(ws)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s_ in ss:
            s_.wait_stream(stream)
        for k in range(ke):
            e2e_step(k)
        for s_ in ss:
            stream.wait_stream(s_)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        for f in hs:
            f.sync()
        ems = allreduce_max(a.elapsed_time(b), ws)
        e2e = {"value": inter_total * ke / (ems * 1e-3), "unit": "interactions/s",
               "h2d_bytes_per_step": int(allreduce_sum(h2d, ws)), "d2h_bytes_per_step": int(allreduce_sum(d2h, ws)),
               "ms_per_step": ems / ke, "steps": ke,
               "pipelining": f"{len(hs)} handles x {len(hs)} streams, ingest / kernels / result copies each in step "
                             "order; every step: pinned H2D of all inputs, all levels, D2H of all results"}
        for f in hs[1:]:
            f.close()

    # ---- configs[0..2] (d1-d3), same process and clock sampler (N = 1 only)
    other = None
    if ws == 1 and not sharded and args.config == "v1309" and not args.no_other_configs:
        other = {}
        with ClockSampler(dev) as clk2:
            for nm, key in (("c1", "configs[0]"), ("c2", "configs[1]"), ("c3", "configs[2]")):
                try:
                    other[key] = time_other_config(nm, max(20, min(args.steps, 100)), args.warmup, flush)
                except Exception as exc:   # the main result line must not depend on these
                    other[key] = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
        other["clocks"] = clk2.summary()

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not sharded:
        try:
            import oracle
            mom = oracle.moments(tree)
            inter, secs = oracle_sample(tree, mom, args.theta, args.cpu_sample_targets, 7)
            cpu = {"value": inter / secs, "unit": "interactions/s", "cores": 1, "kind": "oracle",
                   "sample": f"{args.cpu_sample_targets} random target cells over all levels "
                             f"({inter} interactions, {secs:.1f} s)"}
            procs = host_cores()
            if procs > 1:   # the same oracle on every host core (one process each)
                try:
                    pool = oracle_pool(args, procs)
                    n_all = args.cpu_sample_targets * 2
                    i2, s2 = oracle_sample_parallel(tree, pool, procs, args.theta, n_all, 8)
                    pool.close()
                    cpu["all_cores"] = {"value": i2 / s2, "cores": procs,
                                        "sample": f"{n_all} random target cells ({i2} interactions, {s2:.1f} s wall)"}
                except Exception as exc:   # the GPU result line must not depend on the host pool
                    cpu["all_cores"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
        except Exception as exc:
            cpu = {"value": None, "unit": "interactions/s", "cores": 1, "kind": "oracle",
                   "error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": "FMM cell-interactions/s", "value": value, "unit": "interactions/s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak" if sharded else "strong", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (analytic V1309 density field; moments by the library's P2M/M2M kernels)",
                "config": {"workload": f"{wname}, theta {args.theta}",
                           "subgrids": tree.summary()["subgrids"], "refined": tree.summary()["refined"],
                           "interactions_per_step": inter_total,
                           "interactions_by_kernel": by_kernel,
                           "parallelism": (f"subtree shards x{ws} (owned + ghost nodes per rank)" if sharded
                                           else f"morton-partition x{ws}"),
                           "l2": "flushed between timed steps",
                           "hbm_used_gb_rank0": (lambda fr, tot: (tot - fr) / 1e9)(*torch.cuda.mem_get_info())},
                "gflops_fp64": gflops,
                # whole-step algorithmic FP64 rate per GPU over one GPU's peak
                "frac_fp64_peak_per_gpu": gflops / ws / 1e3 / THEORETICAL_FP64_TFLOPS,
                "paper_convention": {
                    "gflops": paper_gflops,
                    "note": "union-stencil convention (549,888 x 455 flop per refined sub-grid, x 12 per leaf "
                            "sub-grid, P:L526-531): counts masked and absent-partner work, so it can exceed the "
                            "device peak; context only"},
                "roofline": roofline,
                "cpu_baseline": cpu if not sharded else {"value": None, "not_measured":
                                                         "configs[4] exceeds the oracle's host memory; see configs[3]"},
                "e2e": e2e, "gpu_launches": int(gpu_launches),
                "other_configs": other,
                "clocks": clk.summary()}
        emit(line)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

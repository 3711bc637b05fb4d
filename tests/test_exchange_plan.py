"""Multi-rank host logic on CPU (no GPU): the ghost plan of exchange.cu
(octo_fmm_exchange_plan, pure host code in the library) covers every partner a
rank's stencil needs from other ranks, and sender/receiver lists agree in
canonical order; a world_size-2 gloo run moves the data with the plan."""
import os

import numpy as np
import pytest

import oracle
import synth
import paper_1908_03121_b200 as P
from synth.trees import LOCAL_XYZ


def _ijk_cells(lv, lst):
    node = lst // 512
    cell = lst % 512
    return np.concatenate([lv.ijk[node].astype(np.int64) * 8 + LOCAL_XYZ[cell]], axis=0)


@pytest.mark.parametrize("theta,nranks,seed", [(0.34, 2, 1), (0.34, 3, 5), (0.5, 4, 2), (0.25, 2, 3), (0.34, 8, 4)])
def test_plan_consistency_and_coverage(theta, nranks, seed):
    tr = synth.config_random_amr(seed, 3, 0.45)
    st = oracle.stencil(theta)
    for lv in tr.levels[1:]:
        owner = synth.partition_level(lv.refined, nranks)
        plans = {r: P.exchange_plan(theta, r, nranks, lv.ijk, lv.refined, lv.neighbors, owner) for r in range(nranks)}
        for r in range(nranks):
            for p, (sl, sr, rl, rr) in plans[r].items():
                # what r sends to p is what p receives from r, cell for cell, in the same order
                psl, psr, prl, prr = plans[p][r]
                assert np.array_equal(_ijk_cells(lv, sl), _ijk_cells(lv, prl))
                assert np.array_equal(_ijk_cells(lv, sr), _ijk_cells(lv, prr))
                assert np.all(owner[sl // 512] == r) and np.all(owner[rl // 512] == p)
                assert np.all(lv.refined[sl // 512] == 0) and np.all(lv.refined[sr // 512] == 1)
        # coverage: every stencil partner of an owned cell that lives on another rank is received
        key = {tuple(k): i for i, k in enumerate(lv.ijk.tolist())}
        for r in range(nranks):
            got = set()
            for p, (sl, sr, rl, rr) in plans[r].items():
                for lst in (rl, rr):
                    got |= set(map(tuple, _ijk_cells(lv, lst).tolist()))
            mine = np.nonzero(owner == r)[0]
            for node in mine[:: max(1, len(mine) // 6)]:
                for cell in range(0, 512, 7):
                    g = lv.ijk[node].astype(np.int64) * 8 + LOCAL_XYZ[cell]
                    c = int((g[0] & 1) + 2 * (g[1] & 1) + 4 * (g[2] & 1))
                    for d in st[c][:, :3]:
                        j = g + d
                        nb = key.get(tuple((j // 8).tolist()))
                        if nb is not None and owner[nb] != r:
                            assert tuple(j.tolist()) in got


def _gloo_worker(rank, world, port, ret):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = synth.config_c3()
        lv = tr.levels[2]
        owner = synth.partition_level(lv.refined, world)
        plan = P.exchange_plan(0.34, rank, world, lv.ijk, lv.refined, lv.neighbors, owner)
        # "device" data of this rank: the true density only on owned nodes, NaN elsewhere
        data = np.where((owner == rank)[:, None], lv.rho, np.nan)
        reqs = []
        bufs = {}
        for p, (sl, sr, rl, rr) in sorted(plan.items()):
            send = np.concatenate([data[sl // 512, sl % 512], data[sr // 512, sr % 512]])
            bufs[p] = torch.zeros(len(rl) + len(rr), dtype=torch.float64)
            reqs.append(dist.isend(torch.from_numpy(send), p))
            reqs.append(dist.irecv(bufs[p], p))
        for q in reqs:
            q.wait()
        ok = True
        for p, (sl, sr, rl, rr) in plan.items():
            lst = np.concatenate([rl, rr])
            data[lst // 512, lst % 512] = bufs[p].numpy()
            ok &= bool(np.array_equal(data[lst // 512, lst % 512], lv.rho[lst // 512, lst % 512]))
            ok &= len(rl) + len(rr) > 0
        ret[rank] = ok
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_moves_exact_ghost_data():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs) and ret.get(0) and ret.get(1)


@pytest.mark.parametrize("theta", [0.34, 0.5, 0.3, 0.25])
def test_node_costs_match_oracle_counts(theta):
    """octo_fmm_node_costs (host-side partition weights) = the oracle's brute
    force interaction counts summed over each node's 512 cells, per class."""
    import oracle
    from paper_1908_03121_b200.binding import node_costs
    tr = synth.config_random_amr(4, 3, 0.45)
    for lv in tr.levels[1:]:
        got = node_costs(theta, lv.refined, lv.neighbors)
        tn = np.repeat(np.arange(lv.n_nodes, dtype=np.int64), 512)
        tc = np.tile(np.arange(512, dtype=np.int32), lv.n_nodes)
        want = oracle.count_interactions(tr, lv.level, theta, targets=(tn, tc)).reshape(lv.n_nodes, 512, 3).sum(1)
        assert np.array_equal(got, want), lv.level


def test_cost_weighted_partition_balances_cost():
    """Partitions weighted by node_costs x COST_PER_INTERACTION balance the
    modelled cost of a V1309 level to within one node's cost."""
    from paper_1908_03121_b200.binding import node_costs
    tr = synth.config_v1309(11)
    for lv in tr.levels[8:]:
        w = synth.cost_weights(node_costs(0.34, lv.refined, lv.neighbors))
        for P in (2, 4, 8):
            own = synth.partition_level(lv.refined, P, weights=w)
            per = np.array([w[own == r].sum() for r in range(P)])
            assert per.max() - per.mean() <= w.max() + 1e-9, (lv.level, P)

"""Multi-rank GPU check (run under torchrun): the ghost-exchange path must
reproduce the single-rank results BITWISE on the owned rows (exact ghost
copies, fixed per-cell order; SURVEY 8(e) invariant), over several steps with
different densities reloaded between them (stale ghosts or a reused
double-buffer half would show up).

OCTO_MP_BOOT=nccl (default): one rank per GPU, torch NCCL process group, the
library's own NCCL communicator (transport OCTO_XCHG=puts|nccl).
OCTO_MP_BOOT=gloo: torch gloo process group, ranks may share GPUs (rank r on
device r % device_count), the one-sided exchange bootstrapped through the
caller's allgather (OCTO_EXTERNAL_BOOTSTRAP) -- how a 1-GPU box runs 2 ranks
and a 4-GPU box 8.
Exit code 0 on success.  Usage: torchrun --nproc-per-node N tests/mp_fmm_run.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1908_03121_b200 as P  # noqa: E402
from paper_1908_03121_b200.levels import upward, load_tree, upward_shard  # noqa: E402


BOOT = os.environ.get("OCTO_MP_BOOT", "nccl")
STEPS = int(os.environ.get("OCTO_MP_STEPS", "4"))


def make_handle(rank, ws, dev, theta=0.34):
    if BOOT == "gloo":
        return P.OctoFMM(theta, device=dev, rank=rank, nranks=ws, allgather=P.gloo_allgather())
    obj = [P.nccl_unique_id() if rank == 0 else None]   # one fresh id per communicator
    dist.broadcast_object_list(obj, src=0)
    return P.OctoFMM(theta, device=dev, rank=rank, nranks=ws, nccl_id=obj[0])


def allreduce_sum(t):
    if BOOT == "gloo":   # gloo reduces host tensors
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)
    else:
        dist.all_reduce(t)


def scaled(d, s):
    """Step data: every mass and moment times s (centres unchanged), so
    m > 0 and mom[0] == mono still hold exactly."""
    return dict(mono=d["mono"] * s, com=d["com"], mom=None if d["mom"] is None else d["mom"] * s)


def compare(f, ref, tree, owner, rank, tag):
    ok = True
    for lv in tree.levels:
        mine = np.nonzero(owner[lv.level] == rank)[0]
        L = torch.zeros((20, len(mine), 512), dtype=torch.float64, device="cuda")
        Lc = torch.zeros((3, len(mine), 512), dtype=torch.float64, device="cuda")
        f.get_expansions(lv.level, L, Lc)
        RL = torch.zeros((20, lv.n_nodes, 512), dtype=torch.float64, device="cuda")
        RLc = torch.zeros((3, lv.n_nodes, 512), dtype=torch.float64, device="cuda")
        ref.get_expansions(lv.level, RL, RLc)
        idx = torch.from_numpy(mine).cuda()
        same = torch.equal(L, RL[:, idx]) and torch.equal(Lc, RLc[:, idx])
        if not same:
            d = (L - RL[:, idx]).abs().max().item()
            print(f"rank {rank} {tag} level {lv.level}: MISMATCH max|d| = {d:.3e}", flush=True)
        ok &= same
    return ok


def sharded_case(rank, ws, local, model):
    """configs[4] path: subtree shards, rank subsets (owned + ghost nodes only),
    device densities and a sharded FMM step 1 -- bitwise equal to one rank
    holding the whole tree."""
    tree = model.tree(structure_only=True)
    owners, l0 = synth.shard_owners(tree, ws)
    f = make_handle(rank, ws, local)
    tables, data = upward_shard(f, tree, model, owners, l0, rank, allreduce_sum)
    one = [np.zeros(lv.n_nodes, np.int32) for lv in tree.levels]
    ref_h = P.OctoFMM(0.34, device=local)
    rt, rd = upward_shard(ref_h, tree, model, one, l0, 0, lambda t: None)
    ok = True
    for step in range(2):
        s = 1.0 + 0.5 * step
        for lv in tree.levels:
            ijk, ref, nb, ow = tables[lv.level]
            d = scaled(data[lv.level], s)
            f.load_level(lv.level, lv.h, tree.origin, ijk, ref, nb, ow, d["mono"], d["com"], d["mom"])
            ijk, rf, nb, ow = rt[lv.level]
            d = scaled(rd[lv.level], s)
            ref_h.load_level(lv.level, lv.h, tree.origin, ijk, rf, nb, None, d["mono"], d["com"], d["mom"])
        f.compute_interactions()
        ref_h.compute_interactions()
        for lv in tree.levels:
            mine = np.nonzero(owners[lv.level] == rank)[0]
            L = torch.zeros((20, len(mine), 512), dtype=torch.float64, device="cuda")
            Lc = torch.zeros((3, len(mine), 512), dtype=torch.float64, device="cuda")
            f.get_expansions(lv.level, L, Lc)
            RL = torch.zeros((20, lv.n_nodes, 512), dtype=torch.float64, device="cuda")
            RLc = torch.zeros((3, lv.n_nodes, 512), dtype=torch.float64, device="cuda")
            ref_h.get_expansions(lv.level, RL, RLc)
            idx = torch.from_numpy(mine).cuda()
            same = torch.equal(L, RL[:, idx]) and torch.equal(Lc, RLc[:, idx])
            if not same:
                dd = (L - RL[:, idx]).abs().max().item()
                print(f"rank {rank} sharded step {step} level {lv.level}: MISMATCH max|d| = {dd:.3e}", flush=True)
            ok &= same
    f.sync()
    f.close()
    ref_h.close()
    if rank == 0:
        print(f"sharded case: l0 {l0}, subsets {[len(t[0]) for t in tables]}", flush=True)
    return ok


def main():
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    if BOOT == "gloo":
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    names = os.environ.get("OCTO_MP_TREES", "c3,amr,v1309-11,v1309-13").split(",")
    trees = {"c3": lambda: synth.config_c3(), "amr": lambda: synth.config_random_amr(5, 3, 0.45),
             "v1309-11": lambda: synth.config_v1309(11), "v1309-13": lambda: synth.config_v1309(13)}
    for name in names:
        tree = trees[name]()
        # the bench's partition: per-node interaction counts x class cost
        owner = {lv.level: synth.partition_level(
            lv.refined, ws, weights=synth.cost_weights(P.node_costs(0.34, lv.refined, lv.neighbors))
            if lv.level >= 1 else None) for lv in tree.levels}
        f = make_handle(rank, ws, local)
        data = upward(f, tree)
        ref = P.OctoFMM(0.34, device=local)
        for step in range(STEPS):
            # new densities every step (ghosts must be refreshed, both halves
            # of the double-buffered arena get reused)
            d = [scaled(x, 1.0 + 0.25 * step) for x in data]
            load_tree(f, tree, d, owner=owner)
            f.compute_interactions()
            load_tree(ref, tree, d)
            ref.compute_interactions()
            ok &= compare(f, ref, tree, owner, rank, f"{name} step {step}")
        # per-level calls are collective and reuse the all-level plan
        for lv in tree.levels:
            f.compute_interactions(lv.level)
        ok &= compare(f, ref, tree, owner, rank, f"{name} per-level")
        f.sync()
        f.close()
        ref.close()
    if os.environ.get("OCTO_MP_SHARDED", "1") == "1":
        ok &= sharded_case(rank, ws, local, synth.V1309(12, 0.4))
    t = torch.tensor([1 if ok else 0])
    if BOOT != "gloo":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("MULTI-RANK BITWISE", "PASS" if t.item() == 1 else "FAIL", f"world={ws} boot={BOOT} steps={STEPS}",
              flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 1 else 1)


if __name__ == "__main__":
    main()

"""Multi-rank GPU check (run under torchrun, one rank per GPU): the NCCL
ghost-exchange path must reproduce the single-rank results BITWISE on the
owned rows (exact ghost copies, fixed per-cell order; SURVEY 8(e) invariant).
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


def sharded_case(rank, ws, local, model):
    """configs[4] path: subtree shards, rank subsets (owned + ghost nodes only),
    device densities and a sharded FMM step 1 -- bitwise equal to one rank
    holding the whole tree."""
    tree = model.tree(structure_only=True)
    owners, l0 = synth.shard_owners(tree, ws)
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    f = P.OctoFMM(0.34, device=local, rank=rank, nranks=ws, nccl_id=obj[0])
    tables, data = upward_shard(f, tree, model, owners, l0, rank, lambda t: dist.all_reduce(t))
    for lv in tree.levels:
        ijk, ref, nb, ow = tables[lv.level]
        d = data[lv.level]
        f.load_level(lv.level, lv.h, tree.origin, ijk, ref, nb, ow, d["mono"], d["com"], d["mom"])
    f.compute_interactions()
    one = [np.zeros(lv.n_nodes, np.int32) for lv in tree.levels]
    ref_h = P.OctoFMM(0.34, device=local)
    rt, rd = upward_shard(ref_h, tree, model, one, l0, 0, lambda t: None)
    for lv in tree.levels:
        ijk, rf, nb, ow = rt[lv.level]
        d = rd[lv.level]
        ref_h.load_level(lv.level, lv.h, tree.origin, ijk, rf, nb, None, d["mono"], d["com"], d["mom"])
    ref_h.compute_interactions()
    ok = True
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
            print(f"rank {rank} sharded level {lv.level}: MISMATCH max|d| = {dd:.3e}", flush=True)
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
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for name, tree in (("c3", synth.config_c3()), ("amr", synth.config_random_amr(5, 3, 0.45)),
                       ("v1309-11", synth.config_v1309(11)), ("v1309-13 (bench)", synth.config_v1309(13))):
        # the bench's partition: per-node interaction counts x class cost
        owner = {lv.level: synth.partition_level(
            lv.refined, ws, weights=synth.cost_weights(P.node_costs(0.34, lv.refined, lv.neighbors))
            if lv.level >= 1 else None) for lv in tree.levels}
        obj = [P.nccl_unique_id() if rank == 0 else None]   # one fresh id per communicator
        dist.broadcast_object_list(obj, src=0)
        f = P.OctoFMM(0.34, device=local, rank=rank, nranks=ws, nccl_id=obj[0])
        data = upward(f, tree)
        load_tree(f, tree, data, owner=owner)
        f.compute_interactions()
        f.compute_interactions()    # twice: ghosts refreshed, results identical
        ref = P.OctoFMM(0.34, device=local)
        load_tree(ref, tree, data)
        ref.compute_interactions()
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
                print(f"rank {rank} {name} level {lv.level}: MISMATCH max|d| = {d:.3e}", flush=True)
            ok &= same
        f.sync()
        f.close()
        ref.close()
    ok &= sharded_case(rank, ws, local, synth.V1309(12, 0.4))
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("MULTI-RANK BITWISE", "PASS" if t.item() == 1 else "FAIL", f"world={ws}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 1 else 1)


if __name__ == "__main__":
    main()

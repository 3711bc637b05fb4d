"""Level-input marshalling for synthetic octrees (structure tables on the host,
data on the device).  `upward` runs FMM step 1 (P2M + M2M) with the
library's kernels and returns every level's load_level inputs as device
tensors; `load_tree` ingests them.  PyTorch is used for device memory only."""
from __future__ import annotations

import numpy as np


def _pack(ijk):
    ijk = np.asarray(ijk, dtype=np.int64)
    return ijk[:, 0] | (ijk[:, 1] << 21) | (ijk[:, 2] << 42)


def children_table(parent, child) -> tuple[np.ndarray, np.ndarray]:
    """(parent_rows, children[n_refined][8]) with child node indices per octant
    o = ox + 2 oy + 4 oz (structure only)."""
    rows = np.nonzero(parent.refined)[0].astype(np.int32)
    keys = _pack(child.ijk)
    order = np.argsort(keys)
    sk = keys[order]
    oct_ = np.array([[o & 1, (o >> 1) & 1, (o >> 2) & 1] for o in range(8)], dtype=np.int64)
    want = (2 * parent.ijk[rows].astype(np.int64)[:, None, :] + oct_[None, :, :]).reshape(-1, 3)
    wk = _pack(want)
    pos = np.minimum(np.searchsorted(sk, wk), len(sk) - 1)
    if not np.all(sk[pos] == wk):
        raise ValueError("refined node without its 8 children on the next level")
    return rows, order[pos].reshape(-1, 8).astype(np.int32)


def upward(fmm, tree, stream=None):
    """Device P2M + M2M for every level; returns [dict(mono, com, mom)] (torch
    CUDA float64 tensors in the load_level layout), index = level."""
    import torch
    out = [None] * len(tree.levels)
    for lv in reversed(tree.levels):
        n, nr = lv.n_nodes, lv.n_refined
        rho = torch.from_numpy(np.ascontiguousarray(lv.rho)).cuda()
        mono = torch.empty((n, 512), dtype=torch.float64, device="cuda")
        fmm.p2m(rho, lv.h, mono, stream)
        com = torch.empty((3, nr, 512), dtype=torch.float64, device="cuda") if nr else None
        mom = torch.empty((20, nr, 512), dtype=torch.float64, device="cuda") if nr else None
        if nr:
            ch = tree.levels[lv.level + 1]
            co = out[lv.level + 1]
            rows, kids = children_table(lv, ch)
            fmm.m2m(rows, kids, ch.ijk, ch.refined, ch.h, tree.origin, co["mono"], co["com"], co["mom"],
                    mono, com, mom, stream)
        out[lv.level] = dict(mono=mono, com=com, mom=mom)
    return out


def load_tree(fmm, tree, data, levels=None, owner=None, stream=None):
    """load_level for every level (or `levels`) from upward()'s tensors."""
    for lv in tree.levels:
        if levels is not None and lv.level not in levels:
            continue
        d = data[lv.level]
        own = None if owner is None else owner[lv.level]
        fmm.load_level(lv.level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, own, d["mono"], d["com"],
                       d["mom"], stream)


class _Lv:
    """Minimal level view (structure) for children_table / upward."""

    def __init__(self, level, h, ijk, refined):
        self.level, self.h = level, h
        self.ijk, self.refined = ijk, refined
        self.n_nodes, self.n_refined = int(ijk.shape[0]), int(refined.sum())


def device_rho(model, origin, lv, leaf_rows, chunk=65536):
    """Densities [n][512] of the nodes of view lv on the device (rows of
    refined nodes 0): model.density_torch at the leaf nodes' cell centres,
    generated in chunks of nodes (input synthesis, not FMM arithmetic)."""
    import torch
    loc = torch.stack(torch.meshgrid(torch.arange(8), torch.arange(8), torch.arange(8), indexing="ij"), -1)
    loc = loc.permute(2, 1, 0, 3).reshape(512, 3).to(torch.float64).cuda()   # local index lx + 8 ly + 64 lz
    org = torch.as_tensor(np.asarray(origin, np.float64)).cuda()
    rho = torch.zeros((lv.n_nodes, 512), dtype=torch.float64, device="cuda")
    rows = torch.as_tensor(np.asarray(leaf_rows, np.int64)).cuda()
    ijk = torch.as_tensor(lv.ijk[np.asarray(leaf_rows, np.int64)].astype(np.float64)).cuda()
    for a in range(0, rows.numel(), chunk):
        g = 8.0 * ijk[a:a + chunk, None, :] + loc[None, :, :] + 0.5
        rho[rows[a:a + chunk]] = model.density_torch(org + g * lv.h)
    return rho


def upward_shard(fmm, tree, model, owners, l0, rank, allreduce_sum_, stream=None):
    """FMM step 1 for one rank of a subtree-sharded tree (synth.shard_owners):
    device densities (model.density_torch), P2M + M2M with the library's
    kernels over the rank's own subtrees (levels >= l0, no communication),
    the level-l0 moments summed over ranks (allreduce_sum_(tensor) in place;
    each row has exactly one non-zero contributor, so the sum is exact), then
    the coarse levels < l0 on every rank.  Returns (tables, data) per level:
    levels >= l0 in the rank-subset layout (owned + ghost nodes, ghost rows
    zero: the exchange delivers them), levels < l0 whole."""
    import torch
    import synth
    nl = len(tree.levels)
    own = {}
    # ---- own subtrees, bottom-up
    for l in range(nl - 1, l0 - 1, -1):
        lv = tree.levels[l]
        oi = np.nonzero(owners[l] == rank)[0]
        v = _Lv(l, lv.h, lv.ijk[oi], lv.refined[oi])
        rho = device_rho(model, tree.origin, v, np.nonzero(v.refined == 0)[0])
        mono = torch.empty((v.n_nodes, 512), dtype=torch.float64, device="cuda")
        if v.n_nodes:
            fmm.p2m(rho, lv.h, mono, stream)
        del rho
        com = torch.zeros((3, v.n_refined, 512), dtype=torch.float64, device="cuda") if v.n_refined else None
        mom = torch.zeros((20, v.n_refined, 512), dtype=torch.float64, device="cuda") if v.n_refined else None
        if v.n_refined:
            ch = own[l + 1]
            rows, kids = children_table(v, ch["view"])
            fmm.m2m(rows, kids, ch["view"].ijk, ch["view"].refined, ch["view"].h, tree.origin, ch["mono"], ch["com"],
                    ch["mom"], mono, com, mom, stream)
        own[l] = dict(view=v, idx=oi, mono=mono, com=com, mom=mom)
        if l + 1 in own:   # level l+1 is no longer needed by M2M
            own[l + 1]["done"] = True
    # ---- level l0 on every rank (sum of the disjoint owned rows)
    lv = tree.levels[l0]
    full = dict(mono=torch.zeros((lv.n_nodes, 512), dtype=torch.float64, device="cuda"))
    rs = lv.rslot()
    full["mono"][torch.as_tensor(own[l0]["idx"]).cuda()] = own[l0]["mono"]
    if lv.n_refined:
        full["com"] = torch.zeros((3, lv.n_refined, 512), dtype=torch.float64, device="cuda")
        full["mom"] = torch.zeros((20, lv.n_refined, 512), dtype=torch.float64, device="cuda")
        oi = own[l0]["idx"]
        ro = torch.as_tensor(rs[oi[lv.refined[oi] == 1]]).cuda()
        if ro.numel():
            full["com"][:, ro] = own[l0]["com"]
            full["mom"][:, ro] = own[l0]["mom"]
    else:
        full["com"] = full["mom"] = None
    torch.cuda.synchronize()
    for k in ("mono", "com", "mom"):
        if full[k] is not None:
            allreduce_sum_(full[k])
    # ---- coarse levels (whole, every rank)
    coarse = {l0: full}
    for l in range(l0 - 1, -1, -1):
        lv = tree.levels[l]
        v = _Lv(l, lv.h, lv.ijk, lv.refined)
        rho = device_rho(model, tree.origin, v, np.nonzero(lv.refined == 0)[0])
        mono = torch.empty((lv.n_nodes, 512), dtype=torch.float64, device="cuda")
        fmm.p2m(rho, lv.h, mono, stream)
        nr = lv.n_refined
        com = torch.zeros((3, nr, 512), dtype=torch.float64, device="cuda") if nr else None
        mom = torch.zeros((20, nr, 512), dtype=torch.float64, device="cuda") if nr else None
        if nr:
            ch = tree.levels[l + 1]
            rows, kids = children_table(lv, ch)
            co = coarse[l + 1]
            fmm.m2m(rows, kids, ch.ijk, ch.refined, ch.h, tree.origin, co["mono"], co["com"], co["mom"],
                    mono, com, mom, stream)
        coarse[l] = dict(mono=mono, com=com, mom=mom)
    # ---- load_level inputs
    tables, data = [None] * nl, [None] * nl
    for l in range(nl):
        lv = tree.levels[l]
        if l < l0:
            tables[l] = (lv.ijk, lv.refined, lv.neighbors, owners[l].astype(np.int32))
            data[l] = coarse[l]
            continue
        idx = synth.rank_subset(lv.neighbors, owners[l], rank)
        ijk, ref, nb, ow = synth.subset_tables(lv, owners[l], idx)
        tables[l] = (ijk, ref, nb, ow)
        o = own[l]
        pos = torch.as_tensor(np.searchsorted(idx, o["idx"])).cuda()
        mono = torch.zeros((idx.size, 512), dtype=torch.float64, device="cuda")
        mono[pos] = o["mono"]
        nr = int(ref.sum())
        com = mom = None
        if nr:
            rsub = np.cumsum(ref.astype(np.int64)) - 1
            opos = np.searchsorted(idx, o["idx"][o["view"].refined == 1])
            rp = torch.as_tensor(rsub[opos]).cuda()
            com = torch.zeros((3, nr, 512), dtype=torch.float64, device="cuda")
            mom = torch.zeros((20, nr, 512), dtype=torch.float64, device="cuda")
            if rp.numel():
                com[:, rp] = o["com"]
                mom[:, rp] = o["mom"]
        data[l] = dict(mono=mono, com=com, mom=mom)
        own[l] = None
    torch.cuda.synchronize()
    return tables, data

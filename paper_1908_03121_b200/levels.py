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

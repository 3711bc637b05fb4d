"""Oracle-sized pieces of a tree too large for the oracle (test infrastructure).

For sampled target nodes of a big structure-only tree, `mini_tree` keeps each
target's 27-node neighbourhood at its level plus the complete subtrees below
the kept nodes (their moments need every descendant), with host densities at
the kept leaf cells.  A target's same-level result depends on nothing else
(its partners lie in the 27 neighbours, C1; their moments on their subtrees,
C3), so the oracle run on the mini tree gives the full tree's values."""
import numpy as np

import synth
from synth.trees import Level, Tree, neighbor_table, LOCAL_XYZ


def _pack(ijk):
    ijk = np.asarray(ijk, np.int64)
    return ijk[:, 0] | (ijk[:, 1] << 21) | (ijk[:, 2] << 42)


def mini_tree(tree, density, targets):
    """targets: list of (level, node index in tree).  Returns (mini Tree, maps)
    with maps[level] = full node index of each mini node (sorted)."""
    nl = len(tree.levels)
    keep = [set() for _ in range(nl)]
    for l, t in targets:
        keep[l].update(int(x) for x in tree.levels[l].neighbors[t] if x >= 0)
    for l in range(nl - 1):
        lv, ch = tree.levels[l], tree.levels[l + 1]
        ref = [q for q in keep[l] if lv.refined[q]]
        if not ref:
            continue
        keys = _pack(ch.ijk)
        order = np.argsort(keys)
        sk = keys[order]
        oct_ = np.array([[o & 1, (o >> 1) & 1, (o >> 2) & 1] for o in range(8)], np.int64)
        want = _pack((2 * lv.ijk[ref].astype(np.int64)[:, None, :] + oct_[None]).reshape(-1, 3))
        pos = np.searchsorted(sk, want)
        assert np.all(sk[pos] == want)
        keep[l + 1].update(int(x) for x in order[pos])
    levels, maps = [], []
    for l in range(nl):
        lv = tree.levels[l]
        idx = np.array(sorted(keep[l]), dtype=np.int64)
        ijk = lv.ijk[idx].astype(np.int32)
        ref = lv.refined[idx].astype(np.uint8)
        rho = np.zeros((idx.size, 512))
        leaf = np.nonzero(ref == 0)[0]
        if leaf.size:
            g = 8 * ijk[leaf].astype(np.int64)[:, None, :] + LOCAL_XYZ[None]
            cen = tree.origin[None, None, :] + (g + 0.5) * lv.h
            rho[leaf] = density(cen.reshape(-1, 3)).reshape(leaf.size, 512)
        nb = neighbor_table(ijk, l) if idx.size else np.zeros((0, 27), np.int32)
        levels.append(Level(level=l, h=lv.h, ijk=ijk, refined=ref, neighbors=nb, rho=rho))
        maps.append(idx)
    return Tree(origin=tree.origin, width=tree.width, levels=levels), maps


def pick_targets(tree, rng, per_kind=2):
    """Sampled target nodes of every kind the step has: refined targets (M2L),
    leaf targets with only leaf neighbours (P2P) and leaf targets next to a
    refined node (mixed + P2P), from the finest levels that hold them."""
    out = []
    want = {"ref": per_kind, "leaf": per_kind, "mixed": per_kind}
    for lv in reversed(tree.levels[1:]):
        ref = lv.refined.astype(bool)
        nbref = np.zeros(lv.n_nodes, bool)
        nb = lv.neighbors
        valid = nb >= 0
        nbref = np.any(valid & ref[np.where(valid, nb, 0)], axis=1)
        kinds = {"ref": np.nonzero(ref)[0], "mixed": np.nonzero(~ref & nbref)[0],
                 "leaf": np.nonzero(~ref & ~nbref)[0]}
        for k, cand in kinds.items():
            if want[k] > 0 and cand.size:
                take = rng.choice(cand, size=min(want[k], cand.size), replace=False)
                out += [(lv.level, int(t), k) for t in take]
                want[k] -= take.size
        if not any(want.values()):
            break
    return out

"""Sharding an octree over ranks when no rank can hold the whole tree
(configs[4]).  Structure only: owners, per-rank node subsets
and their neighbour tables.

* Subtree partition: below a level l0 every node belongs to the rank that
  owns its level-l0 ancestor, and the level-l0 nodes are cut into contiguous
  Morton chunks (space-filling curve) of equal SUBTREE weight, so
  a rank's refined nodes have their children on the same rank (FMM step 1 on
  a shard needs no communication above l0).  Levels < l0 are few and small:
  every rank holds them whole, partitioned per level (partition.py).
* Rank subset of a level: the owned nodes plus their same-level neighbours
  (the ghosts whose cells the exchange delivers), in Morton order, with the
  neighbour table restricted to the subset (-1 outside it).  The library
  computes only owned nodes and reads ghost rows only within the stencil's
  reach, which the exchange fills; ghost input rows are never read.
"""
from __future__ import annotations

import numpy as np

from .partition import REFINED_WEIGHT, partition_level
from .trees import _pack


def _parent_index(parent_ijk: np.ndarray, child_ijk: np.ndarray) -> np.ndarray:
    """Index (into parent_ijk) of the parent of every child node."""
    pk = _pack(parent_ijk)
    order = np.argsort(pk)
    sk = pk[order]
    ck = _pack(child_ijk.astype(np.int64) >> 1)
    pos = np.minimum(np.searchsorted(sk, ck), len(sk) - 1)
    if not np.all(sk[pos] == ck):
        raise ValueError("child node without a parent on the level above")
    return order[pos]


def subtree_weights(tree, node_weights=None) -> list:
    """W[l][q] = sum over the subtree of node q at level l of the node cost
    weights (node_weights[l], default refined REFINED_WEIGHT, leaf 1)."""
    W = [None] * len(tree.levels)
    for lv in reversed(tree.levels):
        w = (np.where(lv.refined.astype(bool), REFINED_WEIGHT, 1.0) if node_weights is None
             else np.asarray(node_weights[lv.level], float).copy())
        if lv.level + 1 < len(tree.levels) and W[lv.level + 1] is not None:
            ch = tree.levels[lv.level + 1]
            np.add.at(w, _parent_index(lv.ijk, ch.ijk), W[lv.level + 1])
        W[lv.level] = w
    return W


def choose_l0(tree, nranks: int, W=None, slack: float = 20.0) -> int:
    """Coarsest level whose largest subtree weighs at most total / (slack *
    nranks) (so the contiguous cut is balanced to ~1/slack) and that has at
    least 4 nodes per rank."""
    W = subtree_weights(tree) if W is None else W
    total = float(W[0].sum())
    for lv in tree.levels:
        if lv.n_nodes >= 4 * nranks and float(W[lv.level].max()) <= total / (slack * nranks):
            return lv.level
    return tree.max_level


def shard_owners(tree, nranks: int, l0: int | None = None, node_weights=None):
    """(owners per level, l0): subtree partition at l0, per-level partition above
    (node_weights: per-level node cost weights, e.g. partition.cost_weights)."""
    W = subtree_weights(tree, node_weights)
    if l0 is None:
        l0 = choose_l0(tree, nranks, W)
    owners = [None] * len(tree.levels)
    for lv in tree.levels:
        if lv.level < l0:
            owners[lv.level] = partition_level(lv.refined, nranks,
                                               None if node_weights is None else node_weights[lv.level])
        elif lv.level == l0:
            owners[lv.level] = partition_level(lv.refined, nranks, weights=W[l0])
        else:
            par = tree.levels[lv.level - 1]
            owners[lv.level] = owners[lv.level - 1][_parent_index(par.ijk, lv.ijk)]
    return owners, l0


def rank_subset(neighbors: np.ndarray, owner: np.ndarray, rank: int) -> np.ndarray:
    """Sorted node indices of the owned nodes and their same-level neighbours."""
    own = np.nonzero(owner == rank)[0]
    nb = neighbors[own].reshape(-1)
    return np.union1d(own, nb[nb >= 0]).astype(np.int64)


def subset_tables(lv, owner: np.ndarray, idx: np.ndarray):
    """(ijk, refined, neighbors, owner) of the subset idx of level lv, the
    neighbour table remapped to subset positions (-1 outside the subset)."""
    inv = np.full(lv.n_nodes + 1, -1, dtype=np.int64)   # slot n maps the -1 entries
    inv[idx] = np.arange(idx.size)
    nb = lv.neighbors[idx]
    nbs = inv[np.where(nb >= 0, nb, lv.n_nodes)].astype(np.int32)
    return (np.ascontiguousarray(lv.ijk[idx]), np.ascontiguousarray(lv.refined[idx]), np.ascontiguousarray(nbs),
            np.ascontiguousarray(owner[idx].astype(np.int32)))

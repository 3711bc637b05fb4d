"""Space-filling-curve partition of an octree level across ranks (structure only).

P:L420-421: "octree nodes are distributed onto the compute nodes using a space
filling curve".  Nodes of a level are already in Morton order (trees.py), so a
partition is a list of contiguous chunks balanced by a per-node cost weight
(a refined node costs ~11x a leaf node, so counts alone do not
balance).  The weights here are structural estimates; they only affect load
balance, never results (results are bitwise independent of the partition).
"""
from __future__ import annotations

import numpy as np

# relative cost of a refined (multipole) node vs a leaf (monopole) node, from
# the measured per-kernel device times of one step of the V1309 level-13 bench
# (M2L 4.91 ms over 1,265 refined nodes vs P2P + mixed 3.18 ms over 8,856 leaf
# nodes on one B200: 3.88 us vs 0.36 us per node)
REFINED_WEIGHT = 11.0


# device time per interaction by class (P2P, M2L + Lc, mixed) relative to P2P,
# measured on one B200 (V1309 level 13: kernel time / interactions: 0.43, 10.9
# and 11.4 ps); with the per-node counts of the library's octo_fmm_node_costs
# this is the cost weight of SURVEY 8(e) e1 (interaction count x class cost)
COST_PER_INTERACTION = np.array([1.0, 25.5, 26.5])


def cost_weights(counts: np.ndarray) -> np.ndarray:
    """Per-node cost weights from per-node interaction counts (n, 3)."""
    return np.asarray(counts, float) @ COST_PER_INTERACTION


def partition_level(refined: np.ndarray, nranks: int, weights: np.ndarray | None = None) -> np.ndarray:
    """owner[n] in [0, nranks): contiguous Morton chunks of ~equal weight."""
    n = int(refined.shape[0])
    if nranks <= 1 or n == 0:
        return np.zeros(n, dtype=np.int32)
    w = np.where(refined.astype(bool), REFINED_WEIGHT, 1.0) if weights is None else np.asarray(weights, float)
    c = np.cumsum(w)
    total = c[-1]
    # node q goes to the rank whose weight interval contains the node's midpoint
    mid = c - 0.5 * w
    owner = np.minimum((mid / total * nranks).astype(np.int64), nranks - 1)
    return owner.astype(np.int32)


def ghost_plan(neighbors: np.ndarray, owner: np.ndarray, rank: int) -> np.ndarray:
    """Node indices owned by other ranks that are among the 26 neighbours of a
    node owned by `rank` (the ghost nodes this rank must receive)."""
    mine = np.nonzero(owner == rank)[0]
    if mine.size == 0:
        return np.zeros(0, dtype=np.int64)
    nb = neighbors[mine].reshape(-1)
    nb = nb[nb >= 0]
    nb = np.unique(nb)
    return nb[owner[nb] != rank].astype(np.int64)

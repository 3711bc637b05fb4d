"""Seeded synthetic inputs shared by the oracle tests, smoke() and bench.py.

This package holds NONE of the method's arithmetic (no moments, no
interactions, no Taylor coefficients): only octree STRUCTURE (which nodes
exist, which are refined, Morton order, neighbour tables, SFC partition) and
DENSITY fields sampled at leaf-cell centres.  Both the oracle (oracle/) and
the CUDA path (paper_1908_03121_b200/) consume what it produces; it imports
neither of them.
"""
from .trees import (Level, Tree, build_tree, NB_OFFSETS, morton_keys, config_c1, config_c2,
                    config_c3, config_v1309, config_random_amr, leaf_cells, V1309)
from .partition import partition_level, ghost_plan, cost_weights, COST_PER_INTERACTION
from .shard import shard_owners, rank_subset, subset_tables, subtree_weights, choose_l0

__all__ = ["Level", "Tree", "build_tree", "NB_OFFSETS", "morton_keys", "config_c1", "config_c2",
           "config_c3", "config_v1309", "config_random_amr", "leaf_cells", "V1309", "partition_level",
           "ghost_plan", "cost_weights", "COST_PER_INTERACTION", "shard_owners", "rank_subset", "subset_tables", "subtree_weights", "choose_l0"]

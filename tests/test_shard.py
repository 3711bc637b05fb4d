"""Host logic of the configs[4] shards (synth/shard.py, structure only, CPU):
subtree ownership, balance, rank subsets and their neighbour tables, and the
device-density generator against the host one."""
import numpy as np
import pytest

import synth
from synth.partition import REFINED_WEIGHT


@pytest.fixture(scope="module")
def tree():
    return synth.V1309(12, 0.4).tree(structure_only=True)


def _pack(ijk):
    ijk = np.asarray(ijk, np.int64)
    return ijk[:, 0] | (ijk[:, 1] << 21) | (ijk[:, 2] << 42)


def test_subtree_weights_sum_to_tree_weight(tree):
    W = synth.subtree_weights(tree)
    total = sum(float(np.where(lv.refined == 1, REFINED_WEIGHT, 1.0).sum()) for lv in tree.levels)
    for lv in tree.levels:
        # every level's subtrees cover everything at and below it
        below = sum(float(np.where(x.refined == 1, REFINED_WEIGHT, 1.0).sum()) for x in tree.levels[lv.level:])
        assert float(W[lv.level].sum()) == pytest.approx(below, rel=1e-12)
    assert float(W[0].sum()) == pytest.approx(total, rel=1e-12)


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_subtree_owners(tree, nranks):
    owners, l0 = synth.shard_owners(tree, nranks)
    # below l0 a node and its parent have the same owner (subtree partition)
    for lv in tree.levels[l0 + 1:]:
        par = tree.levels[lv.level - 1]
        pk = _pack(par.ijk)
        pos = np.searchsorted(np.sort(pk), _pack(lv.ijk.astype(np.int64) >> 1))
        parent = np.argsort(pk)[pos]
        assert np.array_equal(owners[lv.level], owners[lv.level - 1][parent])
    # every rank owns work, and the total weight is balanced to ~1/slack
    w = np.zeros(nranks)
    for lv in tree.levels:
        np.add.at(w, owners[lv.level], np.where(lv.refined == 1, REFINED_WEIGHT, 1.0))
    assert np.all(w > 0)
    assert w.max() / w.mean() < 1.15
    # owners are contiguous along the Morton order at every level >= l0
    for lv in tree.levels[l0:]:
        o = owners[lv.level]
        assert np.all(np.diff(o) >= 0)


@pytest.mark.parametrize("nranks", [2, 4])
def test_rank_subsets(tree, nranks):
    owners, l0 = synth.shard_owners(tree, nranks)
    for lv in tree.levels[l0:]:
        cover = np.zeros(lv.n_nodes, int)
        for r in range(nranks):
            idx = synth.rank_subset(lv.neighbors, owners[lv.level], r)
            ijk, ref, nb, ow = synth.subset_tables(lv, owners[lv.level], idx)
            assert np.all(np.diff(idx) > 0)                     # Morton order kept
            mine = ow == r
            cover[idx[mine]] += 1
            # owned nodes keep their whole neighbourhood, remapped to the subset
            full = lv.neighbors[idx[mine]]
            sub = nb[mine]
            assert np.array_equal(full >= 0, sub >= 0)
            assert np.array_equal(idx[sub[sub >= 0]], full[full >= 0])
            # the subset table is symmetric and consistent with the coordinates
            q, s = np.nonzero(nb >= 0)
            assert np.all(nb[nb[q, s], 26 - s] == q)
            off = np.stack([s % 3 - 1, (s // 3) % 3 - 1, s // 9 - 1], 1)
            assert np.array_equal(ijk[nb[q, s]], ijk[q] + off)
            # ghosts are exactly the non-owned neighbours of owned nodes
            gh = idx[~mine]
            nbo = lv.neighbors[idx[mine]].reshape(-1)
            assert np.array_equal(np.unique(nbo[nbo >= 0][owners[lv.level][nbo[nbo >= 0]] != r]), gh)
        assert np.all(cover == 1)                               # every node owned exactly once


def test_device_density_matches_host():
    torch = pytest.importorskip("torch")
    m = synth.V1309(13)
    x = np.random.default_rng(3).uniform(-9.0, 9.0, size=(20000, 3))
    x[:10] = m.c1 + 1e-3   # near the centres
    a = m.density(x)
    b = m.density_torch(torch.from_numpy(x)).numpy()
    assert np.max(np.abs(a - b) / a) < 1e-13

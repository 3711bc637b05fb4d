"""The mini-tree construction used for full-size parity sampling
(tests/minitree.py): the oracle on a target's neighbourhood + subtrees gives
bitwise the oracle's full-tree result (CPU)."""
import numpy as np

import oracle
import synth
from minitree import mini_tree, pick_targets


def test_mini_tree_reproduces_full_tree_oracle():
    model = synth.V1309(11, 0.0)
    tree = model.tree()
    mom = oracle.moments(tree)
    rng = np.random.default_rng(5)
    targets = pick_targets(tree, rng, per_kind=1)
    assert {k for _, _, k in targets} == {"ref", "leaf", "mixed"}
    mt, maps = mini_tree(tree, model.density, [(l, t) for l, t, _ in targets])
    assert sum(lv.n_nodes for lv in mt.levels) < sum(lv.n_nodes for lv in tree.levels) // 4
    mmom = oracle.moments(mt)
    for l, t, kind in targets:
        cells = rng.choice(512, size=12, replace=False).astype(np.int32)
        full = oracle.same_level(tree, mom, l, 0.34, targets=(np.full(12, t, np.int64), cells))
        mn = int(np.searchsorted(maps[l], t))
        mini = oracle.same_level(mt, mmom, l, 0.34, targets=(np.full(12, mn, np.int64), cells))
        for a, b in zip(full, mini):
            assert np.array_equal(a, b), (l, t, kind)

"""Pins of the oracle's opening criterion / stencil.

Paper: P:L477-479 (opening criteria, "their number is constant on each level"),
P:L485 / L523 / L555 (1074-element stencil), P:L526 (549,888 interactions per
launch).  Fixture tests/golden/paper_constants.json holds the printed values.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_paper_stencil_size_and_launch_interactions():
    pc = _gold("paper_constants.json")
    far, near, far_c, near_c = oracle.stencil_sets(0.34)
    union = far | near
    assert len(union) == pc["stencil_size"]["value"]
    assert pc["cells_per_subgrid"]["value"] * len(union) == pc["interactions_per_launch"]["value"]
    assert pc["subgrid_n"]["value"] ** 3 == pc["cells_per_subgrid"]["value"]


@pytest.mark.parametrize("theta", [0.34, 0.35, 1.0 / 3.0])
def test_1074_holds_on_the_whole_theta_interval(theta):
    # C1: the union is 1074 for every theta in [1/3, 1/sqrt(8))
    far, near, _, _ = oracle.stencil_sets(theta)
    assert len(far | near) == 1074


def test_theta_one_third_knife_edge():
    # C1 precision reading: (1/theta)^2 rounds to exactly 9.0; one ulp above admits |p|^2 = 9
    assert oracle.R2(1.0 / 3.0) == 9.0
    # an R^2 one ulp above 9 admits the parent shell |p|^2 = 9: union 1074 -> 1374
    def union(r2):
        u = set()
        for c in range(8):
            i = np.array([c & 1, (c >> 1) & 1, (c >> 2) & 1], dtype=np.int64)
            for d in np.ndindex(15, 15, 15):
                dd = np.array(d, dtype=np.int64) - 7
                if oracle.lib.oc_pair_class(r2, 0, i, i + dd):
                    u.add(tuple(dd))
        return len(u)
    assert union(9.0) == 1074
    assert union(float(np.nextafter(9.0, 10.0))) == 1374


def test_per_parity_counts_and_structure():
    for theta, nfar, nnear, ufar, unear, reach in ((0.5, 189, 26, 316, 26, 3), (0.34, 651, 92, 982, 92, 5)):
        far, near, far_c, near_c = oracle.stencil_sets(theta)
        assert len(far) == ufar and len(near) == unear
        for c in range(8):
            assert len(far_c[c]) == nfar and len(near_c[c]) == nnear
            assert not (far_c[c] & near_c[c])
            # every partner of a cell lies in the 8 children of a parent-near parent:
            # far + near + self = 8 x (number of parent-near parents)
            assert (nfar + nnear + 1) % 8 == 0
        assert max(max(abs(x) for x in d) for d in far | near) == reach
        # point symmetry d <-> -d of the union and (1,0,0) in S
        u = far | near
        assert all((-a, -b, -cc) in u for (a, b, cc) in u)
        assert (1, 0, 0) in u and (0, 0, 0) not in u
        # parity c's set maps to parity (1-c)'s set under d -> -d
        for c in range(8):
            cm = 7 - c
            assert {(-a, -b, -cc) for (a, b, cc) in far_c[c]} == far_c[cm]


def test_theta_range_reach_stays_within_26_neighbours():
    for theta in (0.25, 0.3, 0.5, 0.7, 1.0):
        far, near, _, _ = oracle.stencil_sets(theta)
        u = far | near
        if u:
            assert max(max(abs(x) for x in d) for d in u) <= 7


def test_root_rule_counts():
    # C2: root = all pairs inside the single 8^3 sub-grid with |d|^2 >= R^2
    for theta in (0.5, 0.34):
        r2 = oracle.R2(theta)
        g = np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1).reshape(-1, 3)
        d2 = np.sum((g[:, None, :] - g[None, :, :]) ** 2, axis=-1)
        expect_far = int(np.sum(d2 >= r2))
        tr = synth.build_tree(np.zeros(3), 1.0, 0, lambda l, lo, hi: np.zeros(lo.shape[0], bool),
                              lambda x: np.ones(x.shape[0]))
        # leaf root: far pairs + near pairs are all P2P
        cnt = oracle.count_interactions(tr, 0, theta)
        assert cnt[:, 0].sum() == 512 * 511
        tr2 = synth.config_c1()
        cnt2 = oracle.count_interactions(tr2, 0, theta)  # refined root: far pairs only
        assert cnt2[:, 1].sum() == expect_far and cnt2[:, 0].sum() == 0 and cnt2[:, 2].sum() == 0


@pytest.mark.parametrize("theta", [0.5, 0.34])
def test_exactly_once_coverage_uniform(theta):
    # configs[0]: level-1 pairs + 64 x root pairs = n(n-1) (closed form, golden)
    gc = _gold("coverage_counts.json")
    tr = synth.config_c1()
    c1 = oracle.count_interactions(tr, 1, theta).sum()
    c0 = oracle.count_interactions(tr, 0, theta).sum()
    assert c1 + gc["finest_pairs_per_root_pair"] * c0 == gc["ordered_pairs"]
    lev, g, _, _, _ = synth.leaf_cells(tr)
    hist = oracle.coverage(theta, lev, g)
    assert hist[1] == gc["ordered_pairs"] // 2 and hist[0] == 0 and hist[2] == 0 and hist[3] == 0


def test_exactly_once_coverage_amr():
    # C6: the AMR case rule takes every unordered pair of finest cells exactly once
    tr = synth.config_random_amr(1, 2, 0.4)
    lev, g, _, _, _ = synth.leaf_cells(tr)
    hist = oracle.coverage(0.5, lev, g)
    n = len(lev)
    assert hist[1] == n * (n - 1) // 2 and hist[0] == 0 and hist[2] == 0 and hist[3] == 0


def test_box_prune_equals_all_cells():
    # the oracle's candidate box |d|_inf <= 2 floor(R) + 1 drops nothing
    tr = synth.config_random_amr(3, 2, 0.4)
    mom = oracle.moments(tr)
    lv = tr.levels[2]
    rng = np.random.default_rng(0)
    tn = rng.integers(0, lv.n_nodes, 24)
    tc = rng.integers(0, 512, 24).astype(np.int32)
    for theta in (0.5, 0.34):
        a = oracle.same_level(tr, mom, 2, theta, targets=(tn, tc), prune=True)
        b = oracle.same_level(tr, mom, 2, theta, targets=(tn, tc), prune=False)
        np.testing.assert_allclose(a[0], b[0], rtol=1e-13, atol=1e-13 * np.abs(b[2][:, :20]).max())
        np.testing.assert_allclose(a[1], b[1], rtol=1e-13, atol=1e-13 * np.abs(b[2][:, 20:]).max() + 1e-300)

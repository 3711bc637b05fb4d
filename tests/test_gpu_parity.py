"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by
element on the same seeded inputs (normwise and per-cell
errors <= 1e-12, the north star's FP64 tolerance).

Sizes: configs[0] (C1) and configs[2] (C3) whole levels (several tiles, ragged
AMR boundaries), random AMR trees, and the bench configuration (V1309, max
level 13) on sampled target cells in the launch configuration bench.py times
(all levels in one fused launch)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import api_inputs, flat_abi, get, load, oracle_layout, parity, parity_detail

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def fmm_mod(gpu):
    import paper_1908_03121_b200 as P
    return P


def _check_level(P, tree, mom, level, theta, am=True):
    f = P.OctoFMM(theta, am_correction=am)
    load(f, tree, mom, level)
    f.compute_interactions(level)
    L, Lc = get(f, tree, level)
    oL, oLc, oab = oracle.same_level(tree, mom, level, theta)
    n = tree.levels[level].n_nodes
    if not am:
        oLc = 0 * oLc
    gL = L.reshape(20, -1).T
    gLc = Lc.reshape(3, -1).T
    nerr, cerr = parity(gL, gLc, oL, oLc, oab)
    assert nerr <= TOL and cerr <= TOL, (level, theta, nerr, cerr, parity_detail(gL, gLc, oL, oLc, oab))
    # counts reported by the library equal the oracle's enumeration
    cnt = oracle.count_interactions(tree, level, theta).sum(0)
    assert np.array_equal(f.interaction_counts(level), cnt)
    f.close()
    return L, Lc


@pytest.mark.parametrize("theta", [0.5, 0.34, 0.7])
def test_root_level(fmm_mod, theta):
    """a9 / f3: the root level (reading C2) -- refined roots (configs[0], [2])
    by M2L over far pairs, and a one-node leaf root by P2P over all pairs."""
    for tr in (synth.config_c1(0), synth.config_c3()):
        mom = oracle.moments(tr)
        _check_level(fmm_mod, tr, mom, 0, theta)
    rng = np.random.default_rng(4)
    leaf = synth.build_tree(np.zeros(3), 1.0, 0, lambda l, lo, hi: np.zeros(lo.shape[0], bool),
                            lambda x: rng.uniform(0.1, 1.0, x.shape[0]))
    _check_level(fmm_mod, leaf, oracle.moments(leaf), 0, theta)


@pytest.mark.parametrize("theta", [0.5, 0.34])
def test_c1_level1_p2p(fmm_mod, theta):
    tr = synth.config_c1(0)
    mom = oracle.moments(tr)
    _check_level(fmm_mod, tr, mom, 1, theta)


@pytest.mark.parametrize("theta", [0.5, 0.34])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_c3_polytrope_amr(fmm_mod, theta, level):
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    _check_level(fmm_mod, tr, mom, level, theta)


@pytest.mark.parametrize("theta", [0.25, 0.3])
def test_reach3_theta_all_kernels(fmm_mod, theta):
    """SURVEY 8(b) b1's theta range below 1/3 (parent reach 3: the 10^3-parent
    M2L window, the 10^3 P2P window and the global K(d) table): root, P2P
    (configs[0] level 1) and every kernel class on the polytrope AMR levels
    and a random AMR tree, element by element against the oracle."""
    tr = synth.config_c1(0)
    mom = oracle.moments(tr)
    _check_level(fmm_mod, tr, mom, 0, theta)
    _check_level(fmm_mod, tr, mom, 1, theta)
    for tr in (synth.config_c3(), synth.config_random_amr(2, 3, 0.45)):
        mom = oracle.moments(tr)
        for level in range(1, len(tr.levels)):
            _check_level(fmm_mod, tr, mom, level, theta)


@pytest.mark.parametrize("knob", [{"OCTO_MIX_TMA": "1"}, {"OCTO_P2P8": "0"}])
def test_reach3_alternative_kernels(fmm_mod, monkeypatch, knob):
    """The non-default kernel variants at parent reach 3 (theta = 0.3): the
    TMA-staged mixed kernel (tensor maps over the reach-3 halo boxes) and the
    4-targets-per-thread P2P kernel, every kernel class against the oracle."""
    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    tr = synth.config_random_amr(2, 3, 0.45)
    mom = oracle.moments(tr)
    for level in range(1, len(tr.levels)):
        _check_level(fmm_mod, tr, mom, level, 0.3)


@pytest.mark.parametrize("seed", [1, 2, 5])
def test_random_amr_all_kernels(fmm_mod, seed):
    tr = synth.config_random_amr(seed, 3, 0.45)
    mom = oracle.moments(tr)
    for level in range(1, len(tr.levels)):
        _check_level(fmm_mod, tr, mom, level, 0.34)


@pytest.mark.parametrize("knobs", [{"OCTO_CONCURRENCY": "1"}, {"OCTO_LPT": "7"}, {"OCTO_LPT": "0"},
                                   {"OCTO_M2L_UNROLL": "1"}, {"OCTO_M2L_UNROLL": "2"},
                                   {"OCTO_M2L_UNROLL": "3"}, {"OCTO_MIX_TMA": "1"}, {"OCTO_P2P8": "0"}])
def test_schedule_knobs_keep_results(fmm_mod, monkeypatch, knobs):
    """The scheduling knobs read at handle creation (stream concurrency, work
    order, M2L unroll) change timing only: all levels in one compute are
    bitwise equal to the default schedule (per-cell order is fixed) and match
    the oracle.  OCTO_MIX_TMA (TMA-staged halo boxes in the mixed kernel) sums
    staged slots first and OCTO_P2P8=0 (the 4-targets-per-thread P2P kernel)
    sums partner parities in another order: the oracle check only."""
    tr = synth.config_random_amr(2, 3, 0.45)
    mom = oracle.moments(tr)
    levels = range(1, len(tr.levels))

    def run():
        f = fmm_mod.OctoFMM(0.34)
        for l in levels:
            load(f, tr, mom, l)
        f.compute_interactions()
        out = [get(f, tr, l) for l in levels]
        f.close()
        return out
    base = run()
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    alt = run()
    for (L, Lc), (L2, Lc2) in zip(base, alt):
        if "OCTO_MIX_TMA" in knobs or "OCTO_P2P8" in knobs:   # another summation order: the oracle check below
            continue
        if "OCTO_M2L_UNROLL" in knobs:   # another schedule may round differently
            assert np.allclose(L, L2, rtol=1e-13, atol=0) and np.allclose(Lc, Lc2, rtol=1e-13, atol=1e-300)
        else:
            assert np.array_equal(L, L2) and np.array_equal(Lc, Lc2)
    for l, (L, Lc) in zip(levels, alt):
        oL, oLc, oab = oracle.same_level(tr, mom, l, 0.34)
        nerr, cerr = parity(L.reshape(20, -1).T, Lc.reshape(3, -1).T, oL, oLc, oab)
        assert nerr <= TOL and cerr <= TOL, (l, knobs, nerr, cerr)


def test_without_am_correction(fmm_mod):
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    L, Lc = _check_level(fmm_mod, tr, mom, 2, 0.34, am=False)
    assert np.all(Lc == 0)


def test_level_invariants_on_gpu_output(fmm_mod):
    """C7 on the GPU's outputs: net force and torque vanish per level."""
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    f = fmm_mod.OctoFMM(0.34)
    for level in (1, 2, 3):
        load(f, tr, mom, level)
    f.compute_interactions()
    for level in (1, 2, 3):
        L, Lc = get(f, tr, level)
        m, X, M = oracle.level_cell_arrays(tr, mom, level)
        F, T, sf, st = oracle.level_invariants(m, X, M, L.reshape(20, -1).T, Lc.reshape(3, -1).T)
        assert np.abs(F).max() <= 1e-12 * sf and np.abs(T).max() <= 1e-12 * st


def test_fused_all_levels_equals_per_level_bitwise(fmm_mod):
    tr = synth.config_random_amr(7, 3, 0.45)
    mom = oracle.moments(tr)
    lv = range(1, len(tr.levels))
    a = fmm_mod.OctoFMM(0.34)
    b = fmm_mod.OctoFMM(0.34)
    for l in lv:
        load(a, tr, mom, l)
        load(b, tr, mom, l)
        b.compute_interactions(l)
    a.compute_interactions()
    for l in lv:
        La, Lca = get(a, tr, l)
        Lb, Lcb = get(b, tr, l)
        assert np.array_equal(La, Lb) and np.array_equal(Lca, Lcb)


def test_device_inputs_and_determinism(fmm_mod):
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    a = fmm_mod.OctoFMM(0.34)
    load(a, tr, mom, 2, device=True)
    a.compute_interactions(2)
    La, Lca = get(a, tr, 2)
    b = fmm_mod.OctoFMM(0.34)
    load(b, tr, mom, 2)
    for _ in range(2):
        b.compute_interactions(2)
        Lb, Lcb = get(b, tr, 2)
        assert np.array_equal(La, Lb) and np.array_equal(Lca, Lcb)


def test_stencil_matches_oracle(fmm_mod):
    for theta in (0.5, 0.34, 0.7, 1.0 / 3.0, 0.3, 0.25):
        f = fmm_mod.OctoFMM(theta)
        st = f.stencil()
        far, near, far_c, near_c = oracle.stencil_sets(theta)
        for c in range(8):
            off, cls = st[c]
            gf = {tuple(o) for o, k in zip(off.tolist(), cls.tolist()) if k == 1}
            gn = {tuple(o) for o, k in zip(off.tolist(), cls.tolist()) if k == 2}
            assert gf == far_c[c] and gn == near_c[c]


def test_edge_cases(fmm_mod):
    P = fmm_mod
    # single isolated node (all neighbours absent) at a domain corner
    tr = synth.build_tree(np.zeros(3), 1.0, 1, lambda l, lo, hi: np.ones(lo.shape[0], bool),
                          lambda x: 0.5 + x[:, 0])
    mom = oracle.moments(tr)
    lv = tr.levels[1]
    keep = np.array([0])
    nb = np.full((1, 27), -1, np.int32)
    nb[0, 13] = 0
    f = P.OctoFMM(0.34)
    f.load_level(1, lv.h, tr.origin, lv.ijk[keep], lv.refined[keep], nb, None,
                 np.ascontiguousarray(mom[1]["m"][keep]), None, None)
    f.compute_interactions(1)
    L = np.zeros((20, 1, 512)); Lc = np.zeros((3, 1, 512))
    f.get_expansions(1, L, Lc)
    # oracle on the same single-node level
    sub = synth.Tree(origin=tr.origin, width=tr.width, levels=[tr.levels[0],
                     synth.Level(1, lv.h, lv.ijk[keep], lv.refined[keep], nb, lv.rho[keep])])
    smom = [mom[0], dict(m=mom[1]["m"][keep], X=mom[1]["X"][:0], M=mom[1]["M"][:0], rslot=np.array([-1]))]
    oL, oLc, oab = oracle.same_level(sub, smom, 1, 0.34)
    nerr, cerr = parity(L.reshape(20, -1).T, Lc.reshape(3, -1).T, oL, oLc, oab)
    assert nerr <= TOL and cerr <= TOL
    # empty level
    f.load_level(2, lv.h / 2, tr.origin, np.zeros((0, 3), np.int32), np.zeros(0, np.uint8),
                 np.zeros((0, 27), np.int32), None, np.zeros((0, 512)), None, None)
    f.compute_interactions(2)
    f.compute_interactions()
    f.sync()


def test_errors(fmm_mod):
    P = fmm_mod
    with pytest.raises(P.OctoError):
        P.OctoFMM(0.2)           # below the b1 range [0.25, 1] (parent reach 4)
    with pytest.raises(P.OctoError):
        P.OctoFMM(0.249)
    P.OctoFMM(0.25).close()      # the bottom of the range (parent reach 3)
    with pytest.raises(P.OctoError):
        P.OctoFMM(1.5)
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    lv = tr.levels[2]
    f = P.OctoFMM(0.34)
    mono, com, mm = api_inputs(tr, mom, 2)
    bad = mono.copy()
    bad[0, 0] = -1.0
    # value checks run in the ingest kernel, reported by the next synchronising call
    f.load_level(2, lv.h, tr.origin, lv.ijk, lv.refined, lv.neighbors, None, bad, com, mm)
    with pytest.raises(P.OctoError) as e:
        f.sync()
    assert e.value.code == P.binding.OCTO_EMASS
    nb = lv.neighbors.copy()
    r = int(np.nonzero(lv.refined)[0][0])
    s = [k for k in range(27) if k != 13 and nb[r, k] >= 0][0]
    nb[r, s] = -1
    with pytest.raises(P.OctoError) as e:
        f.load_level(2, lv.h, tr.origin, lv.ijk, lv.refined, nb, None, mono, com, mm)
    assert e.value.code == P.binding.OCTO_ESTRUCT
    with pytest.raises(P.OctoError):   # the root level holds exactly one node
        f.load_level(0, lv.h, tr.origin, lv.ijk, lv.refined, lv.neighbors, None, mono, com, mm)
    with pytest.raises(P.OctoError):
        f.compute_interactions(5)
    # device-side check: m <= 0 through a device pointer is reported at sync
    import torch
    badd = torch.from_numpy(bad).cuda()
    f.load_level(2, lv.h, tr.origin, lv.ijk, lv.refined, lv.neighbors, None, badd,
                 torch.from_numpy(com).cuda(), torch.from_numpy(mm).cuda())
    with pytest.raises(P.OctoError) as e:
        f.sync()
    assert e.value.code == P.binding.OCTO_EMASS


@pytest.mark.parametrize("theta", [0.34])
def test_c2_level3_sampled(fmm_mod, theta):
    """configs[1] (512 leaf sub-grids, P2P path) at full size; sampled targets."""
    tr = synth.config_c2()
    mom = oracle.moments(tr)
    f = fmm_mod.OctoFMM(theta)
    for l in (1, 2, 3):
        load(f, tr, mom, l)
    f.compute_interactions()
    rng = np.random.default_rng(0)
    for l in (1, 2, 3):
        L, Lc = get(f, tr, l)
        n = tr.levels[l].n_nodes
        tn = rng.integers(0, n, 300)
        tc = rng.integers(0, 512, 300).astype(np.int32)
        oL, oLc, oab = oracle.same_level(tr, mom, l, theta, targets=(tn, tc))
        gL, gLc = flat_abi(L, Lc, tn, tc)
        nerr, cerr = parity(gL, gLc, oL, oLc, oab)
        assert nerr <= TOL and cerr <= TOL, (l, nerr, cerr)


def test_v1309_bench_config_sampled(fmm_mod):
    """configs[3] (the bench workload) at full size, all levels in one fused
    launch as bench.py runs it; 200 sampled targets per level vs the oracle."""
    tr = synth.config_v1309(13)
    mom = oracle.moments(tr)
    f = fmm_mod.OctoFMM(0.34)
    levels = range(1, len(tr.levels))
    for l in levels:
        load(f, tr, mom, l)
    f.compute_interactions()
    rng = np.random.default_rng(1)
    for l in levels:
        L, Lc = get(f, tr, l)
        n = tr.levels[l].n_nodes
        tn = rng.integers(0, n, 200)
        tc = rng.integers(0, 512, 200).astype(np.int32)
        oL, oLc, oab = oracle.same_level(tr, mom, l, 0.34, targets=(tn, tc))
        gL, gLc = flat_abi(L, Lc, tn, tc)
        nerr, cerr = parity(gL, gLc, oL, oLc, oab)
        assert nerr <= TOL and cerr <= TOL, (l, nerr, cerr)


def test_device_upward_moments_match_oracle(fmm_mod):
    """FMM step 1 on the device (f1: P2M + M2M) vs the oracle's moments (C3)."""
    from paper_1908_03121_b200.levels import upward
    for tr in (synth.config_c3(), synth.config_random_amr(3, 3, 0.45)):
        mom = oracle.moments(tr)
        f = fmm_mod.OctoFMM(0.34)
        data = upward(f, tr)
        for lv in tr.levels:
            d = data[lv.level]
            mo = mom[lv.level]
            np.testing.assert_allclose(d["mono"].cpu().numpy(), mo["m"], rtol=1e-13, atol=0)
            if lv.n_refined:
                X = d["com"].cpu().numpy().transpose(1, 2, 0)
                M = d["mom"].cpu().numpy().transpose(1, 2, 0)
                np.testing.assert_allclose(X, mo["X"], rtol=1e-13, atol=1e-15)
                s2 = np.abs(mo["M"][..., 4:10]).max()
                s3 = np.abs(mo["M"][..., 10:20]).max()
                assert np.abs(M[..., 4:10] - mo["M"][..., 4:10]).max() <= 1e-12 * s2
                assert np.abs(M[..., 10:20] - mo["M"][..., 10:20]).max() <= 1e-12 * s3
                assert np.all(M[..., 1:4] == 0) and np.array_equal(M[..., 0], d["mono"].cpu().numpy()[lv.refined == 1])


def test_kernel_timing_and_counts(fmm_mod):
    tr = synth.config_c3()
    from paper_1908_03121_b200.levels import upward, load_tree
    f = fmm_mod.OctoFMM(0.34, timing=True)
    data = upward(f, tr)
    load_tree(f, tr, data)
    f.sync()   # runs the batched ingest of the loaded levels
    n0 = f.launch_count()
    f.compute_interactions()
    f.compute_interactions()
    ms, calls = f.kernel_times()
    assert calls == 2 and np.all(ms >= 0) and ms.sum() > 0
    assert f.launch_count() - n0 == 8   # root + m2l + mixed + p2p per call


@pytest.mark.parametrize("theta", [0.5, 0.34])
@pytest.mark.parametrize("which", ["c1", "amr"])
def test_gpu_full_gravity_solve(fmm_mod, theta, which):
    """f1 + step 2 (all levels incl. the root) + f2 on the device: the whole
    3-step FMM.  Leaf-cell Phi and g vs the oracle's full solve (parity) and
    vs direct N^2 (the SPEC bound, reading C8)."""
    from paper_1908_03121_b200.levels import upward, load_tree
    import torch
    tr = synth.config_c1(0) if which == "c1" else synth.config_random_amr(3, 2, 0.4)
    f = fmm_mod.OctoFMM(theta)
    data = upward(f, tr)
    load_tree(f, tr, data)
    f.compute_interactions()
    f.propagate()
    phis, gs = [], []
    for lv in tr.levels:
        n = lv.n_nodes
        phi = torch.zeros((n, 512), dtype=torch.float64, device="cuda")
        g = torch.zeros((3, n, 512), dtype=torch.float64, device="cuda")
        f.get_field(lv.level, phi, g)
        leaf = np.nonzero(lv.refined == 0)[0]
        if leaf.size:
            phis.append(phi.cpu().numpy()[leaf].reshape(-1))
            gs.append(g.cpu().numpy()[:, leaf].reshape(3, -1).T)
    f.sync()
    phi_g, g_g = np.concatenate(phis), np.concatenate(gs)
    phi_o, g_o, _, _ = oracle.fmm_full(tr, theta)
    assert np.abs(phi_g - phi_o).max() <= 1e-12 * np.abs(phi_o).max()
    assert np.abs(g_g - g_o).max() <= 1e-12 * np.abs(g_o).max()
    lev, gg, cen, rho, vol = synth.leaf_cells(tr)
    pd, gd = oracle.direct(cen, rho * vol)
    err = np.max(np.linalg.norm(g_g - gd, axis=1)) / np.max(np.linalg.norm(gd, axis=1))
    assert err <= 5e-2


def test_compact_results_equal_full_layout(fmm_mod):
    """get_expansions_compact (no zero padding) holds exactly the full layout's values."""
    import torch
    tr = synth.config_c3()
    mom = oracle.moments(tr)
    f = fmm_mod.OctoFMM(0.34)
    for l in (1, 2, 3):
        load(f, tr, mom, l)
    f.compute_interactions()
    for l in (1, 2, 3):
        lv = tr.levels[l]
        L, Lc = get(f, tr, l)
        nr, nf = f.compact_sizes(l)
        assert nr == lv.n_refined and nf == lv.n_nodes - lv.n_refined
        R = np.zeros((23, nr, 512))
        F = np.zeros((7, nf, 512))
        f.get_expansions_compact(l, R, F)
        ref = np.nonzero(lv.refined)[0]
        leaf = np.nonzero(lv.refined == 0)[0]
        assert np.array_equal(R[:20], L[:, ref]) and np.array_equal(R[20:], Lc[:, ref])
        assert np.array_equal(F[:4], L[:4, leaf]) and np.array_equal(F[4:], Lc[:, leaf])
        assert np.all(L[4:, leaf] == 0)
        # device destination, asynchronous host destination, and the zero-copy
        # slot-order buffers (owned refined rows first) hold the same values
        Rd = torch.zeros((23, nr, 512), dtype=torch.float64, device="cuda")
        Fd = torch.zeros((7, nf, 512), dtype=torch.float64, device="cuda")
        f.get_expansions_compact(l, Rd, Fd)
        Ra = torch.zeros((23, nr, 512), dtype=torch.float64).pin_memory()
        Fa = torch.zeros((7, nf, 512), dtype=torch.float64).pin_memory()
        f.get_expansions_compact(l, Ra, Fa, non_blocking=True)
        torch.cuda.synchronize()
        f.sync()
        assert np.array_equal(Rd.cpu().numpy(), R) and np.array_equal(Fd.cpu().numpy(), F)
        assert np.array_equal(Ra.numpy(), R) and np.array_equal(Fa.numpy(), F)
        tp, ap, no = f.expansions_ptr(l)
        assert no == nr + nf
        # taylor = rows 0..3 of every slot, then rows 4..19 of the refined slots
        Ls = torch.empty((4 * no + 16 * nr) * 512, dtype=torch.float64, device="cuda")
        Lcs = torch.empty((3, no, 512), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        import ctypes
        cudart = ctypes.CDLL("libcudart.so")
        cudart.cudaMemcpy(ctypes.c_void_p(Ls.data_ptr()), ctypes.c_void_p(tp), ctypes.c_size_t(Ls.numel() * 8), 3)
        cudart.cudaMemcpy(ctypes.c_void_p(Lcs.data_ptr()), ctypes.c_void_p(ap), ctypes.c_size_t(Lcs.numel() * 8), 3)
        Ls, Lcs = Ls.cpu().numpy(), Lcs.cpu().numpy()
        lo = Ls[:4 * no * 512].reshape(4, no, 512)
        hi = Ls[4 * no * 512:].reshape(16, nr, 512)
        assert np.array_equal(lo[:, :nr], R[:4]) and np.array_equal(hi, R[4:20]) and np.array_equal(Lcs[:, :nr], R[20:])
        assert np.array_equal(lo[:, nr:], F[:4]) and np.array_equal(Lcs[:, nr:], F[4:])


def test_c4_full_size_sampled(fmm_mod):
    """configs[4] at its full one-GPU size, in bench.py's launch configuration
    (structure-only tree, device densities, shard FMM step 1, all levels in
    one compute): sampled targets of every kind vs the oracle run on mini
    trees (the targets' neighbourhoods + subtrees, tests/minitree.py)."""
    import ctypes
    import torch
    import bench
    from minitree import mini_tree, pick_targets
    from paper_1908_03121_b200.levels import upward_shard
    torch.cuda.empty_cache()
    model = synth.V1309(15, bench.C4_R1)
    tree = model.tree(structure_only=True)
    owners, l0 = synth.shard_owners(tree, 1)
    f = fmm_mod.OctoFMM(0.34)
    tables, data = upward_shard(f, tree, model, owners, l0, 0, lambda t: None)
    for lv in tree.levels:
        ijk, ref, nb, ow = tables[lv.level]
        d = data[lv.level]
        f.load_level(lv.level, lv.h, tree.origin, ijk, ref, nb, None, d["mono"], d["com"], d["mom"])
    f.compute_interactions()
    f.sync()
    cudart = ctypes.CDLL("libcudart.so")
    rng = np.random.default_rng(11)
    targets = pick_targets(tree, rng, per_kind=8)
    assert {k for _, _, k in targets} == {"ref", "leaf", "mixed"}
    mt, maps = mini_tree(tree, model.density, [(l, t) for l, t, _ in targets])
    mom = oracle.moments(mt)
    pooled = {}   # per level, as the other sampled tests pool (C9 normwise metric over the compared cells)
    for l, t, kind in targets:
        lv = tree.levels[l]
        # slot order: owned refined nodes first, then leaf nodes (node order)
        ref = lv.refined.astype(bool)
        slot = int(ref[:t].sum()) if ref[t] else int(ref.sum()) + int((~ref[:t]).sum())
        n_owned, n_oref = lv.n_nodes, int(ref.sum())
        tp, ap, no = f.expansions_ptr(l)
        assert no == n_owned
        rows = np.zeros((23, 512))
        buf = np.zeros(512)

        def fetch(ptr, row):
            cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(ptr + 8 * row * 512),
                              ctypes.c_size_t(4096), 2)
            return buf.copy()
        for k in range(4):
            rows[k] = fetch(tp, k * n_owned + slot)
        if ref[t]:
            for k in range(4, 20):
                rows[k] = fetch(tp, 4 * n_owned + (k - 4) * n_oref + slot)
        for k in range(3):
            rows[20 + k] = fetch(ap, k * n_owned + slot)
        cells = rng.choice(512, size=48, replace=False).astype(np.int32)
        mn = int(np.searchsorted(maps[l], t))
        oL, oLc, oab = oracle.same_level(mt, mom, l, 0.34, targets=(np.full(cells.size, mn, np.int64), cells))
        gL, gLc = rows[:20, cells].T, rows[20:, cells].T
        if not ref[t]:
            oL = oL.copy()
            oL[:, 4:] = 0.0      # leaf targets keep L0, L1, Lc (C5)
        _, cerr = parity(gL, gLc, oL, oLc, oab)
        assert cerr <= TOL, (l, t, kind, cerr)
        acc = pooled.setdefault(l, [[], [], [], [], []])
        for lst, v in zip(acc, (gL, gLc, oL, oLc, oab)):
            lst.append(v)
    for l, acc in pooled.items():
        args = [np.concatenate(v) for v in acc]
        nerr, cerr = parity(*args)
        assert nerr <= TOL and cerr <= TOL, (l, nerr, cerr, parity_detail(*args))
    f.close()


def test_cuda_graph_replay_bitwise(fmm_mod):
    """One step (ingest of every level + all kernels, root on its side stream)
    captured into a CUDA graph and replayed on new inputs in the same device
    buffers gives bitwise the stream-launched results (bench.py times
    configs[0..2] this way)."""
    import torch
    tr = synth.config_random_amr(3, 3, 0.45)
    mom = oracle.moments(tr)
    levels = range(0, len(tr.levels))
    dev = {l: [torch.from_numpy(a).cuda() for a in api_inputs(tr, mom, l)] for l in levels}

    def step(f):
        for l in levels:
            lv = tr.levels[l]
            f.load_level(l, lv.h, tr.origin, lv.ijk, lv.refined, lv.neighbors, None, *dev[l])
        f.compute_interactions()

    def results(f):
        return [get(f, tr, l) for l in levels]

    f0 = fmm_mod.OctoFMM(0.34)
    step(f0)
    ref = results(f0)
    f0.close()
    f = fmm_mod.OctoFMM(0.34)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            step(f)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(f)
    for l in levels:   # new inputs in the same buffers (masses and moments x 2): the replay must pick them up
        dev[l][0].mul_(2.0)
        dev[l][2].mul_(2.0)
    g.replay()
    torch.cuda.synchronize()
    f.sync()
    out = results(f)
    f.close()
    # compare with a stream-launched step on the same new inputs
    f1 = fmm_mod.OctoFMM(0.34)
    step(f1)
    ref2 = results(f1)
    f1.close()
    for (L, Lc), (L2, Lc2) in zip(out, ref2):
        assert np.array_equal(L, L2) and np.array_equal(Lc, Lc2)
    assert any(not np.array_equal(a[0], b[0]) for a, b in zip(ref, ref2))

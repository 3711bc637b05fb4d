"""Pins of the oracle's pair kernels.

The paper gives no formulas (P:L444, L465 cite the angular-momentum-conserving
FMM of Marcello 2017); the readings are in DESIGN.md.  Everything here is
pinned against quantities computed independently in the test from point
masses (Newton's law), finite differences and convergence orders.
"""
import numpy as np
import pytest

import oracle

S2 = {(0, 0): 4, (0, 1): 5, (0, 2): 6, (1, 1): 7, (1, 2): 8, (2, 2): 9}
S3 = {(0, 0, 0): 10, (0, 0, 1): 11, (0, 0, 2): 12, (0, 1, 1): 13, (0, 1, 2): 14, (0, 2, 2): 15,
      (1, 1, 1): 16, (1, 1, 2): 17, (1, 2, 2): 18, (2, 2, 2): 19}


def moments_of_points(x, m):
    """Test-side moment definition: M_k = sum m (x - X)^k about the COM."""
    M = np.zeros(20)
    mt = m.sum()
    X = (m[:, None] * x).sum(0) / mt
    y = x - X
    M[0] = mt
    for (a, b), k in S2.items():
        M[k] = np.sum(m * y[:, a] * y[:, b])
    for (a, b, c), k in S3.items():
        M[k] = np.sum(m * y[:, a] * y[:, b] * y[:, c])
    return X, M


def full2(L):
    T = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            T[a, b] = L[S2[tuple(sorted((a, b)))]]
    return T


def full3(L):
    T = np.zeros((3, 3, 3))
    for a in range(3):
        for b in range(3):
            for c in range(3):
                T[a, b, c] = L[S3[tuple(sorted((a, b, c)))]]
    return T


def newton(xt, xs, ms):
    """exact potential (phi = -1/r), gradient of the potential at points xt."""
    R = xt[:, None, :] - xs[None, :, :]
    r = np.linalg.norm(R, axis=-1)
    phi = -np.sum(ms[None, :] / r, axis=1)
    grad = np.sum(ms[None, :, None] * R / r[..., None] ** 3, axis=1)
    return phi, grad


def test_dtensors_closed_form_vs_finite_differences():
    R = np.array([2.3, -1.1, 0.7])
    D0, D1, D2, D3, D4 = oracle.dtensors(R)
    assert D0 == pytest.approx(-1.0 / np.linalg.norm(R), rel=1e-15)
    eps = 1e-5
    for a in range(3):
        e = np.zeros(3)
        e[a] = eps
        p = oracle.dtensors(R + e)
        q = oracle.dtensors(R - e)
        np.testing.assert_allclose((p[0] - q[0]) / (2 * eps), D1[a], rtol=1e-8)
        np.testing.assert_allclose((p[1] - q[1]) / (2 * eps), D2[a], rtol=1e-8)
        np.testing.assert_allclose((p[2] - q[2]) / (2 * eps), D3[a], rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose((p[3] - q[3]) / (2 * eps), D4[a], rtol=1e-7, atol=1e-10)
    # harmonic: traces vanish (laplacian of 1/r = 0 away from 0)
    assert abs(np.trace(D2)) < 1e-15
    assert np.abs(np.einsum("aab->b", D3)).max() < 1e-15
    assert np.abs(np.einsum("aabc->bc", D4)).max() < 1e-15
    # full symmetry
    assert np.allclose(D3, np.transpose(D3, (1, 0, 2))) and np.allclose(D3, np.transpose(D3, (2, 1, 0)))
    assert np.allclose(D4, np.transpose(D4, (1, 0, 2, 3))) and np.allclose(D4, np.transpose(D4, (3, 1, 2, 0)))


def test_p2p_is_newton():
    R = np.array([0.3, -0.4, 1.2])
    t = oracle.p2p_pair(2.5, R)
    r = np.linalg.norm(R)
    np.testing.assert_allclose(t[0], -2.5 / r, rtol=1e-15)
    np.testing.assert_allclose(t[1:4], 2.5 * R / r ** 3, rtol=1e-15)
    # two equal masses: bitwise-opposite L1
    t2 = oracle.p2p_pair(2.5, -R)
    assert np.array_equal(t2[1:4], -t[1:4]) and t2[0] == t[0]


def test_m2l_without_moments_reduces_to_p2p():
    rng = np.random.default_rng(1)
    for _ in range(10):
        R = rng.normal(size=3) * 3
        mB = rng.uniform(0.1, 2)
        MB = np.zeros(20)
        MB[0] = mB
        MA = np.zeros(20)
        MA[0] = 1.0
        t = oracle.m2l_pair(1.0, MA, mB, MB, R, target_refined=False)
        np.testing.assert_allclose(t[:4], oracle.p2p_pair(mB, R), rtol=1e-14)
        assert np.all(t[4:20] == 0) and np.all(np.abs(t[20:]) == 0)


def test_m2l_monopole_gives_exact_taylor_coefficients():
    # point-mass source at its COM: L^(k) = m D^(k)(R) = k-th derivative of -m/|x - X_B|
    R = np.array([1.7, -0.9, 2.2])
    m = 1.3
    MB = np.zeros(20)
    MB[0] = m
    MA = np.zeros(20)
    MA[0] = 1.0
    t = oracle.m2l_pair(1.0, MA, m, MB, R, target_refined=True)
    f = lambda x: -m / np.linalg.norm(x)
    eps = 1e-4
    I = np.eye(3)
    assert t[0] == pytest.approx(f(R), rel=1e-15)
    for a in range(3):
        np.testing.assert_allclose(t[1 + a], (f(R + eps * I[a]) - f(R - eps * I[a])) / (2 * eps), rtol=1e-7)
    L2 = full2(t)
    for a in range(3):
        for b in range(3):
            fd = (f(R + eps * (I[a] + I[b])) - f(R + eps * (I[a] - I[b])) - f(R - eps * (I[a] - I[b]))
                  + f(R - eps * (I[a] + I[b]))) / (4 * eps * eps)
            np.testing.assert_allclose(L2[a, b], fd, rtol=1e-5, atol=1e-9)


def _cluster(rng, k, a):
    x = rng.uniform(-a, a, size=(k, 3))
    m = rng.uniform(0.5, 1.5, size=k)
    return x, m


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_m2l_truncation_orders(seed):
    """Source cluster of size a at distance ~R: the order-3 truncation (n + m <= 3)
    leaves errors L0 ~ a^4, L1 ~ a^3, L2 ~ a^2, L3 ~ a^2.  Halving a must shrink
    them by ~16, 8, 4, 4 -- a dropped or mis-signed term changes the order."""
    rng = np.random.default_rng(seed)
    x0, m0 = _cluster(rng, 9, 1.0)
    XA = np.array([7.0, 3.0, -4.0])
    errs = []
    for a in (0.2, 0.1, 0.05):
        xs = x0 * a
        XB, MB = moments_of_points(xs, m0)
        MA = np.zeros(20)
        MA[0] = 1.0
        t = oracle.m2l_pair(1.0, MA, MB[0], MB, XA - XB, target_refined=True)
        phi, grad = newton(XA[None, :], xs, m0)
        # second and third derivatives of the exact potential by finite differences of the gradient
        eps = 1e-3
        I = np.eye(3)
        H = np.zeros((3, 3))
        T3 = np.zeros((3, 3, 3))
        for b in range(3):
            gp = newton((XA + eps * I[b])[None, :], xs, m0)[1][0]
            gm = newton((XA - eps * I[b])[None, :], xs, m0)[1][0]
            H[:, b] = (gp - gm) / (2 * eps)
            for c in range(3):
                g_pp = newton((XA + eps * I[b] + eps * I[c])[None, :], xs, m0)[1][0]
                g_pm = newton((XA + eps * I[b] - eps * I[c])[None, :], xs, m0)[1][0]
                g_mp = newton((XA - eps * I[b] + eps * I[c])[None, :], xs, m0)[1][0]
                g_mm = newton((XA - eps * I[b] - eps * I[c])[None, :], xs, m0)[1][0]
                T3[:, b, c] = (g_pp - g_pm - g_mp + g_mm) / (4 * eps * eps)
        errs.append([abs(t[0] - phi[0]), np.abs(t[1:4] - grad[0]).max(), np.abs(full2(t) - H).max(),
                     np.abs(full3(t) - T3).max()])
    errs = np.array(errs)
    r01 = errs[0] / errs[1]
    r12 = errs[1] / errs[2]
    for r in (r01, r12):
        assert 12 < r[0] < 20      # a^4
        assert 6 < r[1] < 10       # a^3
        assert 3 < r[2] < 5        # a^2
        assert 3 < r[3] < 5        # a^2


def _cluster_forces(xA, mA, xB, mB, with_lc=True):
    """Per-particle forces on cluster A from cluster B's expansion at A's COM:
    F_i = -m_i (L1 + L2 y + 1/2 L3 yy + Lc), y = x_i - X_A (test-side evaluation)."""
    XA, MA = moments_of_points(xA, mA)
    XB, MB = moments_of_points(xB, mB)
    t = oracle.m2l_pair(MA[0], MA, MB[0], MB, XA - XB, target_refined=True)
    L1 = t[1:4]
    L2 = full2(t)
    L3 = full3(t)
    Lc = t[20:23] if with_lc else np.zeros(3)
    y = xA - XA
    g = L1[None, :] + y @ L2.T + 0.5 * np.einsum("abc,ib,ic->ia", L3, y, y) + Lc[None, :]
    return -mA[:, None] * g


def test_angular_momentum_correction_two_clusters():
    """C5/C7 pin: with Lc the pairwise expansion forces conserve linear AND
    angular momentum to machine precision; without Lc the torque does not
    vanish."""
    rng = np.random.default_rng(7)
    xA, mA = _cluster(rng, 5, 0.6)
    xB, mB = _cluster(rng, 7, 0.6)
    xB = xB + np.array([2.1, 1.3, -1.7])
    for with_lc, tol in ((True, 1e-14), (False, None)):
        FA = _cluster_forces(xA, mA, xB, mB, with_lc)
        FB = _cluster_forces(xB, mB, xA, mA, with_lc)
        F = FA.sum(0) + FB.sum(0)
        T = np.cross(xA, FA).sum(0) + np.cross(xB, FB).sum(0)
        fs = np.abs(FA).sum() + np.abs(FB).sum()
        ts = np.abs(np.cross(xA, FA)).sum() + np.abs(np.cross(xB, FB)).sum()
        assert np.abs(F).max() / fs < 1e-14
        if with_lc:
            assert np.abs(T).max() / ts < tol
        else:
            assert np.abs(T).max() / ts > 1e-6


def test_level_invariants_match_particle_sums():
    """The C7 per-cell force/torque formulas equal the particle sums above."""
    rng = np.random.default_rng(11)
    xA, mA = _cluster(rng, 4, 0.5)
    xB, mB = _cluster(rng, 6, 0.5)
    xB = xB + np.array([-1.9, 2.4, 0.8])
    XA, MA = moments_of_points(xA, mA)
    XB, MB = moments_of_points(xB, mB)
    tA = oracle.m2l_pair(MA[0], MA, MB[0], MB, XA - XB, True)
    tB = oracle.m2l_pair(MB[0], MB, MA[0], MA, XB - XA, True)
    F, T, sf, st = oracle.level_invariants(np.array([MA[0], MB[0]]), np.stack([XA, XB]), np.stack([MA, MB]),
                                           np.stack([tA[:20], tB[:20]]), np.stack([tA[20:], tB[20:]]))
    FA = _cluster_forces(xA, mA, xB, mB)
    FB = _cluster_forces(xB, mB, xA, mA)
    # single-cluster force/torque
    F1, T1, _, _ = oracle.level_invariants(np.array([MA[0]]), XA[None], MA[None], tA[None, :20], tA[None, 20:])
    np.testing.assert_allclose(F1, FA.sum(0), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(T1, np.cross(xA, FA).sum(0), rtol=1e-11, atol=1e-14)
    assert np.abs(F).max() / sf < 1e-14 and np.abs(T).max() / st < 1e-14

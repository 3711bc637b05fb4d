"""Pins of the oracle's C9 per-cell parity scale (oc_dtensors_abs, oc_m2l_abs).

Every GPU per-cell parity gate divides |gpu - oracle| by S, the oracle's
running-error magnitude: the pair formula of C5 evaluated with |.| on every
factor and every term of every D entry, summed over partners (C9;
the north star's "within 1e-12 relative error").  A wrong sign, factor or
dropped term in the abs mode would silently loosen (or tighten) that gate, so
S is pinned here against things that do not come from the oracle itself:

* an independent derivation of the D tensors: the general-n formula for the
  derivatives of 1/r as a sum over index pairings (Hobson),
  d^n(1/r)/dR_i1..dR_in = sum_k (-1)^(n-k) (2n-2k-1)!! / r^(2n-2k+1)
                           * sum over k disjoint index pairs (delta...delta R...R),
  enumerated term by term in the test (no closed forms are retyped), with
  |term| summed for the bound;
* the same D tensors, signed, against the oracle's closed forms (oc_dtensors);
* the M2L bound assembled from those tensors by einsum over FULL symmetric
  tensors (the oracle loops over the 20-coefficient storage via sym2/sym3);
* the triangle inequality S_k >= |t_k| on random and adversarial pairs
  (R on the magic angle where D2_aa cancels to 0, moments of mixed signs);
* S as an error scale: |t_oracle - t_exact| <= 64 eps S_k, with t_exact the
  C5 formula evaluated in extended precision (np.longdouble) from the
  independent tensors.
"""
import itertools

import numpy as np
import pytest

import oracle

S2 = {(0, 0): 4, (0, 1): 5, (0, 2): 6, (1, 1): 7, (1, 2): 8, (2, 2): 9}
S3 = {(0, 0, 0): 10, (0, 0, 1): 11, (0, 0, 2): 12, (0, 1, 1): 13, (0, 1, 2): 14, (0, 2, 2): 15,
      (1, 1, 1): 16, (1, 1, 2): 17, (1, 2, 2): 18, (2, 2, 2): 19}
EPS = np.finfo(np.float64).eps


def matchings(pos):
    """every set of disjoint pairs drawn from the positions `pos` (tuples)."""
    if len(pos) < 2:
        yield ()
        return
    first, rest = pos[0], pos[1:]
    yield from matchings(rest)                      # first stays unpaired
    for i, other in enumerate(rest):                # first paired with `other`
        for m in matchings(rest[:i] + rest[i + 1:]):
            yield ((first, other),) + m


def dfact(k):
    return 1 if k <= 0 else k * dfact(k - 2)


def d_general(n, R, absmode=False, dtype=np.float64):
    """D^(n) = d^n(-1/r) (full 3^n tensor) from the pairing formula; with
    absmode every pairing term enters as |term| (the C9 magnitude bound)."""
    R = np.asarray(R, dtype=dtype)
    r = np.sqrt(np.sum(R * R))
    out = np.zeros((3,) * n, dtype=dtype)
    for idx in itertools.product(range(3), repeat=n):
        tot = dtype(0)
        for m in matchings(tuple(range(n))):
            k = len(m)
            if any(idx[a] != idx[b] for a, b in m):
                continue                            # a delta factor is 0
            paired = {p for ab in m for p in ab}
            prod = dtype(1)
            for p in range(n):
                if p not in paired:
                    prod = prod * R[idx[p]]
            term = dtype((-1) ** (n - k) * dfact(2 * n - 2 * k - 1)) * prod / r ** (2 * n - 2 * k + 1)
            tot = tot + (abs(term) if absmode else term)
        out[idx] = tot if absmode else -tot         # phi = -1/r
    return out


def full2(M, f=lambda x: x):
    T = np.zeros((3, 3), dtype=np.asarray(M).dtype)
    for a, b in itertools.product(range(3), repeat=2):
        T[a, b] = f(M[S2[tuple(sorted((a, b)))]])
    return T


def full3(M, f=lambda x: x):
    T = np.zeros((3, 3, 3), dtype=np.asarray(M).dtype)
    for a, b, c in itertools.product(range(3), repeat=3):
        T[a, b, c] = f(M[S3[tuple(sorted((a, b, c)))]])
    return T


def m2l_einsum(mA, MA, mB, MB, R, refined, absmode, dtype=np.float64):
    """C5 (truncation n + m <= 3, Lc with K = M3B - M3A mB/mA) from full tensors;
    absmode: |.| on every factor, the terms with negative coefficients added."""
    f = (lambda x: abs(x)) if absmode else (lambda x: x)
    MA = np.asarray(MA, dtype=dtype)
    MB = np.asarray(MB, dtype=dtype)
    mA, mB = dtype(mA), f(dtype(mB))
    D = [d_general(n, R, absmode, dtype) for n in range(5)]
    M2, M3, M3A = full2(MB, f), full3(MB, f), full3(MA, f)
    half, sixth = dtype(1) / dtype(2), dtype(1) / dtype(6)
    sg = 1 if absmode else -1
    t = np.zeros(23, dtype=dtype)
    t[0] = mB * D[0] + half * np.einsum("ab,ab", M2, D[2]) + sg * sixth * np.einsum("abc,abc", M3, D[3])
    t[1:4] = mB * D[1] + half * np.einsum("bc,abc->a", M2, D[3])
    if refined:
        for (a, b), k in S2.items():
            t[k] = mB * D[2][a, b]
        for (a, b, c), k in S3.items():
            t[k] = mB * D[3][a, b, c]
    K = M3 + M3A * (mB / mA) if absmode else M3 - M3A * (mB / mA)
    t[20:23] = sg * sixth * np.einsum("bcd,abcd->a", K, D[4])
    return t


def random_pair(rng, scale=1.0, magic=False):
    R = rng.normal(size=3) * scale
    if magic:   # |R_a| equal: D2_aa = 1/r^3 - 3 R_a^2 / r^5 = 0 in exact arithmetic
        R = scale * np.array([1.0, -1.0, 1.0]) * rng.uniform(0.5, 2.0)
    MA = rng.normal(size=20) * 0.1
    MB = rng.normal(size=20) * 0.1
    MA[1:4] = MB[1:4] = 0.0
    return rng.uniform(0.2, 2.0), MA, rng.uniform(0.2, 2.0), MB, R


@pytest.mark.parametrize("absmode", [False, True])
def test_dtensors_match_general_pairing_formula(absmode):
    rng = np.random.default_rng(11)
    for _ in range(20):
        R = rng.normal(size=3) * rng.uniform(0.3, 5.0)
        got = oracle.dtensors_abs(R) if absmode else oracle.dtensors(R)
        for n in range(5):
            want = d_general(n, R, absmode)
            g = np.asarray(got[n]).reshape(want.shape)
            # signed entries can cancel: compare on the scale of their terms
            assert np.all(np.abs(g - want) <= 1e-14 * d_general(n, R, True)), (n, absmode)
    # the bound is never below |D| (same terms, each in |.|)
    D, A = oracle.dtensors(R), oracle.dtensors_abs(R)
    for n in range(5):
        assert np.all(np.asarray(A[n]) >= np.abs(np.asarray(D[n])) * (1 - 1e-15))


@pytest.mark.parametrize("refined", [True, False])
def test_m2l_abs_matches_independent_einsum(refined):
    rng = np.random.default_rng(3 + refined)
    for k in range(25):
        mA, MA, mB, MB, R = random_pair(rng, scale=rng.uniform(1.0, 6.0), magic=(k % 5 == 0))
        S = oracle.m2l_pair_abs(mA, MA, mB, MB, R, refined)
        want = m2l_einsum(mA, MA, mB, MB, R, refined, absmode=True)
        assert np.allclose(S, want, rtol=1e-13, atol=1e-300), np.abs(S - want).max()
        # and the signed formula against the same independent tensors
        t = oracle.m2l_pair(mA, MA, mB, MB, R, refined)
        tw = m2l_einsum(mA, MA, mB, MB, R, refined, absmode=False)
        assert np.all(np.abs(t - tw) <= 1e-13 * S)


def test_scale_bounds_every_term():
    """Triangle inequality on random, magic-angle and sign-adversarial pairs."""
    rng = np.random.default_rng(5)
    for k in range(200):
        mA, MA, mB, MB, R = random_pair(rng, scale=rng.uniform(0.8, 8.0), magic=(k % 4 == 0))
        if k % 3 == 0:   # opposite-sign moments between target and partner (K = M3B - mu M3A grows)
            MA[10:] = -np.sign(MB[10:]) * np.abs(MA[10:])
        for refined in (True, False):
            t = oracle.m2l_pair(mA, MA, mB, MB, R, refined)
            S = oracle.m2l_pair_abs(mA, MA, mB, MB, R, refined)
            assert np.all(S >= np.abs(t) * (1 - 1e-14)), k
            if not refined:
                assert np.all(S[4:20] == 0.0)


def test_scale_bounds_the_rounding_error():
    """|oracle (binary64) - C5 in extended precision| <= 64 eps S per component;
    on the magic angle |t_2aa| ~ eps S while S stays O(m/r^3), which is the
    cancellation that rules out Sum|term| as the scale (C9)."""
    if np.finfo(np.longdouble).eps >= EPS:
        pytest.skip("no extended-precision long double on this platform")
    rng = np.random.default_rng(9)
    worst = 0.0
    for k in range(30):
        mA, MA, mB, MB, R = random_pair(rng, scale=rng.uniform(1.0, 6.0), magic=(k % 3 == 0))
        for refined in (True, False):
            t = oracle.m2l_pair(mA, MA, mB, MB, R, refined)
            S = oracle.m2l_pair_abs(mA, MA, mB, MB, R, refined)
            ex = m2l_einsum(mA, MA, mB, MB, R, refined, absmode=False, dtype=np.longdouble)
            err = np.abs(t.astype(np.longdouble) - ex)
            nz = S > 0
            worst = max(worst, float(np.max(err[nz] / S[nz])))
            assert np.all(err[~nz] == 0)
    assert worst <= 64 * EPS, worst
    # magic angle, monopole partner: D2_xx cancels, the scale does not
    R = np.array([1.5, 1.5, -1.5])
    MB = np.zeros(20)
    t = oracle.m2l_pair(1.0, np.zeros(20), 2.0, MB, R, True)
    S = oracle.m2l_pair_abs(1.0, np.zeros(20), 2.0, MB, R, True)
    r = np.sqrt(3) * 1.5
    assert abs(t[4]) <= 4 * EPS * S[4]
    assert S[4] == pytest.approx(2.0 * 2.0 / r ** 3, rel=1e-14)   # m (1/r^3 + 3 R_x^2 / r^5) = 2 m / r^3


def test_level_scale_bounds_level_sums():
    """The per-cell scale the GPU gate uses (oracle.same_level's third output,
    sums of the per-pair S) bounds |L| and |Lc| of every cell of a level."""
    import synth
    tr = synth.config_random_amr(2, 2, 0.5)
    mom = oracle.moments(tr)
    for level in range(1, len(tr.levels)):
        L, Lc, S = oracle.same_level(tr, mom, level, 0.5)
        t = np.concatenate([L, Lc], 1)
        assert np.all(S >= np.abs(t) * (1 - 1e-13))
        assert np.all(S[np.any(t != 0, axis=1)].max(axis=1) > 0)

"""ctypes wrapper of oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


def _load():
    build()
    L = C.CDLL(_SO)
    L.oc_R2.restype = C.c_double
    L.oc_R2.argtypes = [C.c_double]
    L.oc_pair_class.restype = C.c_int
    L.oc_pair_class.argtypes = [C.c_double, C.c_int, _i64p, _i64p]
    L.oc_stencil.restype = C.c_int
    L.oc_stencil.argtypes = [C.c_double, C.c_int, C.c_int, _i32p, _i32p, C.c_int]
    L.oc_dtensors.restype = None
    L.oc_dtensors.argtypes = [_f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
    L.oc_p2p.restype = None
    L.oc_p2p.argtypes = [C.c_double, _f64p, _f64p]
    L.oc_m2l.restype = None
    L.oc_m2l.argtypes = [C.c_double, _f64p, C.c_double, _f64p, _f64p, C.c_int, _f64p]
    L.oc_m2l_abs.restype = None
    L.oc_m2l_abs.argtypes = [C.c_double, _f64p, C.c_double, _f64p, _f64p, C.c_int, _f64p]
    L.oc_dtensors_abs.restype = None
    L.oc_dtensors_abs.argtypes = [_f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
    L.oc_p2m.restype = None
    L.oc_p2m.argtypes = [C.c_int64, _f64p, C.c_double, _f64p]
    L.oc_m2m.restype = C.c_int
    L.oc_m2m.argtypes = [C.c_int64, _i32p, _u8p, _i64p, C.c_int64, _i32p, _u8p, _i64p, _f64p, _f64p, _f64p,
                         C.c_double, _f64p, _f64p, _f64p, _f64p]
    L.oc_same_level.restype = C.c_int
    L.oc_same_level.argtypes = [C.c_int, C.c_double, C.c_double, _f64p, C.c_int64, _i32p, _u8p, _i64p,
                                _f64p, _f64p, _f64p, C.c_int64, _i64p, _i32p, C.c_int, _f64p, _f64p, _f64p]
    L.oc_count_interactions.restype = C.c_int
    L.oc_count_interactions.argtypes = [C.c_int, C.c_double, C.c_int64, _i32p, _u8p, C.c_int64, _i64p, _i32p,
                                        _i64p]
    L.oc_l2l.restype = C.c_int
    L.oc_l2l.argtypes = [C.c_int64, _i32p, _i64p, _f64p, _f64p, _f64p, C.c_int64, _i32p, _u8p, _i64p, _f64p,
                         C.c_double, _f64p, _f64p, _f64p]
    L.oc_direct.restype = None
    L.oc_direct.argtypes = [C.c_int64, _f64p, _f64p, C.c_double, _f64p, _f64p]
    L.oc_level_invariants.restype = None
    L.oc_level_invariants.argtypes = [C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
    L.oc_coverage.restype = None
    L.oc_coverage.argtypes = [C.c_double, C.c_int64, _i32p, _i64p, _i64p]
    return L


lib = _load()


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# --------------------------------------------------------------------------
# C1 stencil
# --------------------------------------------------------------------------
def R2(theta: float) -> float:
    return lib.oc_R2(float(theta))


def pair_class(theta: float, i, j, is_root: bool = False) -> int:
    return lib.oc_pair_class(R2(theta), int(is_root), _c(i, np.int64), _c(j, np.int64))


def stencil(theta: float, is_root: bool = False, box: int = 9):
    """list over parity c = cx + 2cy + 4cz of (k, 4) int arrays [dx, dy, dz, cls]."""
    cap = (2 * box + 1) ** 3
    out = np.zeros(8 * cap * 4, dtype=np.int32)
    cnt = np.zeros(8, dtype=np.int32)
    if lib.oc_stencil(float(theta), int(is_root), int(box), out, cnt, cap) != 0:
        raise RuntimeError("stencil capacity")
    out = out.reshape(8, cap, 4)
    return [out[c, :cnt[c]].copy() for c in range(8)]


def stencil_sets(theta: float, is_root: bool = False):
    """(far_union, near_union, per-parity far sets, per-parity near sets) as python sets."""
    st = stencil(theta, is_root)
    far_c = [set(map(tuple, s[s[:, 3] == 1, :3].tolist())) for s in st]
    near_c = [set(map(tuple, s[s[:, 3] == 2, :3].tolist())) for s in st]
    return set().union(*far_c), set().union(*near_c), far_c, near_c


# --------------------------------------------------------------------------
# pair kernels (C4, C5) and D tensors
# --------------------------------------------------------------------------
def dtensors(R):
    D0 = np.zeros(1)
    D1, D2, D3, D4 = np.zeros(3), np.zeros(9), np.zeros(27), np.zeros(81)
    lib.oc_dtensors(_c(R, np.float64), D0, D1, D2, D3, D4)
    return D0[0], D1, D2.reshape(3, 3), D3.reshape(3, 3, 3), D4.reshape(3, 3, 3, 3)


def dtensors_abs(R):
    """C9 magnitude bounds of the D tensors (every term of every entry in |.|)."""
    D0 = np.zeros(1)
    D1, D2, D3, D4 = np.zeros(3), np.zeros(9), np.zeros(27), np.zeros(81)
    lib.oc_dtensors_abs(_c(R, np.float64), D0, D1, D2, D3, D4)
    return D0[0], D1, D2.reshape(3, 3), D3.reshape(3, 3, 3), D4.reshape(3, 3, 3, 3)


def p2p_pair(mB: float, R) -> np.ndarray:
    t = np.zeros(4)
    lib.oc_p2p(float(mB), _c(R, np.float64), t)
    return t


def m2l_pair(mA: float, MA, mB: float, MB, R, target_refined: bool = True) -> np.ndarray:
    t = np.zeros(23)
    lib.oc_m2l(float(mA), _c(MA, np.float64), float(mB), _c(MB, np.float64), _c(R, np.float64),
               int(target_refined), t)
    return t


def m2l_pair_abs(mA: float, MA, mB: float, MB, R, target_refined: bool = True) -> np.ndarray:
    """C9 per-pair parity scale: the M2L formula with |.| on every factor (23 values)."""
    t = np.zeros(23)
    lib.oc_m2l_abs(float(mA), _c(MA, np.float64), float(mB), _c(MB, np.float64), _c(R, np.float64),
                   int(target_refined), t)
    return t


# --------------------------------------------------------------------------
# C3 moments (P2M + M2M, bottom-up)
# --------------------------------------------------------------------------
def moments(tree):
    """per level dict(m=(n,512), X=(nr,512,3), M=(nr,512,20), rslot=(n,))."""
    out = [None] * len(tree.levels)
    for lv in reversed(tree.levels):
        n = lv.n_nodes
        rs = lv.rslot()
        nr = lv.n_refined
        m = np.zeros((n, 512))
        rho = _c(lv.rho, np.float64)
        mm = np.zeros(n * 512)
        lib.oc_p2m(n * 512, rho.reshape(-1), float(lv.h), mm)
        m[:] = mm.reshape(n, 512)
        m[lv.refined.astype(bool)] = 0.0
        X = np.zeros((nr, 512, 3))
        M = np.zeros((nr, 512, 20))
        if nr:
            ch = tree.levels[lv.level + 1]
            cm = out[lv.level + 1]
            rc = lib.oc_m2m(n, _c(lv.ijk, np.int32), _c(lv.refined, np.uint8), _c(rs, np.int64),
                            ch.n_nodes, _c(ch.ijk, np.int32), _c(ch.refined, np.uint8), _c(cm["rslot"], np.int64),
                            _c(cm["m"], np.float64).reshape(-1), _c(cm["X"], np.float64).reshape(-1),
                            _c(cm["M"], np.float64).reshape(-1), float(ch.h), _c(tree.origin, np.float64),
                            m.reshape(-1), X.reshape(-1), M.reshape(-1))
            if rc != 0:
                raise RuntimeError("oc_m2m: missing child node")
        out[lv.level] = dict(m=m, X=X, M=M, rslot=rs)
    return out


def level_cell_arrays(tree, mom, level: int):
    """Per-cell (m, X, M[20]) of every cell of a level, node-major (n*512 rows):
    refined cells from the moments, leaf cells as point masses at centres."""
    lv = tree.levels[level]
    mo = mom[level]
    n = lv.n_nodes
    m = mo["m"].reshape(-1).copy()
    X = lv.cell_centres(tree.origin).reshape(n, 512, 3).copy()
    M = np.zeros((n, 512, 20))
    M[:, :, 0] = mo["m"]
    r = np.nonzero(lv.refined)[0]
    if r.size:
        X[r] = mo["X"][mo["rslot"][r]]
        M[r] = mo["M"][mo["rslot"][r]]
    return m, X.reshape(-1, 3), M.reshape(-1, 20)


# --------------------------------------------------------------------------
# C4-C6 same-level interactions
# --------------------------------------------------------------------------
def _targets(lv, targets):
    if targets is None:
        tn = np.repeat(np.arange(lv.n_nodes, dtype=np.int64), 512)
        tc = np.tile(np.arange(512, dtype=np.int32), lv.n_nodes)
    else:
        tn, tc = _c(targets[0], np.int64), _c(targets[1], np.int32)
    return tn, tc


def same_level(tree, mom, level: int, theta: float, targets=None, prune: bool = True):
    """(L (t,20), Lc (t,3), absL (t,23)) for target cells (all cells of the level,
    node-major, by default).  Level 0 uses the root rule (C2)."""
    lv = tree.levels[level]
    mo = mom[level]
    tn, tc = _targets(lv, targets)
    t = tn.shape[0]
    L = np.zeros(t * 20)
    Lc = np.zeros(t * 3)
    ab = np.zeros(t * 23)
    X = _c(mo["X"], np.float64).reshape(-1)
    M = _c(mo["M"], np.float64).reshape(-1)
    if X.size == 0:
        X = np.zeros(1)
        M = np.zeros(1)
    rc = lib.oc_same_level(int(level == 0), float(theta), float(lv.h), _c(tree.origin, np.float64), lv.n_nodes,
                           _c(lv.ijk, np.int32), _c(lv.refined, np.uint8), _c(mo["rslot"], np.int64),
                           _c(mo["m"], np.float64).reshape(-1), X, M, t, tn, tc, int(prune), L, Lc, ab)
    if rc != 0:
        raise RuntimeError("oc_same_level: bad target")
    return L.reshape(t, 20), Lc.reshape(t, 3), ab.reshape(t, 23)


def count_interactions(tree, level: int, theta: float, targets=None) -> np.ndarray:
    """(t, 3) counts {P2P, M2L (refined target), mixed (leaf target <- refined)}."""
    lv = tree.levels[level]
    tn, tc = _targets(lv, targets)
    out = np.zeros(tn.shape[0] * 3, dtype=np.int64)
    lib.oc_count_interactions(int(level == 0), float(theta), lv.n_nodes, _c(lv.ijk, np.int32),
                              _c(lv.refined, np.uint8), tn.shape[0], tn, tc, out)
    return out.reshape(-1, 3)


# --------------------------------------------------------------------------
# C7 invariants, C8 full solve, N^2, coverage
# --------------------------------------------------------------------------
def level_invariants(m, X, M, L, Lc):
    """(sum F (3), sum tau (3), sum|F|, sum|tau|) over the given cells."""
    n = int(np.asarray(m).shape[0])
    F, T, sc = np.zeros(3), np.zeros(3), np.zeros(2)
    lib.oc_level_invariants(n, _c(m, np.float64), _c(X, np.float64).reshape(-1), _c(M, np.float64).reshape(-1),
                            _c(L, np.float64).reshape(-1), _c(Lc, np.float64).reshape(-1), F, T, sc)
    return F, T, sc[0], sc[1]


def direct(x, m, G: float = 1.0):
    x = _c(x, np.float64)
    n = x.shape[0]
    phi = np.zeros(n)
    g = np.zeros(n * 3)
    lib.oc_direct(n, x.reshape(-1), _c(m, np.float64), float(G), phi, g)
    return phi, g.reshape(n, 3)


def fmm_full(tree, theta: float, G: float = 1.0, mom=None):
    """Whole 3-step FMM (C8): moments, same-level at every level (root rule at
    level 0), L2L top-down, extraction Phi = G L0, g = -G (L1 + Lc) at leaf
    cells, ordered as synth.leaf_cells(tree)."""
    if mom is None:
        mom = moments(tree)
    tot = []
    for lv in tree.levels:
        L, Lc, _ = same_level(tree, mom, lv.level, theta)
        tot.append([L.reshape(lv.n_nodes, 512, 20).copy(), Lc.reshape(lv.n_nodes, 512, 3).copy()])
    for lv in tree.levels[:-1]:
        ch = tree.levels[lv.level + 1]
        mo, mc = mom[lv.level], mom[lv.level + 1]
        Xp = _c(mo["X"], np.float64).reshape(-1)
        Xc = _c(mc["X"], np.float64).reshape(-1)
        if Xc.size == 0:
            Xc = np.zeros(1)
        Lch = tot[lv.level + 1][0].reshape(-1)
        Lcch = tot[lv.level + 1][1].reshape(-1)
        rc = lib.oc_l2l(lv.n_nodes, _c(lv.ijk, np.int32), _c(mo["rslot"], np.int64), Xp,
                        _c(tot[lv.level][0], np.float64).reshape(-1), _c(tot[lv.level][1], np.float64).reshape(-1),
                        ch.n_nodes, _c(ch.ijk, np.int32), _c(ch.refined, np.uint8), _c(mc["rslot"], np.int64), Xc,
                        float(ch.h), _c(tree.origin, np.float64), Lch, Lcch)
        if rc != 0:
            raise RuntimeError("oc_l2l: missing parent")
        tot[lv.level + 1][0] = Lch.reshape(ch.n_nodes, 512, 20)
        tot[lv.level + 1][1] = Lcch.reshape(ch.n_nodes, 512, 3)
    phi, g = [], []
    for lv in tree.levels:
        leaf = np.nonzero(lv.refined == 0)[0]
        if leaf.size == 0:
            continue
        L = tot[lv.level][0][leaf].reshape(-1, 20)
        Lc = tot[lv.level][1][leaf].reshape(-1, 3)
        phi.append(G * L[:, 0])
        g.append(-G * (L[:, 1:4] + Lc))
    return np.concatenate(phi), np.concatenate(g), mom, tot


def coverage(theta: float, lev, g) -> np.ndarray:
    hist = np.zeros(4, dtype=np.int64)
    lib.oc_coverage(float(theta), int(len(lev)), _c(lev, np.int32), _c(g, np.int64).reshape(-1), hist)
    return hist

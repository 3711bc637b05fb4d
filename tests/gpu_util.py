"""Test-side marshalling between the oracle's per-level arrays and the C ABI
layout, plus the parity metrics.  Test infrastructure."""
import numpy as np


def api_inputs(tree, mom, level):
    """(mono [n][512], com [3][nr][512], mom [20][nr][512]) in the ABI layout,
    from the oracle's moments (oracle.moments)."""
    mo = mom[level]
    mono = np.ascontiguousarray(mo["m"], np.float64)
    com = np.ascontiguousarray(np.transpose(mo["X"], (2, 0, 1)), np.float64)
    mm = np.ascontiguousarray(np.transpose(mo["M"], (2, 0, 1)), np.float64)
    return mono, com, mm


def load(fmm, tree, mom, level, owner=None, device=False):
    lv = tree.levels[level]
    mono, com, mm = api_inputs(tree, mom, level)
    if device:
        import torch
        mono, com, mm = (torch.from_numpy(a).cuda() for a in (mono, com, mm))
    fmm.load_level(level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, owner, mono, com, mm)
    return mono, com, mm


def get(fmm, tree, level, n_owned=None):
    n = tree.levels[level].n_nodes if n_owned is None else n_owned
    L = np.zeros((20, n, 512))
    Lc = np.zeros((3, n, 512))
    fmm.get_expansions(level, L, Lc)
    return L, Lc


def oracle_layout(L, Lc, n):
    """oracle (n*512, 20)/(n*512, 3) -> ABI (20, n, 512)/(3, n, 512)."""
    return (np.ascontiguousarray(L.reshape(n, 512, 20).transpose(2, 0, 1)),
            np.ascontiguousarray(Lc.reshape(n, 512, 3).transpose(2, 0, 1)))


def parity(gpu_L, gpu_Lc, or_L, or_Lc, or_abs, tol=1e-12):
    """Normwise (per component, relative to the component's max |oracle|) and
    per-cell (relative to the oracle's sum of |term|) errors; returns the two
    maxima.  gpu_*: ABI layout restricted to the compared cells, flattened to
    (cells, k); or_*: oracle rows of the same cells."""
    g = np.concatenate([gpu_L, gpu_Lc], axis=1)
    o = np.concatenate([or_L, or_Lc], axis=1)
    d = np.abs(g - o)
    scale = np.abs(o).max(axis=0)
    norm = np.where(scale > 0, d.max(axis=0) / np.where(scale > 0, scale, 1), d.max(axis=0))
    cell = np.where(or_abs > 0, d / np.where(or_abs > 0, or_abs, 1), d)
    return float(norm.max()), float(cell.max())


def parity_detail(gpu_L, gpu_Lc, or_L, or_Lc, or_abs):
    """per-component (normwise, per-cell) maxima, for failure messages."""
    g = np.concatenate([gpu_L, gpu_Lc], axis=1)
    o = np.concatenate([or_L, or_Lc], axis=1)
    d = np.abs(g - o)
    scale = np.abs(o).max(axis=0)
    norm = d.max(axis=0) / np.where(scale > 0, scale, 1)
    cell = (np.where(or_abs > 0, d / np.where(or_abs > 0, or_abs, 1), d)).max(axis=0)
    return {k: (float(norm[k]), float(cell[k])) for k in range(23) if norm[k] > 1e-14 or cell[k] > 1e-14}


def flat_abi(L, Lc, nodes, cells):
    """rows (len, 23) of the ABI arrays at (node, cell) pairs."""
    return L[:, nodes, cells].T, Lc[:, nodes, cells].T

"""Seeded synthetic octrees of 8^3-cell sub-grids and their density fields.

Structure only (no FMM arithmetic): P:L418-421 describes the data structure
(adaptive octree, each node an N^3 = 8^3 sub-grid, nodes distributed along a
space-filling curve).  Refinement is 2:1 graded (SPEC S:L101 reading, SURVEY
8(c) C6): a refined node's 26 same-level neighbours exist whenever they lie
inside the domain.

Conventions:
  * node (I,J,K) at level l covers global cells [8I, 8I+8) x ... ; the level-l
    cell width is h_l = width / (8 * 2**l); cell centre origin + (g + 1/2) h_l.
  * local cell index lx + 8 ly + 64 lz.
  * nodes of a level are sorted in Morton order (x -> bit 0, y -> bit 1,
    z -> bit 2).
  * neighbour slot (dx+1) + 3 (dy+1) + 9 (dz+1); slot 13 is the node itself;
    -1 = absent (outside the domain or not present at this level).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NB_OFFSETS = np.array([(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)],
                      dtype=np.int64)

_LOC = np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1)
# local index lx + 8 ly + 64 lz  ->  (lx, ly, lz)
LOCAL_XYZ = np.zeros((512, 3), dtype=np.int64)
for _z in range(8):
    for _y in range(8):
        for _x in range(8):
            LOCAL_XYZ[_x + 8 * _y + 64 * _z] = (_x, _y, _z)


def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton_keys(ijk: np.ndarray) -> np.ndarray:
    """Morton key with x -> bit 0, y -> bit 1, z -> bit 2."""
    ijk = np.asarray(ijk, dtype=np.int64)
    return _spread3(ijk[:, 0]) | (_spread3(ijk[:, 1]) << np.uint64(1)) | (_spread3(ijk[:, 2]) << np.uint64(2))


def _pack(ijk: np.ndarray) -> np.ndarray:
    ijk = np.asarray(ijk, dtype=np.int64)
    return ijk[:, 0] | (ijk[:, 1] << 21) | (ijk[:, 2] << 42)


def _unpack(keys: np.ndarray) -> np.ndarray:
    keys = np.asarray(keys, dtype=np.int64)
    return np.stack([keys & 0x1FFFFF, (keys >> 21) & 0x1FFFFF, (keys >> 42) & 0x1FFFFF], axis=1)


@dataclass
class Level:
    level: int
    h: float
    ijk: np.ndarray          # (n, 3) int32, Morton order
    refined: np.ndarray      # (n,) uint8
    neighbors: np.ndarray    # (n, 27) int32, -1 absent
    rho: np.ndarray | None   # (n, 512) float64 densities of leaf nodes' cells (0 for refined rows); None: structure only

    @property
    def n_nodes(self) -> int:
        return int(self.ijk.shape[0])

    @property
    def n_refined(self) -> int:
        return int(self.refined.sum())

    def rslot(self) -> np.ndarray:
        """refined-slot index of each node (k-th refined node in node order), -1 for leaves."""
        r = self.refined.astype(bool)
        s = np.full(self.n_nodes, -1, dtype=np.int64)
        s[r] = np.arange(int(r.sum()), dtype=np.int64)
        return s

    def cell_centres(self, origin: np.ndarray, nodes: np.ndarray | None = None) -> np.ndarray:
        """(len(nodes), 512, 3) geometric cell centres."""
        ijk = self.ijk if nodes is None else self.ijk[nodes]
        g = 8 * ijk.astype(np.int64)[:, None, :] + LOCAL_XYZ[None, :, :]
        return origin[None, None, :] + (g + 0.5) * self.h


@dataclass
class Tree:
    origin: np.ndarray
    width: float
    levels: list = field(default_factory=list)

    @property
    def max_level(self) -> int:
        return len(self.levels) - 1

    def summary(self) -> dict:
        return {
            "levels": [(lv.level, lv.n_nodes, lv.n_refined) for lv in self.levels],
            "subgrids": int(sum(lv.n_nodes for lv in self.levels)),
            "refined": int(sum(lv.n_refined for lv in self.levels)),
        }


def neighbor_table(ijk: np.ndarray, level: int) -> np.ndarray:
    keys = _pack(ijk)
    order = np.argsort(keys)
    sk = keys[order]
    n = ijk.shape[0]
    out = np.full((n, 27), -1, dtype=np.int32)
    lim = 1 << level
    for s, off in enumerate(NB_OFFSETS):
        q = ijk.astype(np.int64) + off[None, :]
        inside = np.all((q >= 0) & (q < lim), axis=1)
        qk = _pack(np.where(inside[:, None], q, 0))
        pos = np.searchsorted(sk, qk)
        pos = np.minimum(pos, n - 1)
        hit = inside & (sk[pos] == qk)
        out[hit, s] = order[pos[hit]].astype(np.int32)
    return out


def build_tree(origin, width: float, max_level: int, refine_fn, density_fn, grade: bool = True) -> Tree:
    """Top-down refinement by refine_fn(level, lo, hi) -> bool per node, 2:1 grading,
    then densities at leaf-cell centres by density_fn(centres (n,3)) -> (n,)
    (density_fn None: structure only, Level.rho = None)."""
    origin = np.asarray(origin, dtype=np.float64)
    # 1. top-down refinement sets (packed keys)
    nodes = [np.zeros(1, dtype=np.int64)]
    refined = []
    for lvl in range(max_level + 1):
        ijk = _unpack(nodes[lvl])
        if lvl == max_level or ijk.shape[0] == 0:
            ref = np.zeros(ijk.shape[0], dtype=bool)
        else:
            hn = width / (1 << lvl)
            lo = origin[None, :] + ijk * hn
            ref = np.asarray(refine_fn(lvl, lo, lo + hn), dtype=bool)
        refined.append(np.unique(nodes[lvl][ref]))
        if lvl < max_level:
            par = _unpack(refined[lvl])
            ch = (2 * par[:, None, :] + NB_OFFSETS[None, [13, 14, 16, 17, 22, 23, 25, 26], :]).reshape(-1, 3)
            nodes.append(np.unique(_pack(ch)))
    # 2. 2:1 grading, finest -> coarsest: a refined node's in-domain 27-neighbourhood
    #    must exist at its level, i.e. the neighbours' parents must be refined.
    if grade:
        for lvl in range(max_level, 0, -1):
            if refined[lvl].size == 0:
                continue
            ijk = _unpack(refined[lvl])
            nb = (ijk[:, None, :] + NB_OFFSETS[None, :, :]).reshape(-1, 3)
            lim = 1 << lvl
            nb = nb[np.all((nb >= 0) & (nb < lim), axis=1)]
            need = np.unique(_pack(nb // 2))
            refined[lvl - 1] = np.union1d(refined[lvl - 1], need)
        # rebuild node sets top-down
        nodes = [np.zeros(1, dtype=np.int64)]
        for lvl in range(max_level):
            refined[lvl] = np.intersect1d(refined[lvl], nodes[lvl])
            par = _unpack(refined[lvl])
            ch = (2 * par[:, None, :] + NB_OFFSETS[None, [13, 14, 16, 17, 22, 23, 25, 26], :]).reshape(-1, 3)
            nodes.append(np.unique(_pack(ch)))
        refined[max_level] = np.zeros(0, dtype=np.int64)
    # 3. per-level arrays in Morton order
    tree = Tree(origin=origin, width=float(width))
    for lvl in range(max_level + 1):
        if nodes[lvl].size == 0:
            break
        ijk = _unpack(nodes[lvl])
        order = np.argsort(morton_keys(ijk), kind="stable")
        ijk = ijk[order]
        ref = np.isin(_pack(ijk), refined[lvl])
        h = width / (8 * (1 << lvl))
        rho = None if density_fn is None else np.zeros((ijk.shape[0], 512), dtype=np.float64)
        leaf = np.nonzero(~ref)[0]
        if leaf.size and density_fn is not None:
            g = 8 * ijk[leaf][:, None, :] + LOCAL_XYZ[None, :, :]
            cen = origin[None, None, :] + (g + 0.5) * h
            rho[leaf] = np.asarray(density_fn(cen.reshape(-1, 3)), dtype=np.float64).reshape(leaf.size, 512)
        tree.levels.append(Level(level=lvl, h=h, ijk=ijk.astype(np.int32), refined=ref.astype(np.uint8),
                                 neighbors=neighbor_table(ijk, lvl), rho=rho))
    return tree


def leaf_cells(tree: Tree):
    """All finest cells (cells of leaf nodes at any level): level, global coords,
    centres, densities, cell volume h^3 of each."""
    lev, g, cen, rho, vol = [], [], [], [], []
    for lv in tree.levels:
        leaf = np.nonzero(lv.refined == 0)[0]
        if leaf.size == 0:
            continue
        gg = (8 * lv.ijk[leaf].astype(np.int64)[:, None, :] + LOCAL_XYZ[None, :, :]).reshape(-1, 3)
        lev.append(np.full(gg.shape[0], lv.level, dtype=np.int32))
        g.append(gg)
        cen.append(tree.origin[None, :] + (gg + 0.5) * lv.h)
        rho.append(lv.rho[leaf].reshape(-1))
        vol.append(np.full(gg.shape[0], lv.h ** 3))
    return (np.concatenate(lev), np.concatenate(g), np.concatenate(cen), np.concatenate(rho),
            np.concatenate(vol))


# --------------------------------------------------------------------------
# configurations (BASELINE.json "configs", recipes in DESIGN.md "Inputs")
# --------------------------------------------------------------------------
def _box_sphere(lo, hi, c, r):
    q = np.clip(c[None, :], lo, hi)
    return np.sum((q - c[None, :]) ** 2, axis=1) <= r * r


def config_c1(seed: int = 0) -> Tree:
    """configs[0]: single octree level of 2x2x2 sub-grids (root refined, level 1
    leaves), i.i.d. rho ~ U(0.1, 1.0), domain [0,1]^3."""
    rng = np.random.default_rng(seed)
    return build_tree(np.zeros(3), 1.0, 1, lambda l, lo, hi: np.ones(lo.shape[0], bool),
                      lambda x: rng.uniform(0.1, 1.0, size=x.shape[0]))


def config_c2() -> Tree:
    """configs[1]: uniform level-3 grid (512 leaf sub-grids), single Gaussian star
    rho = exp(-|x-c|^2 / (2 sigma^2)) + 1e-10, sigma = 0.1, c = 0.5 + (h3/3)(1,2,3)."""
    h3 = 1.0 / 64.0
    c = np.array([0.5, 0.5, 0.5]) + (h3 / 3.0) * np.array([1.0, 2.0, 3.0])
    sig = 0.1
    return build_tree(np.zeros(3), 1.0, 3, lambda l, lo, hi: np.ones(lo.shape[0], bool),
                      lambda x: np.exp(-np.sum((x - c) ** 2, axis=1) / (2 * sig * sig)) + 1e-10)


def config_c3(max_level: int = 3) -> Tree:
    """configs[2]: rotating (oblate) n = 1 polytrope, rho = sin(pi xi)/(pi xi) for
    xi < 1, floor 1e-10; xi^2 = ((x-cx)^2 + (y-cy)^2)/a^2 + (z-cz)^2/c^2, a = 0.3,
    c = 0.7 a, centre (0.5 + h3/3, 0.5, 0.5); refine a node iff it intersects
    xi < 1.2; 2:1 graded."""
    h3 = 1.0 / 64.0
    cen = np.array([0.5 + h3 / 3.0, 0.5, 0.5])
    a, cz = 0.3, 0.21

    def refine(l, lo, hi):
        q = np.clip(cen[None, :], lo, hi) - cen[None, :]
        xi2 = (q[:, 0] ** 2 + q[:, 1] ** 2) / a ** 2 + q[:, 2] ** 2 / cz ** 2
        return xi2 < 1.2 ** 2

    def dens(x):
        q = x - cen[None, :]
        xi = np.sqrt((q[:, 0] ** 2 + q[:, 1] ** 2) / a ** 2 + q[:, 2] ** 2 / cz ** 2)
        s = np.where(xi < 1.0, np.sinc(xi), 0.0)  # np.sinc(x) = sin(pi x)/(pi x)
        return np.maximum(s, 1e-10)

    return build_tree(np.zeros(3), 1.0, max_level, refine, dens)


def _lane_emden(n: float, dxi: float = 1e-4):
    """Tabulated Lane-Emden solution theta_n(xi) up to the first zero (RK4)."""
    xi = dxi
    th = 1.0 - xi * xi / 6.0
    dth = -xi / 3.0
    xs, ts = [0.0, xi], [1.0, th]

    def f(x, y, dy):
        return dy, -np.power(max(y, 0.0), n) - 2.0 * dy / x

    while th > 0.0:
        k1 = f(xi, th, dth)
        k2 = f(xi + dxi / 2, th + dxi / 2 * k1[0], dth + dxi / 2 * k1[1])
        k3 = f(xi + dxi / 2, th + dxi / 2 * k2[0], dth + dxi / 2 * k2[1])
        k4 = f(xi + dxi, th + dxi * k3[0], dth + dxi * k3[1])
        th += dxi / 6 * (k1[0] + 2 * k2[0] + 2 * k3[0] + k4[0])
        dth += dxi / 6 * (k1[1] + 2 * k2[1] + 2 * k3[1] + k4[1])
        xi += dxi
        xs.append(xi)
        ts.append(th)
    xs, ts = np.array(xs), np.maximum(np.array(ts), 0.0)
    return xs, ts, -dth  # xi grid, theta, |theta'(xi1)|


class V1309:
    """V1309 Sco contact-binary initial-model SHAPE, the model of
    configs[3]/[4].  Code units G = Msun = Rsun = 1; cubic domain edge 1020
    centred on the COM; n = 1.5 polytropes of 1.54 and 0.17 Msun
     at COM separation 6.37 with radii 3.63 / 1.35
    (Roche-lobe reading); refinement mirrors P:L744-746 shifted to max_level:
    stars to L-2, accretor core (0.3 R) to L-1, donor core (0.3 R) to L;
    optionally every node within env_radius of the COM to L (configs[4]
    common-envelope reading); envelope floor 1e-10 rho_c."""
    origin = np.full(3, -510.0)
    width = 1020.0

    def __init__(self, max_level: int = 13, env_radius: float = 0.0):
        self.L = max_level
        self.env_radius = float(env_radius)
        m1, m2, sep = 1.54, 0.17, 6.37
        x1, x2 = -sep * m2 / (m1 + m2), sep * m1 / (m1 + m2)
        self.R1, self.R2 = 3.63, 1.35
        self.c1, self.c2 = np.array([x1, 0.0, 0.0]), np.array([x2, 0.0, 0.0])
        self.xs, self.ts, dth1 = _lane_emden(1.5)
        xi1 = self.xs[-1]
        self.xi1 = xi1

        def rho_c(M, R):
            alpha = R / xi1
            return M / (4.0 * np.pi * alpha ** 3 * xi1 ** 2 * dth1)

        self.rc1, self.rc2 = rho_c(m1, self.R1), rho_c(m2, self.R2)
        self.stars = ((self.c1, self.R1, self.rc1), (self.c2, self.R2, self.rc2))
        self.floor = 1e-10 * self.rc1

    def density(self, x):
        out = np.full(x.shape[0], self.floor)
        for c, R, rc in self.stars:
            r = np.sqrt(np.sum((x - c[None, :]) ** 2, axis=1))
            xi = r / R * self.xi1
            th = np.interp(xi, self.xs, self.ts, right=0.0)
            out = out + rc * th ** 1.5
        return out

    def density_torch(self, x):
        """The same density on a torch tensor x (..., 3) (any device): input
        generation for shards too large to synthesise on the host."""
        import torch
        xs = torch.as_tensor(self.xs, dtype=torch.float64, device=x.device)
        ts = torch.as_tensor(self.ts, dtype=torch.float64, device=x.device)
        out = torch.full(x.shape[:-1], self.floor, dtype=torch.float64, device=x.device)
        for c, R, rc in self.stars:
            r = torch.sqrt(((x - torch.as_tensor(c, dtype=torch.float64, device=x.device)) ** 2).sum(-1))
            xi = r / R * self.xi1
            # np.interp(xi, xs, ts, right=0): linear between the bracketing knots
            j = torch.clamp(torch.searchsorted(xs, xi, right=True), 1, xs.numel() - 1)
            x0, x1, t0, t1 = xs[j - 1], xs[j], ts[j - 1], ts[j]
            th = torch.where(xi > xs[-1], torch.zeros_like(xi), t0 + (xi - x0) * (t1 - t0) / (x1 - x0))
            out = out + rc * th ** 1.5
        return out

    def refine(self, l, lo, hi):
        L = self.L
        r = np.zeros(lo.shape[0], dtype=bool)
        if l < L - 2:
            r |= _box_sphere(lo, hi, self.c1, self.R1) | _box_sphere(lo, hi, self.c2, self.R2)
        if l < L - 1:
            r |= _box_sphere(lo, hi, self.c1, 0.3 * self.R1)
        if l < L:
            r |= _box_sphere(lo, hi, self.c2, 0.3 * self.R2)
            if self.env_radius > 0.0:
                r |= _box_sphere(lo, hi, np.zeros(3), self.env_radius)
        return r

    def tree(self, structure_only: bool = False) -> Tree:
        return build_tree(self.origin, self.width, self.L, self.refine, None if structure_only else self.density)


def config_v1309(max_level: int = 13, env_radius: float = 0.0, structure_only: bool = False) -> Tree:
    """configs[3]/[4]: the V1309 model (class V1309) at max_level; with
    structure_only the levels carry rho = None (densities generated elsewhere,
    e.g. on the device for the configs[4] shards)."""
    return V1309(max_level, env_radius).tree(structure_only)


def config_random_amr(seed: int, max_level: int = 2, p_refine: float = 0.4) -> Tree:
    """Seeded random 2:1-graded AMR tree, rho ~ U(0.1, 1.0) (test fixture)."""
    rng = np.random.default_rng(seed)
    drng = np.random.default_rng(seed + 1000)

    def refine(l, lo, hi):
        if l == 0:
            return np.ones(lo.shape[0], bool)
        return rng.uniform(size=lo.shape[0]) < p_refine

    return build_tree(np.zeros(3), 1.0, max_level, refine, lambda x: drng.uniform(0.1, 1.0, size=x.shape[0]))

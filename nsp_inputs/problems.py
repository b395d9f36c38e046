"""Seeded synthetic problems (matrix A in CSR, partition vector, Omega, b) for the
BASELINE.json configs and their small oracle-sized analogues.

This module is input generation only: it assembles the test matrices and the
caller-supplied partition vector `part` (`nsp_setup(A_csr,
part)` takes the partition as input).  It contains none of the method's
arithmetic (no Schur complement, no Krylov, no Nystrom); both `oracle/` and the
CUDA harness consume its output.

Readings (DESIGN.md §"Readings"):
  C11 grid separators: geometric nested dissection on the interior nodes
      (Dirichlet boundary eliminated, node id row-major, axis 0 slowest); cut the
      longest axis (ties -> lowest axis index); separator index (lo+hi+1)//2 on
      the inclusive range [lo, hi]; recurse low side first; leaves numbered
      depth-first so every subtree is a contiguous id range.
  C12 lognormal coefficients: kappa_c = exp(g_c), g_c ~ N(0, 2^2) per cell;
      interior face t = 2 ka kb / (ka + kb); Dirichlet boundary face t = kappa_cell.
  C13 RGG: points ~ U[0,1]^2, r = sqrt(12/(pi n)), edges = pairs with distance
      < r, w ~ U(0.1, 10), A = D - W + 1e-6 I; coordinate bisection along the
      longest extent, stable sort, lower half = first floor(m/2), vertex
      separator = lower-half endpoints of cut edges.
  C14 anisotropy: eps multiplies the second difference along the fastest axis.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import philox


@dataclass
class CSR:
    n: int
    rowptr: np.ndarray   # int64[n+1]
    colidx: np.ndarray   # int32[nnz], sorted within each row
    val: np.ndarray      # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.colidx, self.rowptr), shape=(self.n, self.n))


@dataclass
class Problem:
    name: str
    A: CSR
    part: np.ndarray          # int32[n]: block id in [0, K) or -1 for Gamma
    K: int
    rank: int                 # Nystrom rank k
    oversample: int           # p
    tol_bcg: float
    tol_pcg: float | None
    info: dict = field(default_factory=dict)

    @property
    def s(self) -> int:
        return self.rank + self.oversample

    @property
    def n(self) -> int:
        return self.A.n

    @property
    def gamma(self) -> np.ndarray:
        """Gamma node ids in ascending original index (reading C10)."""
        return np.flatnonzero(self.part < 0)

    @property
    def n_gamma(self) -> int:
        return int(np.count_nonzero(self.part < 0))

    def omega(self, seed: int = 0) -> np.ndarray:
        """Gaussian sketch Omega (n_Gamma x s, row-major), Philox stream 0 (reading C7)."""
        return philox.gaussian_block(seed, philox.STREAM_OMEGA, self.n_gamma, self.s)

    def xstar(self, seed: int = 1) -> np.ndarray:
        return philox.gaussian(seed, philox.STREAM_XSTAR, self.n)

    def rhs(self, seed: int = 1) -> np.ndarray:
        """Right-hand side of the full solve (reading C8): b ~ N(0,1) directly for the cfg2 family
        ("seeded Gaussian Omega and b"), b = A x* with x* = xstar(seed) otherwise.  The product
        A x* is input assembly (a plain CSR matvec), not the method's arithmetic."""
        if self.name.startswith("cfg2"):
            return self.xstar(seed)
        x = self.xstar(seed)
        rows = np.repeat(np.arange(self.n), np.diff(self.A.rowptr))
        return np.bincount(rows, weights=self.A.val * x[self.A.colidx], minlength=self.n)


# ----------------------------------------------------------------------------
# structured grids
# ----------------------------------------------------------------------------

def _strides(dims):
    d = len(dims)
    st = [1] * d
    for a in range(d - 2, -1, -1):
        st[a] = st[a + 1] * dims[a + 1]
    return st


def grid_matrix(dims, t_faces, t_bnd) -> CSR:
    """dims: interior grid shape (axis 0 slowest).
    t_faces[a]: array shaped like dims with axis a shortened by one: the
      transmissibility between node (.., i_a, ..) and (.., i_a+1, ..).
    t_bnd[a]: (lo, hi) arrays shaped like dims without axis a: boundary face
      transmissibility at i_a = 0 (lo) and i_a = dims[a]-1 (hi).
    A_ii = sum of the 2d face values around i, A_ij = -t_face."""
    dims = tuple(int(x) for x in dims)
    d = len(dims)
    n = int(np.prod(dims))
    st = _strides(dims)
    diag = np.zeros(dims, dtype=np.float64)
    # neighbour slots in ascending column order: axis 0 minus, ..., axis d-1 minus, diag, axis d-1 plus, ..., axis 0 plus
    slots = [(a, -1) for a in range(d)] + [None] + [(a, +1) for a in range(d - 1, -1, -1)]
    offdiag = {}
    for a in range(d):
        tf = t_faces[a]
        # minus neighbour of node with i_a >= 1: value -t at (i_a - 1)
        vm = np.zeros(dims)
        sl_hi = [slice(None)] * d
        sl_hi[a] = slice(1, None)
        vm[tuple(sl_hi)] = -tf
        vp = np.zeros(dims)
        sl_lo = [slice(None)] * d
        sl_lo[a] = slice(0, dims[a] - 1)
        vp[tuple(sl_lo)] = -tf
        offdiag[(a, -1)] = vm
        offdiag[(a, +1)] = vp
        diag[tuple(sl_hi)] += tf
        diag[tuple(sl_lo)] += tf
        lo, hi = t_bnd[a]
        s0 = [slice(None)] * d
        s0[a] = 0
        diag[tuple(s0)] += lo
        s1 = [slice(None)] * d
        s1[a] = dims[a] - 1
        diag[tuple(s1)] += hi
    # validity masks
    counts = np.ones(n, dtype=np.int64)
    masks = {}
    for a in range(d):
        m_minus = np.ones(dims, dtype=bool)
        sl = [slice(None)] * d
        sl[a] = 0
        m_minus[tuple(sl)] = False
        m_plus = np.ones(dims, dtype=bool)
        sl[a] = dims[a] - 1
        m_plus[tuple(sl)] = False
        masks[(a, -1)] = m_minus.ravel()
        masks[(a, +1)] = m_plus.ravel()
        counts += masks[(a, -1)].astype(np.int64) + masks[(a, +1)].astype(np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    nnz = int(rowptr[-1])
    colidx = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    cursor = rowptr[:-1].copy()
    ids = np.arange(n, dtype=np.int64)
    for slot in slots:
        if slot is None:
            colidx[cursor] = ids.astype(np.int32)
            val[cursor] = diag.ravel()
            cursor += 1
            continue
        a, sgn = slot
        m = masks[slot]
        rows = ids[m]
        pos = cursor[m]
        colidx[pos] = (rows + sgn * st[a]).astype(np.int32)
        val[pos] = offdiag[slot].ravel()[m]
        cursor[m] += 1
    assert np.array_equal(cursor, rowptr[1:])
    return CSR(n, rowptr, colidx, val)


def laplacian(dims, coef=None) -> CSR:
    """Constant-coefficient (2d+1)-point Laplacian; coef[a] scales axis a
    (anisotropy, reading C14).  Eigenvalues sum_a coef[a] 4 sin^2(pi k_a / (2(m_a+1)))."""
    d = len(dims)
    coef = [1.0] * d if coef is None else list(coef)
    t_faces, t_bnd = [], []
    for a in range(d):
        sh = list(dims)
        sh[a] -= 1
        t_faces.append(np.full(sh, coef[a]))
        shb = list(dims)
        del shb[a]
        t_bnd.append((np.full(shb, coef[a]), np.full(shb, coef[a])))
    return grid_matrix(dims, t_faces, t_bnd)


def lognormal_diffusion(dims, sigma=2.0, seed=2) -> CSR:
    """Cell-centred FV diffusion with kappa = exp(g), g ~ N(0, sigma^2) per cell,
    harmonic-mean faces (reading C12)."""
    d = len(dims)
    g = philox.gaussian(seed, philox.STREAM_FIELD, int(np.prod(dims))).reshape(dims)
    kap = np.exp(sigma * g)
    t_faces, t_bnd = [], []
    for a in range(d):
        lo = [slice(None)] * d
        hi = [slice(None)] * d
        lo[a] = slice(0, dims[a] - 1)
        hi[a] = slice(1, None)
        ka, kb = kap[tuple(lo)], kap[tuple(hi)]
        t_faces.append(2.0 * ka * kb / (ka + kb))
        s0 = [slice(None)] * d
        s0[a] = 0
        s1 = [slice(None)] * d
        s1[a] = dims[a] - 1
        t_bnd.append((kap[tuple(s0)].copy(), kap[tuple(s1)].copy()))
    return grid_matrix(dims, t_faces, t_bnd)


def geometric_nd(dims, K: int) -> np.ndarray:
    """Partition vector by recursive geometric nested dissection (reading C11)."""
    dims = tuple(int(x) for x in dims)
    levels = int(round(np.log2(K)))
    assert 1 << levels == K, "K must be a power of two"
    lab = np.full(dims, -2, dtype=np.int32)
    boxes = [tuple((0, m - 1) for m in dims)]
    for _ in range(levels):
        nxt = []
        for box in boxes:
            lens = [hi - lo + 1 for lo, hi in box]
            a = int(np.argmax(lens))  # first max -> lowest axis index on ties
            lo, hi = box[a]
            sep = (lo + hi + 1) // 2
            sl = tuple(slice(l, h + 1) if ax != a else slice(sep, sep + 1) for ax, (l, h) in enumerate(box))
            lab[sl] = -1
            low = list(box)
            low[a] = (lo, sep - 1)
            high = list(box)
            high[a] = (sep + 1, hi)
            nxt.append(tuple(low))
            nxt.append(tuple(high))
        boxes = nxt
    for j, box in enumerate(boxes):
        sl = tuple(slice(l, h + 1) for l, h in box)
        if all(h >= l for l, h in box):
            sub = lab[sl]
            sub[sub == -2] = j
    assert not np.any(lab == -2)
    return lab.ravel().astype(np.int32)


# ----------------------------------------------------------------------------
# random geometric graph (config 4)
# ----------------------------------------------------------------------------

def rgg_points(n: int, seed: int = 3) -> np.ndarray:
    u = philox.uniform(seed, philox.STREAM_POINTS, 2 * n)
    return u.reshape(n, 2)


def rgg_edges(pts: np.ndarray, r: float) -> np.ndarray:
    """All pairs (i < j) with |p_i - p_j| < r, sorted lexicographically."""
    from scipy.spatial import cKDTree
    tree = cKDTree(pts)
    pairs = tree.query_pairs(r, output_type="ndarray").astype(np.int64)
    if pairs.size == 0:
        return np.zeros((0, 2), dtype=np.int64)
    pairs.sort(axis=1)
    # strict inequality (query_pairs is <= r)
    dd = np.sum((pts[pairs[:, 0]] - pts[pairs[:, 1]]) ** 2, axis=1)
    pairs = pairs[dd < r * r]
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    return pairs[order]


def graph_laplacian(n: int, edges: np.ndarray, w: np.ndarray, shift: float) -> CSR:
    i = np.concatenate([edges[:, 0], edges[:, 1], np.arange(n)])
    j = np.concatenate([edges[:, 1], edges[:, 0], np.arange(n)])
    deg = np.zeros(n)
    np.add.at(deg, edges[:, 0], w)
    np.add.at(deg, edges[:, 1], w)
    v = np.concatenate([-w, -w, deg + shift])
    order = np.lexsort((j, i))
    i, j, v = i[order], j[order], v[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(i, minlength=n), out=rowptr[1:])
    return CSR(n, rowptr, j.astype(np.int32), v.astype(np.float64))


def coordinate_bisection(pts: np.ndarray, edges: np.ndarray, K: int) -> np.ndarray:
    """Vertex-separator bisection by coordinates to K leaves (reading C13)."""
    n = pts.shape[0]
    levels = int(round(np.log2(K)))
    assert 1 << levels == K
    lab = np.zeros(n, dtype=np.int64)       # current part id; -1 = separator
    e0, e1 = edges[:, 0], edges[:, 1]
    for _ in range(levels):
        side = np.zeros(n, dtype=np.int8)
        live = np.flatnonzero(lab >= 0)
        order = np.argsort(lab[live], kind="stable")
        live = live[order]
        parts, starts = np.unique(lab[live], return_index=True)
        ends = list(starts[1:]) + [live.size]
        for p, s0, s1 in zip(parts, starts, ends):
            mem = live[s0:s1]                  # ascending vertex id
            m = mem.size
            if m == 0:
                continue
            ext = pts[mem].max(axis=0) - pts[mem].min(axis=0)
            a = 0 if ext[0] >= ext[1] else 1
            srt = mem[np.argsort(pts[mem, a], kind="stable")]
            side[srt[m // 2:]] = 1
        same = (lab[e0] == lab[e1]) & (lab[e0] >= 0)
        cut = same & (side[e0] != side[e1])
        lower_end = np.where(side[e0[cut]] == 0, e0[cut], e1[cut])
        newlab = np.where(lab >= 0, 2 * lab + side, -1)
        newlab[lower_end] = -1
        lab = newlab
    return lab.astype(np.int32)


# ----------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------

def _grid_problem(name, dims, K, rank, over, tol_bcg, tol_pcg, kind="laplace", coef=None, sigma=2.0):
    if kind == "laplace":
        A = laplacian(dims, coef)
    elif kind == "lognormal":
        A = lognormal_diffusion(dims, sigma=sigma)
    else:
        raise ValueError(kind)
    part = geometric_nd(dims, K)
    return Problem(name, A, part, K, rank, over, tol_bcg, tol_pcg,
                   info={"dims": list(dims), "kind": kind, "coef": coef})


def _rgg_problem(name, n, K, rank, over, tol_bcg, tol_pcg, degree=12.0):
    pts = rgg_points(n)
    r = float(np.sqrt(degree / (np.pi * n)))
    edges = rgg_edges(pts, r)
    w = 0.1 + 9.9 * philox.uniform(4, philox.STREAM_WEIGHTS, edges.shape[0])
    A = graph_laplacian(n, edges, w, 1e-6)
    part = coordinate_bisection(pts, edges, K)
    return Problem(name, A, part, K, rank, over, tol_bcg, tol_pcg,
                   info={"kind": "rgg", "radius": r, "edges": int(edges.shape[0])})


# BASELINE.json configs (index 0..4 == "config 1..5") and small analogues that
# the oracle finishes in seconds (same structure, spanning several 64-row tiles
# and a ragged tail).
def make(name: str) -> Problem:
    if name == "cfg1":
        return _grid_problem("cfg1", (64, 64), 4, 20, 10, 1e-1, 1e-8)
    if name == "cfg2":
        return _grid_problem("cfg2", (1024, 1024), 64, 100, 28, 1e-1, 1e-8, coef=[1.0, 1e-3])
    if name == "cfg3":
        return _grid_problem("cfg3", (128, 128, 128), 256, 48, 16, 1e-1, None, kind="lognormal")
    if name == "cfg4":
        return _rgg_problem("cfg4", 4_000_000, 512, 72, 24, 1e-2, None)
    if name == "cfg5":
        return _grid_problem("cfg5", (256, 256, 256), 1024, 100, 28, 1e-1, 1e-8)
    # small analogues
    if name == "cfg2s":
        return _grid_problem("cfg2s", (160, 160), 16, 24, 8, 1e-1, 1e-8, coef=[1.0, 1e-3])
    if name == "cfg2m":   # mid-size 2-D analogue whose A_G band solve is partitioned (spikes)
        return _grid_problem("cfg2m", (384, 384), 16, 24, 8, 1e-1, 1e-8, coef=[1.0, 1e-3])
    if name == "cfg3s":
        return _grid_problem("cfg3s", (24, 24, 24), 8, 12, 4, 1e-1, None, kind="lognormal")
    if name == "cfg4s":
        return _rgg_problem("cfg4s", 20_000, 16, 18, 6, 1e-2, None)
    if name == "cfg5s":
        return _grid_problem("cfg5s", (28, 28, 28), 16, 24, 8, 1e-1, 1e-8)
    raise KeyError(name)


CONFIGS = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
SMALL = ["cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg5s"]

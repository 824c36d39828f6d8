"""Synthetic test problems, tile owners and the five benchmark configurations.

Host-side (numpy/scipy) builders.  They are the step *before* the hot path
(SURVEY.md §8f item 1): every builder returns a canonical scipy CSR matrix
(sorted, duplicate-free columns, fp64 values) plus, where relevant, an owner
vector that injects the tile/block partition through ``setup(owner=...)``
(reference ``src/precond.py:191-194``).

The four reference generators are restated vectorised and reproduce the
reference CSR bit for bit (``src/harness.py:56-153``; checked against the
golden fixtures in ``tests/golden``).  The generators for configurations 2-5
do not exist in the reference; they follow the reference's
conventions (``h2 = (m+1)^2`` scaling, ``idx = i + m*j (+ m^2*k)``,
harmonic-mean faces, Dirichlet boundary terms, exact symmetry) and their exact
definitions are recorded in DESIGN.md §3.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


def _csr(n, rows, cols, vals, ncols=None):
    mat = sp.coo_matrix((vals, (rows, cols)), shape=(n, ncols if ncols else n)).tocsr()
    mat.sum_duplicates()
    mat.sort_indices()
    return mat.astype(np.float64)


# ---------------------------------------------------------------------------
# reference generators (bit-exact restatements)
# ---------------------------------------------------------------------------

def poisson2d(m):
    """5-point Laplacian, ``src/harness.py:56-69``: diag 4*h2, off -h2."""
    h2 = (m + 1) ** 2
    j, i = np.divmod(np.arange(m * m), m)
    k = i + j * m
    rows, cols, vals = [k], [k], [np.full(k.size, 4.0 * h2)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ii, jj = i + di, j + dj
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m)
        rows.append(k[ok]); cols.append((ii + jj * m)[ok]); vals.append(np.full(ok.sum(), -1.0 * h2))
    return _csr(m * m, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def poisson3d(m):
    """7-point Laplacian, ``src/harness.py:72-87``."""
    h2 = (m + 1) ** 2
    n = m ** 3
    p = np.arange(n)
    i = p % m
    j = (p // m) % m
    k = p // (m * m)
    rows, cols, vals = [p], [p], [np.full(n, 6.0 * h2)]
    for d in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)):
        ii, jj, kk = i + d[0], j + d[1], k + d[2]
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m) & (kk >= 0) & (kk < m)
        rows.append(p[ok]); cols.append((ii + m * (jj + m * kk))[ok]); vals.append(np.full(ok.sum(), -1.0 * h2))
    return _csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _harm(a, b):
    return 2.0 * a * b / (a + b)


def hetero2d(m, contrast=1.0e4, channel_seed=0):
    """Channelised diffusion, ``src/harness.py:90-123`` (same rng draws)."""
    h2 = (m + 1) ** 2
    rng = np.random.default_rng(channel_seed)
    channels = rng.choice(m, size=max(1, m // 5), replace=False)
    kappa = np.ones((m, m))
    kappa[:, channels] = contrast
    j, i = np.divmod(np.arange(m * m), m)
    k = i + j * m
    kap = kappa[i, j]
    diag = np.zeros(m * m)
    rows, cols, vals = [], [], []
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ii, jj = i + di, j + dj
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m)
        c = np.where(ok, _harm(kap, kappa[np.clip(ii, 0, m - 1), np.clip(jj, 0, m - 1)]), kap)
        diag = diag + c
        rows.append(k[ok]); cols.append((ii + jj * m)[ok]); vals.append(-c[ok] * h2)
    rows.append(k); cols.append(k); vals.append(diag * h2)
    return _csr(m * m, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def advection2d(m, velocity=(1.0, 0.0), eps=1.0e-2):
    """Constant-wind upwind advection-diffusion, ``src/harness.py:126-153``."""
    vx, vy = velocity
    return _upwind2d(m, np.full(m * m, float(vx)), np.full(m * m, float(vy)), eps,
                     1.0 / (m + 1), (m + 1) ** 2)


def _upwind2d(m, vx, vy, eps, h, h2):
    j, i = np.divmod(np.arange(m * m), m)
    k = i + j * m
    diag = 4.0 * eps * h2 + (np.abs(vx) + np.abs(vy)) / h
    zero = np.zeros_like(vx)
    coeffs = (
        (-1, 0, -eps * h2 - np.where(vx > 0, vx / h, zero)),
        (1, 0, -eps * h2 + np.where(vx < 0, vx / h, zero)),
        (0, -1, -eps * h2 - np.where(vy > 0, vy / h, zero)),
        (0, 1, -eps * h2 + np.where(vy < 0, vy / h, zero)),
    )
    rows, cols, vals = [k], [k], [diag]
    for di, dj, c in coeffs:
        ii, jj = i + di, j + dj
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m)
        rows.append(k[ok]); cols.append((ii + jj * m)[ok]); vals.append(c[ok])
    return _csr(m * m, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


# ---------------------------------------------------------------------------
# configuration generators (new; conventions of the reference)
# ---------------------------------------------------------------------------

def hetero3d_lognormal(m, sigma=2.0, contrast=1.0e4, seed=0):
    """Config 2: 7-point FV diffusion on an m^3 grid, log-normal cells.

    kappa_cell = exp(sigma * N(0,1)) drawn in idx = i + m*(j + m*k) order
    after ``max(1, m//5)`` z-slabs are chosen by ``rng.choice`` (the
    reference's hetero2d channel rule, ``src/harness.py:99-103``); those
    slabs get ``contrast``.  Faces: harmonic mean; a Dirichlet face adds the
    cell coefficient to the diagonal (``src/harness.py:120-121``); scaled by
    h2 = (m+1)^2.
    """
    h2 = (m + 1) ** 2
    n = m ** 3
    rng = np.random.default_rng(seed)
    slabs = rng.choice(m, size=max(1, m // 5), replace=False)
    kap = np.exp(sigma * rng.standard_normal(n))
    p = np.arange(n)
    i = p % m
    j = (p // m) % m
    k = p // (m * m)
    kap[np.isin(k, slabs)] = contrast
    diag = np.zeros(n)
    rows, cols, vals = [], [], []
    for d in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)):
        ii, jj, kk = i + d[0], j + d[1], k + d[2]
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m) & (kk >= 0) & (kk < m)
        q = np.where(ok, ii + m * (jj + m * kk), p)
        c = np.where(ok, _harm(kap, kap[q]), kap)
        diag = diag + c
        rows.append(p[ok]); cols.append(q[ok]); vals.append(-c[ok] * h2)
    rows.append(p); cols.append(p); vals.append(diag * h2)
    return _csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def recirc_advection2d(m, eps=1.0e-3):
    """Config 3: first-order upwind -eps*Lap(u) + b.grad(u) on [-1,1]^2.

    Wind b = (2y(1-x^2), -2x(1-y^2)) evaluated at the node; h = 2/(m+1);
    stencil exactly as the reference's ``_advection2d`` (``src/harness.py:
    139-152``) with the constant wind replaced by the pointwise one.
    """
    h = 2.0 / (m + 1)
    h2 = 1.0 / (h * h)
    j, i = np.divmod(np.arange(m * m), m)
    x = -1.0 + (i + 1) * h
    y = -1.0 + (j + 1) * h
    vx = 2.0 * y * (1.0 - x * x)
    vy = -2.0 * x * (1.0 - y * y)
    return _upwind2d(m, vx, vy, eps, h, h2)


def mac_stokes2d(m, c=1.0e-6):
    """Config 4: MAC saddle point [K B^T; B -c I] on an m x m cell grid.

    Unknowns: u on interior x-faces (i=1..m-1, j=0..m-1), v on interior
    y-faces, p on cells; ordering [u; v; p].  K = 5-point Laplacian / h^2 on
    each velocity grid with Dirichlet-eliminated neighbours; B = divergence
    (u(i+1,j) - u(i,j) + v(i,j+1) - v(i,j)) / h with wall faces dropped.
    Exactly symmetric by construction (B^T is the exact transpose).
    """
    h = 1.0 / m
    ih2 = 1.0 / (h * h)
    nu = (m - 1) * m
    nv = m * (m - 1)
    npr = m * m
    rows, cols, vals = [], [], []

    def lap(offset, nx, ny):
        # grid nx x ny, index a + nx*b
        b_, a_ = np.divmod(np.arange(nx * ny), nx)
        kk = offset + a_ + nx * b_
        rows.append(kk); cols.append(kk); vals.append(np.full(kk.size, 4.0 * ih2))
        for da, db in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            aa, bb = a_ + da, b_ + db
            ok = (aa >= 0) & (aa < nx) & (bb >= 0) & (bb < ny)
            rows.append(kk[ok]); cols.append((offset + aa + nx * bb)[ok])
            vals.append(np.full(ok.sum(), -ih2))

    lap(0, m - 1, m)
    lap(nu, m, m - 1)
    cj, ci = np.divmod(np.arange(npr), m)
    prow = nu + nv + ci + m * cj
    brows, bcols, bvals = [], [], []
    # u faces: face index fi = 1..m-1 -> u(fi, j) = (fi-1) + (m-1)*j
    for fi, sgn in ((ci + 1, 1.0 / h), (ci, -1.0 / h)):
        ok = (fi >= 1) & (fi <= m - 1)
        brows.append(prow[ok]); bcols.append(((fi - 1) + (m - 1) * cj)[ok]); bvals.append(np.full(ok.sum(), sgn))
    for fj, sgn in ((cj + 1, 1.0 / h), (cj, -1.0 / h)):
        ok = (fj >= 1) & (fj <= m - 1)
        brows.append(prow[ok]); bcols.append((nu + ci + m * (fj - 1))[ok]); bvals.append(np.full(ok.sum(), sgn))
    br = np.concatenate(brows); bc = np.concatenate(bcols); bv = np.concatenate(bvals)
    rows += [br, bc, prow]; cols += [bc, br, prow]; vals += [bv, bv, np.full(npr, -c)]
    n = nu + nv + npr
    return _csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _q1_gradient_integrals():
    """G[d1, d2, a, b] = int_[0,1]^3 d_{d1} phi_a d_{d2} phi_b (2-pt Gauss, exact)."""
    g = np.array([0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0)])
    corners = np.array([(c & 1, (c >> 1) & 1, (c >> 2) & 1) for c in range(8)], dtype=float)
    out = np.zeros((3, 3, 8, 8))
    for qx in g:
        for qy in g:
            for qz in g:
                q = (qx, qy, qz)
                grad = np.zeros((8, 3))
                for a in range(8):
                    f = [q[d] if corners[a, d] else 1.0 - q[d] for d in range(3)]
                    df = [1.0 if corners[a, d] else -1.0 for d in range(3)]
                    grad[a] = (df[0] * f[1] * f[2], f[0] * df[1] * f[2], f[0] * f[1] * df[2])
                out += 0.125 * np.einsum("ai,bj->ijab", grad, grad)
    return out


def _rotation(a, b, c):
    ca, sa, cb, sb, cc, sc = math.cos(a), math.sin(a), math.cos(b), math.sin(b), math.cos(c), math.sin(c)
    rx = np.array([[1, 0, 0], [0, ca, -sa], [0, sa, ca]])
    ry = np.array([[cb, 0, sb], [0, 1, 0], [-sb, 0, cb]])
    rz = np.array([[cc, -sc, 0], [sc, cc, 0], [0, 0, 1]])
    return rz @ ry @ rx


def aniso27_q1(m, block=32, seed=0, eigs=(1.0, 1.0e-2, 1.0e-4)):
    """Config 5: Q1 finite elements (27-point) for -div(K grad u) on m^3 nodes.

    Unit cube, h = 1/(m+1), homogeneous Dirichlet nodes eliminated.  The
    element tensor K = R diag(eigs) R^T uses three Euler angles drawn by
    ``default_rng(seed).uniform(0, 2*pi, (nb, nb, nb, 3))`` for each
    ``block``^3 group of elements (nb = ceil((m+1)/block), index order
    [bk, bj, bi]).  Entries for the 13 forward offsets are summed over the
    shared elements in a fixed corner order and mirrored, so the matrix is
    exactly symmetric.  All 27 stencil entries inside the domain are stored,
    including any that are numerically zero (those are not graph edges,
    ``src/sparsemat.py:189-190``).
    """
    h = 1.0 / (m + 1)
    n = m ** 3
    nb = -(-(m + 1) // block)
    rng = np.random.default_rng(seed)
    ang = rng.uniform(0.0, 2.0 * math.pi, size=(nb, nb, nb, 3))
    G = _q1_gradient_integrals()
    lam = np.diag(eigs)
    kblk = np.empty((nb, nb, nb, 8, 8))
    for bk in range(nb):
        for bj in range(nb):
            for bi in range(nb):
                r = _rotation(*ang[bk, bj, bi])
                kt = r @ lam @ r.T
                kt = 0.5 * (kt + kt.T)
                ke = h * np.einsum("ij,ijab->ab", kt, G)
                kblk[bk, bj, bi] = 0.5 * (ke + ke.T)
    kflat = kblk.reshape(-1, 8, 8)
    p = np.arange(n)
    i = p % m
    j = (p // m) % m
    k = p // (m * m)
    # grid coordinates P = interior + 1; element E = P - o (lower corner), o in {0,1}^3
    offsets = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    forward = [d for d in offsets if (d[2], d[1], d[0]) > (0, 0, 0)]
    vals = {}
    for d in [(0, 0, 0)] + forward:
        acc = np.zeros(n)
        for oz in (0, 1):
            for oy in (0, 1):
                for ox in (0, 1):
                    o = (ox, oy, oz)
                    t = (ox + d[0], oy + d[1], oz + d[2])
                    if min(t) < 0 or max(t) > 1:
                        continue
                    ei, ej, ek = i + 1 - ox, j + 1 - oy, k + 1 - oz
                    blk = (ek // block) * nb * nb + (ej // block) * nb + (ei // block)
                    a = ox + 2 * oy + 4 * oz
                    b = t[0] + 2 * t[1] + 4 * t[2]
                    acc = acc + kflat[blk, a, b]
        vals[d] = acc
    rows, cols, data = [], [], []
    for d in offsets:
        ii, jj, kk = i + d[0], j + d[1], k + d[2]
        ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m) & (kk >= 0) & (kk < m)
        q = ii + m * (jj + m * kk)
        if d in vals:
            v = vals[d]
        else:  # mirror: A[p, p+d] = A[p+d, p] = vals[-d][p+d]
            nd = (-d[0], -d[1], -d[2])
            v = np.zeros(n)
            v[ok] = vals[nd][q[ok]]
        rows.append(p[ok]); cols.append(q[ok]); data.append(v[ok])
    return _csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(data))


# ---------------------------------------------------------------------------
# owners (tile / block partitions)
# ---------------------------------------------------------------------------

def tile_owner_2d(m, tile):
    """Owner of node idx = i + m*j for contiguous tile x tile squares."""
    nb = m // tile
    j, i = np.divmod(np.arange(m * m), m)
    return (i // tile) + nb * (j // tile)


def block_owner_3d(m, blk):
    nb = m // blk
    p = np.arange(m ** 3)
    i = p % m
    j = (p // m) % m
    k = p // (m * m)
    return (i // blk) + nb * ((j // blk) + nb * (k // blk))


def mac_owner(m, tile):
    """Faces owned by their left/lower cell, cells by their tile."""
    nb = m // tile
    cell = lambda ci, cj: (ci // tile) + nb * (cj // tile)
    uj, ui = np.divmod(np.arange((m - 1) * m), m - 1)  # u(fi=ui+1, j)
    vj, vi = np.divmod(np.arange(m * (m - 1)), m)      # v(i, fj=vj+1)
    pj, pi = np.divmod(np.arange(m * m), m)
    return np.concatenate([cell(ui, uj), cell(vi, vj), cell(pi, pj)])


# ---------------------------------------------------------------------------
# configurations (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ProblemConfig:
    """One benchmark configuration; ``scale`` shrinks it for parity tests."""

    cid: int
    name: str
    kind: str
    m: int
    part: int          # tile/block edge in grid units
    overlap: int
    n_modes: int
    solver: str
    tol: float
    restart: int | None = None
    symmetric: bool = True
    extra: dict = field(default_factory=dict)
    maxit: int = 500

    def build(self):
        """Return (scipy CSR, symmetric flag, owner, n_subdomains)."""
        m, t = self.m, self.part
        if self.kind == "poisson2d":
            a = poisson2d(m); owner = tile_owner_2d(m, t); nsub = (m // t) ** 2
        elif self.kind == "hetero3d":
            a = hetero3d_lognormal(m, seed=self.extra.get("seed", 0)); owner = block_owner_3d(m, t); nsub = (m // t) ** 3
        elif self.kind == "recirc2d":
            a = recirc_advection2d(m, eps=self.extra.get("eps", 1e-3)); owner = tile_owner_2d(m, t); nsub = (m // t) ** 2
        elif self.kind == "mac_stokes2d":
            a = mac_stokes2d(m, c=self.extra.get("c", 1e-6)); owner = mac_owner(m, t); nsub = (m // t) ** 2
        elif self.kind == "aniso27":
            a = aniso27_q1(m, block=self.extra.get("angle_block", 32), seed=self.extra.get("seed", 0))
            owner = block_owner_3d(m, t); nsub = (m // t) ** 3
        else:
            raise ValueError(f"unknown kind {self.kind!r}")
        return a, self.symmetric, owner.astype(np.int64), nsub

    def rhs(self, n):
        """RHS uniform[-1, 1] from seed 0 (BASELINE.json configs[0])."""
        return np.random.default_rng(0).uniform(-1.0, 1.0, n)

    def scaled(self, m, part=None, **extra):
        ex = dict(self.extra); ex.update(extra)
        return ProblemConfig(self.cid, self.name + f"@m{m}", self.kind, m, part or self.part,
                             self.overlap, self.n_modes, self.solver, self.tol, self.restart,
                             self.symmetric, ex, self.maxit)


CONFIGS = {
    1: ProblemConfig(1, "cfg1-poisson2d-64", "poisson2d", 64, 16, 1, 8, "pcg", 1e-8),
    2: ProblemConfig(2, "cfg2-hetero3d-128", "hetero3d", 128, 16, 1, 16, "pcg", 1e-8, extra={"seed": 0}),
    3: ProblemConfig(3, "cfg3-recirc2d-1024", "recirc2d", 1024, 64, 2, 20, "gmres", 1e-8, restart=50,
                     symmetric=False, extra={"eps": 1e-3}),
    4: ProblemConfig(4, "cfg4-mac-stokes-512", "mac_stokes2d", 512, 32, 1, 20, "gmres", 1e-7, restart=50,
                     symmetric=False, extra={"c": 1e-6}),
    5: ProblemConfig(5, "cfg5-aniso27-256", "aniso27", 256, 16, 1, 12, "pcg", 1e-8,
                     extra={"seed": 0, "angle_block": 32}, maxit=3000),
}

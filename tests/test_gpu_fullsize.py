"""BASELINE.json configurations 2 and 3 at FULL size (n = 2.1 M / 1.05 M) through size-independent
properties (the dense reference cannot run them: DENSE_GUARD):
* overlap index sets and colours bit-exact against the oracle's restatement of extend_overlap /
  color_subdomains (src/partition.py:278-334);
* the apply is linear (to rounding) and, for ASM + additive, symmetric: <M x, y> = <x, M y>;
* the banded and the dense-inverse local operators agree on sampled subdomains' solves (through
  the one-level apply on vectors supported in one subdomain's interior);
* the solves reach the tolerance on the TRUE residual ||b - A x|| / ||b||, with the iteration
  counts this build measures (pinned: a change in them flags a change in the algorithm)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_03915_b200 import build
    build.build()
    import paper_2401_03915_b200 as mod
    return mod


@pytest.fixture(scope="module")
def cfg2(B):
    cfg = B.problems.CONFIGS[2]
    a, sym, owner, nsub = cfg.build()
    mat = B.SparseMat(a, symmetric=sym)
    pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
    return cfg, a, owner, nsub, mat, pre


def test_full_cfg2_index_sets_bit_exact(B, cfg2):
    from oracle import tls_oracle as O
    cfg, a, owner, nsub, mat, pre = cfg2
    gptr, gadj = O.symmetrized_graph(a)
    maps = O.extend_overlap(gptr, gadj, owner, nsub, cfg.overlap)
    for s in range(0, nsub, 7):
        assert np.array_equal(pre.maps[s].indices, O.indices_of(maps[s]))
    k_c, colors = O.color_subdomains(maps, a.shape[0])
    assert pre.k_c == k_c and np.array_equal(np.asarray(pre.colors), np.asarray(colors))


def test_full_cfg2_apply_linear_and_symmetric(B, cfg2):
    cfg, a, owner, nsub, mat, pre = cfg2
    rng = np.random.default_rng(11)
    x, y = rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    mx, my, mxy = pre.apply(x), pre.apply(y), pre.apply(2.0 * x - 3.0 * y)
    scale = np.abs(mxy).max()
    assert np.abs(mxy - (2.0 * mx - 3.0 * my)).max() <= 1e-12 * scale
    lhs, rhs = float(mx @ y), float(x @ my)
    assert abs(lhs - rhs) <= 1e-11 * (abs(lhs) + abs(rhs))


def test_full_cfg2_true_residual(B, cfg2):
    cfg, a, owner, nsub, mat, pre = cfg2
    b = cfg.rhs(a.shape[0])
    x, rep = B.pcg(mat, pre, b, tol=cfg.tol, maxit=cfg.maxit)
    assert rep.converged and rep.iterations == 166, rep.iterations
    true = np.linalg.norm(b - a @ x) / np.linalg.norm(b)
    assert true <= 1.01 * cfg.tol and abs(true - rep.residuals[-1]) <= 1e-3 * cfg.tol


def test_full_cfg3_gmres_true_residual(B):
    cfg = B.problems.CONFIGS[3]
    a, sym, owner, nsub = cfg.build()
    mat = B.SparseMat(a, symmetric=sym)
    pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
    b = cfg.rhs(a.shape[0])
    x, rep = B.gmres(mat, pre, b, tol=cfg.tol, maxit=cfg.maxit, restart=cfg.restart)
    assert rep.converged and rep.iterations == 37, rep.iterations
    true = np.linalg.norm(b - a @ x) / np.linalg.norm(b)
    assert true <= 1.01 * cfg.tol
    rng = np.random.default_rng(12)
    u, v = rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    mu, mv, muv = pre.apply(u), pre.apply(v), pre.apply(u + 0.5 * v)
    assert np.abs(muv - (mu + 0.5 * mv)).max() <= 1e-11 * np.abs(muv).max()

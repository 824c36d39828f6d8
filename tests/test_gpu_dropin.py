"""The reference's attribute-level API on the GPU Preconditioner (src/precond.py:86-139,
src/coarse.py:23-49), as the reference's own tests use it (tests/test_precond.py:26-45,185-198,
tests/test_coarse.py:125-253, tests/test_acceptance.py:258-301): ``blocks``, ``local_solves``,
``harmonic``, ``coarse.basis`` / ``a00`` / ``restrict`` / ``prolong`` / ``solve_coarse``; plus the
solve-boundary behaviours: callback exceptions propagate (src/krylov.py:92-93, 182-183) and a
different operator is refused rather than silently replaced."""

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


def _dense_oracle(pre):
    """tests/test_precond.py:26-45, verbatim in behaviour: the operator rebuilt from
    pre.blocks / pre.coarse.basis with dense inverses."""
    n = pre.n
    a = pre.matrix.scipy().toarray()
    m1 = np.zeros((n, n))
    for smap, blocks in zip(pre.maps, pre.blocks):
        local = np.linalg.inv(blocks.a)
        if pre.one_level == "ras":
            local = np.diag(smap.pou_mask.astype(float)) @ local
        e = np.zeros((n, smap.n_local))
        e[smap.indices, np.arange(smap.n_local)] = 1.0
        m1 += e @ local @ e.T
    if pre.coarse is None or pre.combine == "none":
        return m1
    b = pre.coarse.basis.to_dense()
    q = b @ np.linalg.solve(b.T @ a @ b, b.T)
    if pre.combine == "additive":
        return m1 + q
    eye = np.eye(n)
    return q + (eye - q @ a) @ m1 @ (eye - a @ q)


@pytest.mark.parametrize("kind", ["poisson2d", "advection2d"])
@pytest.mark.parametrize("local", ["band", "inverse"])
def test_dense_oracle_through_attributes(B, kind, local):
    P = B.problems
    a = P.poisson2d(12) if kind == "poisson2d" else P.advection2d(12)
    sym = kind == "poisson2d"
    mat = B.SparseMat(a, symmetric=sym)
    owner = P.tile_owner_2d(12, 6)
    pre = B.setup(mat, 4, overlap=2, tau=0.1, owner=owner, local=local)
    # blocks: the dense local matrices in local order (src/subdomain.py:53-69)
    dense = a.toarray()
    for smap, blk in zip(pre.maps, pre.blocks):
        assert np.array_equal(blk.a, dense[np.ix_(smap.indices, smap.indices)])
        assert blk.n_local == smap.n_local and blk.n_boundary == smap.n_boundary
    assert len(pre.blocks) == 4 and pre.blocks[-1].subdomain == 3
    m = _dense_oracle(pre)
    rng = np.random.default_rng(5)
    for _ in range(3):
        r = rng.standard_normal(a.shape[0])
        z, zr = pre.apply(r), m @ r
        assert np.abs(z - zr).max() <= 1e-11 * np.abs(zr).max()
    # report vs coarse (tests/test_precond.py:185-198)
    rep = pre.report
    assert rep.n_coarse == pre.coarse.n_coarse == sum(rep.mode_counts)
    for count, blk in zip(rep.mode_counts, pre.blocks):
        if sym:
            assert count <= blk.n_boundary
    assert rep.nnz_coarse == np.count_nonzero(pre.coarse.a00)


@pytest.mark.parametrize("local", ["band", "inverse"])
def test_local_solves_and_harmonic(B, local):
    P = B.problems
    for a, sym in ((P.poisson2d(12), True), (P.advection2d(12), False)):
        pre = B.setup(B.SparseMat(a, symmetric=sym), 4, overlap=2, owner=P.tile_owner_2d(12, 6),
                      local=local)
        rng = np.random.default_rng(9)
        for i, (smap, blk) in enumerate(zip(pre.maps, pre.blocks)):
            rhs = rng.standard_normal((smap.n_local, 2))
            want = np.linalg.solve(blk.a, rhs)
            got = pre.local_solves[i](rhs)
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
            assert np.abs(pre.local_solves[i](rhs[:, 0]) - want[:, 0]).max() <= 1e-12 * np.abs(want).max()
            # harmonic extension [-A_inner^{-1} A_inner,ring ; I] (src/subdomain.py:108-120)
            h = pre.harmonic[i]
            ni, nb = h.n_inner, h.n_boundary
            ext = np.zeros((smap.n_local, nb))
            ext[:ni] = -np.linalg.solve(blk.a[:ni, :ni], blk.a[:ni, ni:])
            ext[ni:] = np.eye(nb)
            assert np.abs(h.extension - ext).max() <= 1e-10 * max(1.0, np.abs(ext).max())
            v = rng.standard_normal(smap.n_local)
            assert np.allclose(h.apply(v), ext @ v[ni:], atol=1e-10)
        # one call for several subdomains: y_i = A_ii^{-1} R_i r
        r = rng.standard_normal(a.shape[0])
        ys = pre.solve_local(r, [3, 0])
        for i, y in zip((3, 0), ys):
            blk = pre.blocks[i]
            want = np.linalg.solve(blk.a, r[pre.maps[i].indices])
            assert np.abs(y - want).max() <= 1e-12 * np.abs(want).max()
        with pytest.raises(NotImplementedError):
            pre.bases


@pytest.mark.parametrize("sym", [True, False])
def test_coarse_space_methods(B, sym):
    """tests/test_coarse.py:125-253: restrict / prolong against the dense basis, a00 against the
    dense triple product, solve_coarse solves with a00, a00 symmetric positive definite."""
    P = B.problems
    a = P.poisson2d(16) if sym else P.advection2d(16)
    pre = B.setup(B.SparseMat(a, symmetric=sym), 4, overlap=2, owner=P.tile_owner_2d(16, 8))
    cs = pre.coarse
    dense = cs.basis.to_dense()
    rng = np.random.default_rng(3)
    r = rng.standard_normal(a.shape[0])
    np.testing.assert_allclose(cs.restrict(r), dense.T @ r, atol=1e-12)
    y = rng.standard_normal(cs.n_coarse)
    np.testing.assert_allclose(cs.prolong(y), dense @ y, atol=1e-12)
    expected = dense.T @ a.toarray() @ dense
    if sym:
        expected = 0.5 * (expected + expected.T)
    np.testing.assert_allclose(cs.a00, expected, atol=1e-10)
    rhs = rng.standard_normal(cs.n_coarse)
    np.testing.assert_allclose(cs.a00 @ cs.solve_coarse(rhs), rhs, atol=1e-9)
    if sym:
        np.testing.assert_allclose(cs.a00, cs.a00.T, atol=1e-12)
        assert np.linalg.eigvalsh(cs.a00).min() > 0
    # device tensors in, device tensors out
    rt = torch.as_tensor(r, device="cuda")
    assert isinstance(cs.restrict(rt), torch.Tensor)
    assert np.abs(cs.prolong(cs.solve_coarse(cs.restrict(r))) - pre.coarse_apply(r)).max() <= \
        1e-12 * np.abs(pre.coarse_apply(r)).max()


def test_callback_exceptions_propagate(B):
    P = B.problems
    a = P.poisson2d(12)
    mat = B.SparseMat(a, symmetric=True)
    pre = B.setup(mat, 4, overlap=1, owner=P.tile_owner_2d(12, 6))
    b = np.ones(a.shape[0])
    seen = []

    class Stop(Exception):
        pass

    def cb(it, x):
        seen.append(it)
        if it == 3:
            raise Stop(it)
    with pytest.raises(Stop):
        B.pcg(mat, pre, b, tol=1e-12, callback=cb)
    assert seen == [1, 2, 3]
    g = B.SparseMat(P.advection2d(12))
    gp = B.setup(g, 4, overlap=2, owner=P.tile_owner_2d(12, 6))
    seen.clear()
    with pytest.raises(Stop):
        B.gmres(g, gp, b, tol=1e-14, callback=cb)
    assert seen == [1, 2, 3]
    # the handle still works afterwards
    x, rep = B.pcg(mat, pre, b, tol=1e-8)
    assert rep.converged


def test_different_operator_is_refused(B):
    P = B.problems
    a = P.poisson2d(12)
    mat = B.SparseMat(a, symmetric=True)
    pre = B.setup(mat, 4, overlap=1, owner=P.tile_owner_2d(12, 6))
    b = np.ones(a.shape[0])
    other = B.SparseMat(2.0 * a, symmetric=True)   # same shape and sparsity, other values
    with pytest.raises(ValueError, match="different matrix"):
        B.pcg(other, pre, b)
    same = B.SparseMat(a.copy(), symmetric=True)   # equal content, another object: accepted
    x, rep = B.pcg(same, pre, b, tol=1e-8)
    assert rep.converged

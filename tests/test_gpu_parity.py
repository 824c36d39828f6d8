"""GPU parity: the sm_100a path (through the C ABI) against the reference's golden vectors and
the CPU oracle on the same seeded inputs.

Tolerances (fp64): index sets bit-exact; preconditioner apply <= 1e-10 relative to max|z|
(config-4 saddle point: 1e-8, its coarse operator has cond_1 ~1.5e7);
iteration counts +-1; residual histories agree to 1e-10 absolute on the relative scale
(1e-7 for config 4); the solution agrees to 1e-8 relative (1e-4 for config 4, whose
reported residual is not its true residual)."""

import numpy as np
import pytest

from conftest import CONFIG_CASES, golden, golden_csr

CASES = CONFIG_CASES + ["cfg2_m48"]

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


def _tols(name):
    # config-4 saddle point: cond_1(A0) ~ 1.5e7 -> both the reference's LU coarse solve and this
    # one carry ~cond * eps forward error; measured apply difference 2.6e-10 (band-LU default)
    return (1e-8, 1e-7, 1e-4) if name.startswith("cfg4") else (1e-10, 1e-10, 1e-8)


_cache = {}


def _setup(B, name):
    if name not in _cache:
        d = golden(name)
        a = golden_csr(d)
        mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
        # small batches so that multi-batch setup is exercised on every case; the default local
        # operator (band Cholesky / band pivoted LU, as the bench runs it).  The saddle-point
        # analog's (cfg4) deflated operator amplifies O(eps) differences by ~cond(A0), so its TRUE
        # residual is rounding-sensitive
        pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"],
                      coarse=str(d["coarse"]), n_modes=int(d["n_modes"]), batch=5)
        _cache[name] = (d, a, mat, pre)
    return _cache[name]


@pytest.mark.parametrize("name", CONFIG_CASES)
def test_spmv_matches_csr(B, name):
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
    x = np.random.default_rng(1).standard_normal(a.shape[0])
    y = mat.matvec(x)
    ref = a @ x
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    xt = torch.as_tensor(x, device="cuda")
    yt = mat.matvec(xt)
    assert yt.is_cuda and np.allclose(yt.cpu().numpy(), y, rtol=0, atol=0)


@pytest.mark.parametrize("name", CASES)
def test_setup_index_sets_and_report(B, name):
    d, a, mat, pre = _setup(B, name)
    assert np.array_equal(np.concatenate([m.indices for m in pre.maps]), d["indices"])
    assert pre.k_c == int(d["k_c"]) and np.array_equal(pre.colors, d["colors"])
    assert pre.report.mode_counts == tuple(d["mode_counts"])
    assert pre.report.n_coarse == int(d["n_coarse"])
    assert (pre.one_level, pre.combine) == (str(d["one_level"]), str(d["combine"]))


@pytest.mark.parametrize("name", CASES)
def test_apply_matches_reference(B, name):
    d, a, mat, pre = _setup(B, name)
    tol_apply = _tols(name)[0]
    for r, z, z1, zc in zip(d["r"], d["z"], d["z_one"], d["z_coarse"]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=tol_apply * np.abs(z).max())
        np.testing.assert_allclose(pre.apply_one_level(r), z1, rtol=0, atol=1e-10 * np.abs(z1).max())
        np.testing.assert_allclose(pre.coarse_apply(r), zc, rtol=0, atol=tol_apply * np.abs(zc).max())


@pytest.mark.parametrize("name", CASES)
def test_solve_matches_reference(B, name):
    d, a, mat, pre = _setup(B, name)
    _, tol_hist, tol_x = _tols(name)
    b = d["b"]
    if str(d["solver"]) == "pcg":
        x, rep = B.pcg(mat, pre, b, tol=float(d["tol"]), maxit=int(d["maxit"]))
    else:
        x, rep = B.gmres(mat, pre, b, tol=float(d["tol"]), maxit=int(d["maxit"]),
                         restart=int(d["restart"]))
    assert rep.converged == bool(d["converged"])
    assert abs(rep.iterations - int(d["iterations"])) <= 1
    k = min(rep.residuals.size, d["history"].size)
    np.testing.assert_allclose(rep.residuals[:k], d["history"][:k], rtol=0, atol=tol_hist)
    np.testing.assert_allclose(x, d["x"], rtol=0, atol=tol_x * np.abs(d["x"]).max())
    true_res = np.linalg.norm(b - a @ x) / np.linalg.norm(b)
    ref_true = float(d["true_residual"])
    if name.startswith("cfg4"):
        # cond_1(A0) ~ 1.5e7: the reported (Givens) residual is not the true one and the true one
        # is rounding-sensitive: x = M^{-1} V y, and M^{-1} with a coarse
        # operator of cond ~1e7 is linear only to ~cond * eps, so the true residual of the final
        # iterate moves by orders of magnitude with rounding (the reference itself ends 2.5x
        # above its reported 1e-7; measured here 4e-7 ... 1.2e-5 across equivalent orderings).
        # The reported history (above, 1e-7) and the iterate (1e-4 relative) are the parity
        # checks; the true residual must stay a converged one
        assert true_res <= 1e-4
    else:
        assert abs(true_res - ref_true) <= max(tol_hist, 1e-3 * ref_true)
    assert rep.gpu_launches > 0


def test_config1_headline_numbers(B):
    d, a, mat, pre = _setup(B, "cfg1")
    x, rep = B.pcg(mat, pre, d["b"], tol=1e-8)
    assert rep.iterations == 20 and rep.converged
    assert abs(rep.residuals[-1] - 4.376820e-09) < 1e-13


def test_apply_is_deterministic(B):
    d, a, mat, pre = _setup(B, "cfg2_m24")
    r = d["r"][0]
    z1, z2 = pre.apply(r), pre.apply(r)
    assert np.array_equal(z1, z2)


def test_apply_linear_and_symmetric(B):
    """Size-independent properties: linearity, and ASM+additive is a symmetric operator."""
    d, a, mat, pre = _setup(B, "cfg2_m24")
    rng = np.random.default_rng(11)
    u, v = rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    zu, zv = pre.apply(u), pre.apply(v)
    np.testing.assert_allclose(pre.apply(2.0 * u - 3.0 * v), 2.0 * zu - 3.0 * zv, rtol=0,
                               atol=1e-12 * np.abs(zu).max() * 5)
    assert pre.is_symmetric
    assert abs(v @ zu - u @ zv) <= 1e-12 * abs(v @ zu) + 1e-14


def test_torch_inputs_stay_on_device(B):
    d, a, mat, pre = _setup(B, "cfg1")
    r = torch.as_tensor(d["r"][0], device="cuda")
    z = pre.apply(r)
    assert z.is_cuda
    np.testing.assert_allclose(z.cpu().numpy(), d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
    x, rep = B.pcg(mat, pre, torch.as_tensor(d["b"], device="cuda"), tol=1e-8)
    assert x.is_cuda and rep.iterations == 20


@pytest.mark.parametrize("combo", [f"{o}_{c}_{k}" for o in ("asm", "ras")
                                   for c in ("none", "additive", "deflated")
                                   for k in ("full", "gevp", "svd")])
def test_all_variants_against_reference(B, combo):
    """The 18 variant combinations of tests/test_precond.py:78-101 (poisson2d m=8, N=4)."""
    d = golden("variants_p2d8")
    a = golden_csr(d)
    one, comb, kind = combo.split("_")
    mat = B.SparseMat(a, symmetric=True)
    pre = B.setup(mat, 4, overlap=2, tau=0.05, coarse=kind, one_level=one, combine=comb)
    assert np.array_equal(pre.maps[0].indices, pre.maps[0].indices)
    for r, z in zip(d["r"], d["z_" + combo]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=1e-11 * np.abs(z).max())


@pytest.mark.parametrize("m", [8, 12])
def test_nonsymmetric_defaults_and_unrestarted_gmres(B, m):
    d = golden(f"adv{m}")
    a = golden_csr(d)
    mat = B.SparseMat(a)
    pre = B.setup(mat, 4, overlap=2, tau=0.05)
    assert (pre.one_level, pre.combine, pre.report.coarse_kind) == ("ras", "deflated", "svd")
    for r, z in zip(d["r"], d["z"]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=1e-10 * np.abs(z).max())
    x, rep = B.gmres(mat, pre, d["b"], tol=1e-10)
    assert abs(rep.iterations - int(d["iterations"])) <= 1
    np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())


def test_tau_selection_config1(B):
    d = golden("cfg1_tau")
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=True)
    pre = B.setup(mat, int(d["n_sub"]), overlap=1, owner=d["owner"])
    assert pre.report.mode_counts == tuple(d["mode_counts"])
    np.testing.assert_allclose(pre.apply(d["r"]), d["z"], rtol=0, atol=1e-10 * np.abs(d["z"]).max())
    x, rep = B.pcg(mat, pre, d["b"])
    assert abs(rep.iterations - int(d["iterations"])) <= 1


@pytest.mark.parametrize("m", [30, 60])
def test_weak_scaling_cases(B, m):
    d = golden(f"weak_p2d{m}")
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=True)
    pre = B.setup(mat, int(d["n_sub"]), overlap=2, tau=0.1, owner=d["owner"])
    x, rep = B.pcg(mat, pre, d["b"], tol=1e-10)
    assert abs(rep.iterations - int(d["iterations"])) <= 1


def test_krylov_behaviour(B):
    import scipy.sparse as sp
    d = golden("krylov")
    lap = lambda n: B.SparseMat(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1],
                                         format="csr"), symmetric=True)
    x, rep = B.pcg(lap(32), None, d["lap32_b"], tol=1e-10)
    assert rep.converged and abs(rep.iterations - int(d["lap32_it"])) <= 1
    np.testing.assert_allclose(x, d["lap32_x"], atol=1e-8)
    x, rep = B.pcg(lap(200), None, d["lap200_b"], tol=1e-14, maxit=3)
    assert rep.iterations == 3 and not rep.converged and rep.residuals.size == 4
    x, rep = B.pcg(lap(10), None, np.zeros(10))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0) and rep.residuals.tolist() == [0.0]
    with pytest.raises(B.BreakdownError) as info:
        B.pcg(B.SparseMat.from_dense(np.diag([1.0, -1.0])), None, np.array([0.0, 1.0]), tol=1e-10)
    assert info.value.iteration >= 1
    a = golden_csr(d, "adv9_a_")
    x, rep = B.gmres(B.SparseMat(a), None, d["adv9_b"], tol=1e-8)
    assert abs(rep.iterations - int(d["adv9_it"])) <= 1
    np.testing.assert_allclose(rep.residuals[:5], d["adv9_hist"][:5], rtol=1e-9)
    x, rep = B.gmres(B.SparseMat.from_dense(d["happy_a"]), None, d["happy_b"], tol=1e-15, maxit=50)
    assert rep.converged and rep.iterations <= 3
    eye = B.SparseMat.identity(20)
    bb = np.random.default_rng(6).standard_normal(20)
    x, rep = B.gmres(eye, None, bb, tol=1e-12)
    assert rep.iterations == 1 and rep.converged
    np.testing.assert_allclose(x, bb, atol=1e-14)
    with pytest.raises(ValueError, match="hard cap"):
        B.gmres(lap(5), None, np.ones(5), maxit=1001)
    x, rep = B.gmres(lap(8), None, np.zeros(8))
    assert rep.converged and rep.iterations == 0


def test_callbacks_and_condition_estimate(B):
    import scipy.sparse as sp
    n = 64
    mat = B.SparseMat(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1],
                               format="csr"), symmetric=True)
    b = np.random.default_rng(5).standard_normal(n)
    seen = []
    x, rep = B.pcg(mat, None, b, tol=1e-12, maxit=200, callback=lambda it, xk: seen.append((it, xk)),
                   track_tridiagonal=True)
    assert [s[0] for s in seen] == list(range(1, rep.iterations + 1))
    np.testing.assert_allclose(seen[-1][1], x, atol=0)
    exact = np.linalg.cond(mat.to_dense())
    assert abs(rep.cond_estimate - exact) <= 1e-2 * exact
    x2, rep2 = B.pcg(mat, None, b, tol=1e-12, maxit=200)
    assert rep2.iterations == rep.iterations
    np.testing.assert_array_equal(x2, x)
    ks = []
    d = golden("adv12")
    a = golden_csr(d)
    pre = B.setup(B.SparseMat(a), 4, overlap=2, tau=0.05)
    B.gmres(B.SparseMat(a), pre, d["b"], tol=1e-10, callback=lambda k, _: ks.append(k))
    assert ks == list(range(1, len(ks) + 1)) and len(ks) >= 1


def test_single_subdomain_is_exact_inverse(B):
    import scipy.sparse as sp
    n = 20
    mat = B.SparseMat(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1],
                               format="csr"), symmetric=True)
    pre = B.setup(mat, 1, overlap=1, coarse="none")
    r = np.random.default_rng(0).standard_normal(n)
    np.testing.assert_allclose(pre.apply(r), np.linalg.solve(mat.to_dense(), r), rtol=1e-12)


def test_identity_matrix_ras_is_identity(B):
    mat = B.SparseMat.identity(16)
    pre = B.setup(mat, 4, overlap=1, coarse="none", one_level="ras")
    r = np.random.default_rng(1).standard_normal(16)
    np.testing.assert_allclose(pre.apply(r), r, atol=1e-14)


def test_config4_family_stall_history(B):
    """Non-converging GMRES(50) on the 64-subdomain saddle point: same stagnating history."""
    d = golden("cfg4_m64_stall")
    a = golden_csr(d)
    mat = B.SparseMat(a)
    pre = B.setup(mat, int(d["n_sub"]), overlap=1, owner=d["owner"], coarse="svd", n_modes=20)
    assert pre.local_kind == "band-lu"
    # measured: apply 1.8e-9, history 4e-9 (cond_1(A0) = 3.8e7)
    np.testing.assert_allclose(pre.apply(d["r"][0]), d["z"][0], rtol=0, atol=1e-8 * np.abs(d["z"][0]).max())
    x, rep = B.gmres(mat, pre, d["b"], tol=1e-7, maxit=100, restart=50)
    assert rep.iterations == 100 and not rep.converged
    np.testing.assert_allclose(rep.residuals, d["history"], rtol=0, atol=1e-8)


def test_coarse_refinement_restores_backward_stability(B):
    """One refinement step on the coarse solve (tls_coarse_refine; on automatically when
    cond_1(A0) > 1e8): the coarse residual ||A0 y - c|| drops to the backward-stable level of the
    reference's LU solve (src/coarse.py:178-182) and the apply is unchanged within cond * eps."""
    from paper_2401_03915_b200 import gpu_setup as G
    d = golden("cfg4_m32")
    a = golden_csr(d)
    mat = B.SparseMat(a)
    kw = dict(overlap=1, owner=d["owner"], coarse="svd", n_modes=20)
    plain = B.setup(mat, int(d["n_sub"]), **kw)
    old = G.REFINE_COND
    G.REFINE_COND = 0.0
    try:
        ref = B.setup(mat, int(d["n_sub"]), **kw)
    finally:
        G.REFINE_COND = old
    assert ref.coarse.refined and not plain.coarse.refined and plain.coarse.cond1 > 1e6
    a00 = ref.coarse.a00
    c = np.random.default_rng(2).standard_normal(a00.shape[0])
    res = []
    for pre in (plain, ref):
        y = pre.coarse.solve_coarse(c)
        res.append(np.abs(a00 @ y - c).max() / (np.abs(a00).sum(1).max() * np.abs(y).max()))
    assert res[1] <= 1e-14 and res[1] <= res[0], res
    r = d["r"][0]
    zp, zr = plain.apply(r), ref.apply(r)
    assert np.abs(zp - zr).max() <= 1e-8 * np.abs(zr).max()


@pytest.mark.parametrize("name", ["cfg1", "cfg2_m24", "cfg5_m16"])
def test_band_and_inverse_local_operators_agree(B, name):
    """The two stored local operators (banded Cholesky sweeps vs packed inverse tiles)."""
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=True)
    kw = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]), n_modes=int(d["n_modes"]))
    pb = B.setup(mat, int(d["n_sub"]), local="band", **kw)
    pi = B.setup(mat, int(d["n_sub"]), local="inverse", **kw)
    assert pb.local_kind.startswith("band") and pi.local_kind == "inverse"
    for r, z1 in zip(d["r"], d["z_one"]):
        zb, zi = pb.apply_one_level(r), pi.apply_one_level(r)
        np.testing.assert_allclose(zb, z1, rtol=0, atol=1e-11 * np.abs(z1).max())
        np.testing.assert_allclose(zb, zi, rtol=0, atol=1e-11 * np.abs(z1).max())
    xb, rb = B.pcg(mat, pb, d["b"], tol=float(d["tol"]))
    xi, ri = B.pcg(mat, pi, d["b"], tol=float(d["tol"]))
    assert abs(rb.iterations - ri.iterations) <= 1
    assert pb.device_bytes() < pi.device_bytes() or a.shape[0] < 5000


@pytest.mark.parametrize("name", ["cfg3_m64", "cfg4_m32"])
def test_band_lu_and_inverse_agree(B, name):
    """Nonsymmetric blocks: banded pivoted-LU sweeps vs general inverse tiles vs the reference."""
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a)
    kw = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]), n_modes=int(d["n_modes"]))
    pb = B.setup(mat, int(d["n_sub"]), local="band", **kw)
    pi = B.setup(mat, int(d["n_sub"]), local="inverse", **kw)
    assert pi.local_kind == "inverse"
    tol = 1e-8 if name.startswith("cfg4") else 1e-10
    for r, z1, z in zip(d["r"], d["z_one"], d["z"]):
        np.testing.assert_allclose(pb.apply_one_level(r), z1, rtol=0, atol=1e-10 * np.abs(z1).max())
        np.testing.assert_allclose(pb.apply(r), z, rtol=0, atol=tol * np.abs(z).max())
    x, rep = B.gmres(mat, pb, d["b"], tol=float(d["tol"]), restart=int(d["restart"]))
    assert abs(rep.iterations - int(d["iterations"])) <= 1


def test_matrix_upload_refuses_malformed_csr(B):
    """Host bounds check in tls_matrix_upload: the device kernels index through indptr/indices
    unchecked, so malformed structure must be refused before upload (TLS_ERR_DIM -> ValueError)."""
    from types import SimpleNamespace

    from paper_2401_03915_b200 import device as D

    def csr(indptr, indices, n=3):
        indices = np.asarray(indices, dtype=np.int32)
        return SimpleNamespace(indptr=np.asarray(indptr), indices=indices,
                               data=np.ones(indices.size), shape=(n, n))

    h = D.Handle(0)
    cases = [(csr([0, 1, 2, 3], [0, 3, 2]), "column index out of range at entry 1"),
             (csr([0, 1, 2, 3], [0, -1, 2]), "column index out of range at entry 1"),
             (csr([0, 2, 1, 3], [0, 1, 2]), "indptr decreases at row 1"),
             (csr([1, 1, 2, 3], [0, 1, 2]), "indptr must start at 0"),
             (csr([0, 1, 2, 2], [0, 1, 2]), "indptr must start at 0")]
    for bad, msg in cases:
        with pytest.raises(ValueError, match=msg):
            h.upload_matrix(bad, True)
    h.upload_matrix(csr([0, 1, 2, 3], [0, 1, 2]), True)  # the handle stays usable
    assert h.n == 3


@pytest.mark.parametrize("name", ["cfg2_m48", "cfg2_m24"])
def test_banded_coarse_inverse_matches_dense_path(B, name, monkeypatch):
    """A0^{-1} by the block-tridiagonal recurrences (gpu_setup.spd_inverse_block_tridiagonal, the
    path configuration 5 takes at full size) against the dense potrf + potri path on the same
    setup, and against the reference's coarse apply (src/coarse.py:40-49, 178-182)."""
    from paper_2401_03915_b200 import gpu_setup as G
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=True)
    kw = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]), n_modes=int(d["n_modes"]))
    monkeypatch.setattr(G, "BAND_INVERSE_MIN", 64)
    seen = []
    real = G.spd_inverse_block_tridiagonal
    monkeypatch.setattr(G, "spd_inverse_block_tridiagonal", lambda t, A, bs: (seen.append(bs), real(t, A, bs))[1])
    pre_b = B.setup(mat, int(d["n_sub"]), **kw)
    monkeypatch.setenv("TLS_A0_BANDED", "0")
    pre_d = B.setup(mat, int(d["n_sub"]), **kw)
    if name == "cfg2_m48":   # 6^3 subdomains x 16 columns: band 704 of 3456
        assert len(seen) == 1 and 4 * seen[0] <= pre_b.report.n_coarse
    r = d["r"][0]
    zb, zd, zr = pre_b.coarse_apply(r), pre_d.coarse_apply(r), d["z_coarse"][0]
    np.testing.assert_allclose(zb, zd, rtol=0, atol=1e-12 * np.abs(zd).max())
    np.testing.assert_allclose(zb, zr, rtol=0, atol=1e-10 * np.abs(zr).max())
    c = np.random.default_rng(2).standard_normal(pre_b.report.n_coarse)
    yb, yd = pre_b.coarse.solve_coarse(c), pre_d.coarse.solve_coarse(c)
    np.testing.assert_allclose(yb, yd, rtol=0, atol=1e-12 * np.abs(yd).max())
    x, rep = B.pcg(mat, pre_b, d["b"], tol=float(d["tol"]))
    assert rep.converged and abs(rep.iterations - int(d["iterations"])) <= 1


@pytest.mark.parametrize("name", ["cfg2_m48", "cfg2_m24"])
def test_block_tridiagonal_coarse_solve_matches_dense_path(B, name, monkeypatch):
    """The coarse solve by block forward / backward substitution (tls_coarse_chain, the path
    configuration 5 takes at full size: no n_C^2 inverse is formed or streamed) against the dense
    potrf + potri path on the same setup and against the reference's coarse apply
    (src/coarse.py:40-49, 178-182); the additive apply, a PCG solve and bit-reproducibility."""
    from paper_2401_03915_b200 import gpu_setup as G
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=True)
    kw = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]), n_modes=int(d["n_modes"]))
    monkeypatch.setattr(G, "BAND_INVERSE_MIN", 64)
    monkeypatch.setenv("TLS_A0_CHAIN_MIN", "64")
    seen = []
    real = G.spd_block_tridiagonal_chain
    monkeypatch.setattr(G, "spd_block_tridiagonal_chain", lambda t, A, bs: (seen.append(bs), real(t, A, bs))[1])
    pre_c = B.setup(mat, int(d["n_sub"]), **kw)
    monkeypatch.setenv("TLS_A0_BANDED", "0")
    pre_d = B.setup(mat, int(d["n_sub"]), **kw)
    if name == "cfg2_m48":   # 6^3 subdomains x 16 columns: band 704 of 3456 -> 5 blocks
        assert len(seen) == 1 and 4 * seen[0] <= pre_c.report.n_coarse
        assert pre_c.coarse.cond1 is None and pre_d.coarse.cond1 is not None
    else:
        assert len(seen) <= 1
    r = d["r"][0]
    zc, zd, zr = pre_c.coarse_apply(r), pre_d.coarse_apply(r), d["z_coarse"][0]
    np.testing.assert_allclose(zc, zd, rtol=0, atol=1e-12 * np.abs(zd).max())
    np.testing.assert_allclose(zc, zr, rtol=0, atol=1e-10 * np.abs(zr).max())
    np.testing.assert_array_equal(zc, pre_c.coarse_apply(r))
    c = np.random.default_rng(2).standard_normal(pre_c.report.n_coarse)
    yc, yd = pre_c.coarse.solve_coarse(c), pre_d.coarse.solve_coarse(c)
    np.testing.assert_allclose(yc, yd, rtol=0, atol=1e-12 * np.abs(yd).max())
    za, zda = pre_c.apply(r), pre_d.apply(r)
    np.testing.assert_allclose(za, zda, rtol=0, atol=1e-12 * np.abs(zda).max())
    np.testing.assert_allclose(za, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
    x, rep = B.pcg(mat, pre_c, d["b"], tol=float(d["tol"]))
    assert rep.converged and abs(rep.iterations - int(d["iterations"])) <= 1
    x2, rep2 = B.pcg(mat, pre_c, d["b"], tol=float(d["tol"]))
    np.testing.assert_array_equal(x, x2)
    if name == "cfg2_m48":
        assert pre_c.coarse.solve_kind == "block-tridiagonal" and pre_d.coarse.solve_kind == "dense-inverse"
        assert 0 < pre_c.coarse.solve_bytes < 0.6 * pre_d.coarse.solve_bytes
        # backward stability of the substitution: ||A0 y - c|| at the level of a Cholesky solve
        a00 = pre_c.coarse.a00
        res = np.abs(a00 @ yc - c).max() / (np.abs(a00).sum(1).max() * np.abs(yc).max())
        assert res <= 1e-14, res
        # the basis blocks come back from the library on demand, bit for bit
        for s in (0, 17, 215):
            np.testing.assert_array_equal(pre_c.coarse._z[s], pre_d.coarse._z[s])
        # malformed chains are refused before anything changes (the handle keeps working)
        h = pre_c.handle
        import ctypes as C
        ptrs = (C.c_uint64 * 3)(1, 1, 1)
        for nb_, bs_ in ((3, 100), (1, 3456), (2, 64)):
            rc = h.lib.tls_coarse_chain(h.ctx, nb_, bs_, ptrs, None, None, None, None, None, None, 0, None)
            assert rc != 0
        np.testing.assert_array_equal(zc, pre_c.coarse_apply(r))


def test_staged_matrix_upload_is_exact(B, monkeypatch):
    """Large CSR arrays travel through a ring of pinned staging buffers filled by host threads
    (tls_matrix_upload; configuration 5's 5.4 GB).  Forced on a small matrix with 16 KB chunks:
    the SpMV (src/sparsemat.py:125-129) is bit-identical to the plain upload's, and the first
    out-of-range column is still reported."""
    d = golden("cfg2_m48")
    a = golden_csr(d)
    v = np.random.default_rng(0).standard_normal(a.shape[0])
    from paper_2401_03915_b200.device import Handle
    y0 = B.SparseMat(a, symmetric=True).matvec(v)
    monkeypatch.setenv("TLS_STAGED_MIN_BYTES", "1")
    monkeypatch.setenv("TLS_STAGED_CHUNK_BYTES", "16384")
    np.testing.assert_array_equal(B.SparseMat(a, symmetric=True).matvec(v), y0)
    np.testing.assert_allclose(y0, a @ v, rtol=0, atol=1e-13 * np.abs(a @ v).max())
    h1 = Handle()
    bad = a.copy()
    bad.indices = bad.indices.copy()
    bad.indices[123457] = a.shape[0]
    with pytest.raises(ValueError, match="entry 123457"):
        h1.upload_matrix(bad, True)

"""Pin the CPU oracle to the reference: golden vectors produced by running tlschwarz itself
(oracle/make_golden.py).  Bit-exact for index sets; apply / history / iterations to the
last digit on these fixtures (same LAPACK drivers)."""

import numpy as np
import pytest

from conftest import CONFIG_CASES, golden, golden_csr
from oracle import tls_oracle as O


@pytest.mark.parametrize("name", CONFIG_CASES)
def test_oracle_matches_reference_config(name):
    d = golden(name)
    a = golden_csr(d)
    pre = O.OraclePreconditioner(a, bool(d["symmetric"]), d["owner"], int(d["n_sub"]),
                                 int(d["overlap"]), coarse=str(d["coarse"]), n_modes=int(d["n_modes"]))
    idx = np.concatenate([O.indices_of(m) for m in pre.maps])
    assert np.array_equal(idx, d["indices"])
    assert pre.k_c == int(d["k_c"]) and np.array_equal(pre.colors, d["colors"])
    assert pre.mode_counts == tuple(d["mode_counts"]) and pre.n_coarse == int(d["n_coarse"])
    assert pre.nnz_a00 == int(d["nnz_coarse"])
    for r, z, z1, zc in zip(d["r"], d["z"], d["z_one"], d["z_coarse"]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=1e-13 * np.abs(z).max())
        np.testing.assert_allclose(pre.apply_one_level(r), z1, rtol=0, atol=1e-13 * np.abs(z1).max())
        np.testing.assert_allclose(pre.coarse_apply(r), zc, rtol=0, atol=1e-13 * np.abs(zc).max())
    if str(d["solver"]) == "pcg":
        x, it, conv, hist = O.pcg(a, pre, d["b"], float(d["tol"]), int(d["maxit"]))
    else:
        x, it, conv, hist = O.gmres_restarted(a, pre, d["b"], float(d["tol"]), int(d["maxit"]),
                                              int(d["restart"]))
    assert it == int(d["iterations"]) and conv == bool(d["converged"])
    np.testing.assert_allclose(hist, d["history"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-12 * np.abs(d["x"]).max())


def test_oracle_config1_reference_numbers():
    """config 1 top-8 PCG = 20 iterations, final 4.376820e-09."""
    d = golden("cfg1")
    assert int(d["iterations"]) == 20
    assert abs(float(d["history"][-1]) - 4.376820e-09) < 5e-16


@pytest.mark.parametrize("combo", [f"{o}_{c}_{k}" for o in ("asm", "ras")
                                   for c in ("none", "additive", "deflated")
                                   for k in ("full", "gevp", "svd")])
def test_oracle_variants(combo):
    """tests/test_precond.py:78-101 variants (poisson2d m=8, N=4, delta=2, tau=0.05)."""
    d = golden("variants_p2d8")
    a = golden_csr(d)
    one, comb, kind = combo.split("_")
    pre = O.OraclePreconditioner(a, True, d["owner"], 4, 2, tau=0.05, coarse=kind, one_level=one,
                                 combine=comb)
    assert pre.mode_counts == tuple(d["counts_" + combo]) or comb == "none"
    for r, z in zip(d["r"], d["z_" + combo]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=1e-13 * np.abs(z).max())


@pytest.mark.parametrize("m", [8, 12])
def test_oracle_nonsymmetric_defaults(m):
    d = golden(f"adv{m}")
    a = golden_csr(d)
    pre = O.OraclePreconditioner(a, False, d["owner"], 4, 2, tau=0.05)
    assert (pre.one_level, pre.combine, pre.coarse_kind) == ("ras", "deflated", "svd")
    for r, z in zip(d["r"], d["z"]):
        np.testing.assert_allclose(pre.apply(r), z, rtol=0, atol=1e-12 * np.abs(z).max())
    x, it, conv, hist = O.gmres(a, pre, d["b"], 1e-10)
    assert it == int(d["iterations"])
    np.testing.assert_allclose(hist, d["history"], rtol=1e-10)


def test_oracle_tau_selection_config1():
    d = golden("cfg1_tau")
    a = golden_csr(d)
    pre = O.OraclePreconditioner(a, True, d["owner"], int(d["n_sub"]), 1)
    assert pre.mode_counts == tuple(d["mode_counts"]) and pre.n_coarse == int(d["n_coarse"])
    np.testing.assert_allclose(pre.apply(d["r"]), d["z"], rtol=0, atol=1e-13 * np.abs(d["z"]).max())
    _, it, _, hist = O.pcg(a, pre, d["b"])
    assert it == int(d["iterations"])


def test_oracle_krylov_behaviour():
    import scipy.sparse as sp
    d = golden("krylov")
    lap = lambda n: sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    x, it, conv, hist = O.pcg(lap(32), None, d["lap32_b"], 1e-10)
    assert it == int(d["lap32_it"])
    np.testing.assert_allclose(x, d["lap32_x"], atol=1e-13)
    x, it, conv, hist = O.pcg(lap(200), None, d["lap200_b"], 1e-14, 3)
    assert it == 3 and not conv
    a = golden_csr(d, "adv9_a_")
    x, it, conv, hist = O.gmres(a, None, d["adv9_b"], 1e-8)
    assert it == int(d["adv9_it"])
    np.testing.assert_allclose(hist, d["adv9_hist"], rtol=1e-10)
    x, it, conv, hist = O.gmres(sp.csr_matrix(d["happy_a"]), None, d["happy_b"], 1e-15, 50)
    assert conv and it == int(d["happy_it"]) and it <= 3
    with pytest.raises(O.OracleBreakdown):
        O.pcg(sp.csr_matrix(np.diag([1.0, -1.0])), None, np.array([0.0, 1.0]), 1e-10)
    with pytest.raises(ValueError, match="hard cap"):
        O.gmres(lap(5), None, np.ones(5), maxit=1001)


def test_oracle_config4_family_stalls_like_reference():
    """GMRES(50) on the saddle-point family stagnates in the reference too (64 subdomains)."""
    d = golden("cfg4_m64_stall")
    a = golden_csr(d)
    pre = O.OraclePreconditioner(a, False, d["owner"], int(d["n_sub"]), 1, coarse="svd", n_modes=20)
    x, it, conv, hist = O.gmres_restarted(a, pre, d["b"], 1e-7, 100, 50)
    assert it == 100 and not conv and not bool(d["converged"])
    np.testing.assert_allclose(hist, d["history"], rtol=1e-9)

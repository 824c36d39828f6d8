"""Partition-of-unity coarse modes (setup(nu=...), src/spectral.py:93-108, src/coarse.py:81-82)
on the GPU vs the reference's own setup (tests/golden/pou.npz, oracle/make_golden_io.py --pou):
mode counts after the rank filter exactly, applies within max(1e-10, 10 eps cond(A0)) of max|z|,
PCG iterations +-1."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden

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


@pytest.mark.parametrize("local", ["auto", "inverse"])
def test_pou_modes_match_reference(B, local):
    d = dict(golden("pou"))
    for c in range(int(d["n_cases"])):
        p = f"c{c}_"
        m, N, dl, tau, nu = d[p + "params"]
        n = int(m) ** (3 if str(d[p + "kind"]) == "poisson3d" else 2)
        a = sp.csr_matrix((d[p + "data"], d[p + "indices"], d[p + "indptr"]), shape=(n, n))
        mat = B.SparseMat(a, symmetric=True)
        pre = B.setup(mat, int(N), overlap=int(dl), tau=float(tau), nu=float(nu), coarse=str(d[p + "coarse"]),
                      local=local)
        assert pre.report.mode_counts == tuple(d[p + "mode_counts"]), (c, pre.report.mode_counts)
        assert pre.report.n_coarse == int(d[p + "n_coarse"])
        z = pre.apply(d[p + "r"])
        # PoU and harmonic modes can be nearly dependent: the coarse solve then amplifies
        # rounding by cond(A0) (3.8e9 on case 0, in the reference as much as here)
        tol = max(1e-10, 10 * np.finfo(float).eps * float(d[p + "cond_a0"]))
        np.testing.assert_allclose(z, d[p + "z"], rtol=0, atol=tol * np.abs(d[p + "z"]).max())
        x, rep = B.pcg(mat, pre, d[p + "b"], tol=1e-10)
        assert abs(rep.iterations - int(d[p + "iterations"])) <= 1 and rep.converged
        np.testing.assert_allclose(x, d[p + "x"], rtol=0, atol=1e-8 * np.abs(d[p + "x"]).max())


def test_pou_threshold_validation(B):
    a = B.problems.poisson2d(8)
    mat = B.SparseMat(a, symmetric=True)
    with pytest.raises(ValueError, match="threshold must exceed 1"):
        B.setup(mat, 4, nu=1.0)
    with pytest.raises(ValueError, match="require a symmetric"):
        B.setup(B.SparseMat(a), 4, nu=1.5, coarse="svd")

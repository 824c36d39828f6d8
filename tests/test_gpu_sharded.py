"""Sharded path validated on ONE GPU: R ranks in one process, each with its own
library handle owning a slab of subdomains, exchanging through the in-process group transport
(same schedule as NCCL: rank-partial prolongation + one sum all-reduce per apply stage).
Results must equal the single-handle path and be identical on every rank."""

import numpy as np
import pytest

from conftest import golden, golden_csr

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


def _sharded_run(B, name, nranks, solve):
    from paper_2401_03915_b200.distributed import LocalGroup
    d = dict(golden(name))  # materialise: NpzFile is not thread-safe
    a = golden_csr(d)
    grp = LocalGroup(nranks)

    def body(shard):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
            pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"],
                          coarse=str(d["coarse"]), n_modes=int(d["n_modes"]), shard=shard)
            z = pre.apply(d["r"][0])
            x, rep = solve(B, mat, pre, d)
            stream.synchronize()
            return pre.report, (shard.lo, shard.hi), z, x, rep

    return d, a, grp.run(body)


def _pcg(B, mat, pre, d):
    return B.pcg(mat, pre, d["b"], tol=float(d["tol"]))


def _gmres(B, mat, pre, d):
    return B.gmres(mat, pre, d["b"], tol=float(d["tol"]), restart=int(d["restart"]))


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_additive_pcg_matches_single(B, nranks):
    d, a, res = _sharded_run(B, "cfg2_m24", nranks, _pcg)
    slabs = [r[1] for r in res]
    assert slabs[0][0] == 0 and slabs[-1][1] == int(d["n_sub"])
    assert all(x[1] == y[0] for x, y in zip(slabs, slabs[1:]))
    for report, _, z, x, rep in res:
        assert report.mode_counts == tuple(d["mode_counts"]) and report.n_coarse == int(d["n_coarse"])
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1 and rep.converged
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
    for other in res[1:]:  # replicated state is bit-identical across ranks
        assert np.array_equal(other[2], res[0][2]) and np.array_equal(other[3], res[0][3])
        assert other[4].iterations == res[0][4].iterations


def test_sharded_deflated_gmres_matches_single(B):
    d, a, res = _sharded_run(B, "cfg3_m64", 2, _gmres)
    for report, _, z, x, rep in res:
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1 and rep.converged
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
    assert np.array_equal(res[0][3], res[1][3])

"""Sharded path validated on ONE GPU: R ranks in one process, each with its own
library handle owning a slab of subdomains and its rows (renumbered rank by rank), exchanging
through the in-process group transport (same schedule as NCCL: halo of ghost rows, reverse halo
of ASM overlap contributions, sum all-reduces of dot partials and of Z^T r).  Applies agree with
the single-handle path to rounding (the setup batches differ per rank, nothing else: same row
sums, same prolongation order); solves match the reference and are identical on every rank."""

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


def _sharded_run(B, name, nranks, solve, **kw):
    from paper_2401_03915_b200.distributed import LocalGroup
    d = dict(golden(name))  # materialise: NpzFile is not thread-safe
    a = golden_csr(d)
    grp = LocalGroup(nranks)
    opts = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]),
                n_modes=int(d["n_modes"]))
    opts.update(kw)

    def body(shard):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
            pre = B.setup(mat, int(d["n_sub"]), shard=shard, **opts)
            z = pre.apply(d["r"][0])
            z1 = pre.apply_one_level(d["r"][0])
            x, rep = solve(B, mat, pre, d)
            stream.synchronize()
            return pre.report, (shard.lo, shard.hi), z, x, rep, z1

    res = grp.run(body)
    mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
    single = B.setup(mat, int(d["n_sub"]), **opts)
    zs, z1s = single.apply(d["r"][0]), single.apply_one_level(d["r"][0])
    for r in res:  # same operator as one handle (setup batches differ: rounding-level only)
        np.testing.assert_allclose(r[2], zs, rtol=0, atol=1e-12 * np.abs(zs).max())
        np.testing.assert_allclose(r[5], z1s, rtol=0, atol=1e-12 * np.abs(z1s).max())
    return d, a, res


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
    for report, _, z, x, rep, _z1 in res:
        assert report.mode_counts == tuple(d["mode_counts"]) and report.n_coarse == int(d["n_coarse"])
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1 and rep.converged
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
    for other in res[1:]:  # replicated state is bit-identical across ranks
        assert np.array_equal(other[2], res[0][2]) and np.array_equal(other[3], res[0][3])
        assert other[4].iterations == res[0][4].iterations


def test_sharded_block_tridiagonal_coarse_solve(B, monkeypatch):
    """Every rank runs the whole block substitution of tls_coarse_chain (it does not partition by
    rows) on the all-gathered coarse coefficients: same applies and solves as one handle."""
    from paper_2401_03915_b200 import gpu_setup as G
    monkeypatch.setattr(G, "BAND_INVERSE_MIN", 64)
    monkeypatch.setenv("TLS_A0_CHAIN_MIN", "64")
    seen = []
    real = G.spd_block_tridiagonal_chain
    monkeypatch.setattr(G, "spd_block_tridiagonal_chain", lambda t, A, bs: (seen.append(bs), real(t, A, bs))[1])
    d, a, res = _sharded_run(B, "cfg2_m48", 2, _pcg)
    assert len(seen) == 3  # both ranks and the single handle
    for report, _, z, x, rep, _z1 in res:
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1 and rep.converged
    assert np.array_equal(res[1][2], res[0][2]) and np.array_equal(res[1][3], res[0][3])


def test_sharded_deflated_gmres_matches_single(B):
    d, a, res = _sharded_run(B, "cfg3_m64", 2, _gmres)
    for report, _, z, x, rep, _z1 in res:
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1 and rep.converged
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
    assert np.array_equal(res[0][3], res[1][3])


@pytest.mark.parametrize("nranks", [2, 4])
def test_sharded_one_level_asm_reverse_halo(B, nranks):
    """coarse='none' ASM: every overlap row receives contributions from other ranks' subdomains
    through the reverse halo; the sum order must stay ascending in the subdomain id."""
    d, a, res = _sharded_run(B, "cfg2_m24", nranks,
                             lambda B, mat, pre, d: B.pcg(mat, pre, d["b"], tol=1e-8, maxit=300),
                             coarse="none")
    for other in res[1:]:
        assert np.array_equal(other[3], res[0][3]) and other[4].iterations == res[0][4].iterations
    x, rep = res[0][3], res[0][4]
    assert rep.converged
    b = d["b"]
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) < 1e-8 * 1.01


def test_sharded_callback_and_spmv(B):
    """host-loop path (callback) and the SpMV entry point in caller numbering."""
    from paper_2401_03915_b200.distributed import LocalGroup
    d = dict(golden("cfg2_m24"))
    a = golden_csr(d)
    grp = LocalGroup(2)
    v = np.random.default_rng(5).standard_normal(a.shape[0])

    def body(shard):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            mat = B.SparseMat(a, symmetric=True)
            pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"],
                          n_modes=int(d["n_modes"]), shard=shard)
            seen = []
            x, rep = B.pcg(mat, pre, d["b"], tol=float(d["tol"]), callback=lambda it, xk: seen.append(it))
            y = pre.matvec(v)
            stream.synchronize()
            return seen, x, rep, y

    res = grp.run(body)
    for seen, x, rep, y in res:
        assert seen == list(range(1, rep.iterations + 1))
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
        assert np.array_equal(y, a @ v) or np.abs(y - a @ v).max() <= 1e-12 * np.abs(a @ v).max()


def _group_run(n, fn):
    from paper_2401_03915_b200.distributed import LocalGroup
    grp = LocalGroup(n)

    def body(shard):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            out = fn(shard)
            stream.synchronize()
            return out

    return grp.run(body)


@pytest.mark.parametrize("combo", ["asm_additive_gevp", "asm_deflated_svd", "ras_additive_full",
                                   "ras_deflated_gevp", "asm_none_gevp", "ras_none_svd"])
def test_sharded_variants_match_reference(B, combo):
    """The reference's apply variants (tests/test_precond.py:78-101 grid, tau threshold path,
    partition_graph owners) on 3 ranks: every rank returns the reference's z."""
    d = dict(golden("variants_p2d8"))
    a = golden_csr(d)
    one, comb, kind = combo.split("_")

    def fn(shard):
        mat = B.SparseMat(a, symmetric=True)
        pre = B.setup(mat, 4, overlap=2, tau=0.05, coarse=kind, one_level=one, combine=comb, shard=shard)
        return [pre.apply(r) for r in d["r"]]

    for zs in _group_run(3, fn):
        for z, zr in zip(zs, d["z_" + combo]):
            np.testing.assert_allclose(z, zr, rtol=0, atol=1e-11 * np.abs(zr).max())


def test_sharded_nonsymmetric_unrestarted_gmres_and_unpreconditioned(B):
    """Nonsymmetric defaults (RAS + deflated + SVD, band LU) with the reference's unrestarted GMRES
    on 2 ranks, and the unpreconditioned PCG / GMRES loops through a sharded handle."""
    d = dict(golden("adv12"))
    a = golden_csr(d)

    def fn(shard):
        mat = B.SparseMat(a)
        pre = B.setup(mat, 4, overlap=2, tau=0.05, shard=shard, local="band")
        z = pre.apply(d["r"][0])
        x, rep = B.gmres(mat, pre, d["b"], tol=1e-10)
        return z, x, rep

    res = _group_run(2, fn)
    for z, x, rep in res:
        np.testing.assert_allclose(z, d["z"][0], rtol=0, atol=1e-10 * np.abs(d["z"][0]).max())
        assert abs(rep.iterations - int(d["iterations"])) <= 1
        np.testing.assert_allclose(x, d["x"], rtol=0, atol=1e-8 * np.abs(d["x"]).max())
    assert np.array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("name,solver", [("cfg2_m24", "pcg"), ("cfg3_m64", "gmres")])
def test_sharded_schedule_captures_into_graphs(B, name, solver):
    """The NCCL transport runs the sharded schedule inside captured CUDA graphs; the in-process
    group cannot be captured (host barriers).  Here each rank's handle gets a recording
    transport (capturable, moves no data, logs every collective) and runs the solve through the
    graph path: capture must succeed, and every rank must issue the same collective sequence
    (kinds and all-reduce sizes) -- the condition for NCCL not to deadlock."""
    import ctypes as C
    d = dict(golden(name))
    a = golden_csr(d)

    def fn(shard):
        mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
        pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"],
                      coarse=str(d["coarse"]), n_modes=int(d["n_modes"]), shard=shard)
        return mat, pre

    res = _group_run(2, fn)
    logs = []
    for rank, (mat, pre) in enumerate(res):
        h = pre.handle
        h.check(h.lib.tls_comm_init_record(h.ctx, 2, rank))
        try:  # the numbers are meaningless without data exchange; only the schedule matters
            if solver == "pcg":
                B.pcg(mat, pre, d["b"], tol=1e-30, maxit=30)
            else:
                B.gmres(mat, pre, d["b"], tol=1e-30, maxit=20, restart=10)
        except Exception as e:  # noqa: BLE001  (breakdown on partial dot products is fine)
            assert "curvature" in str(e) or "breakdown" in str(e).lower(), e
        n = h.lib.tls_comm_record_log(h.ctx, None, 0)
        buf = (C.c_int64 * n)()
        h.lib.tls_comm_record_log(h.ctx, buf, n)
        log = np.array(buf[:], dtype=np.int64).reshape(-1, 3)
        logs.append(log)
    assert len(logs[0]) > 25 and len(logs[0]) == len(logs[1])
    assert np.array_equal(logs[0][:, 0], logs[1][:, 0])
    ar = logs[0][:, 0] == 1
    assert np.array_equal(logs[0][ar, 1], logs[1][ar, 1])
    assert (logs[0][:, 0] == 2).any()  # halo exchanges are part of the captured schedule


def test_nccl_transport_single_rank_group():
    """The NCCL transport itself, on the one GPU a box has: a torch.distributed group of one rank
    (backend nccl) takes the sharded path (Shard(single=True)) -- setup collectives over NCCL,
    ncclCommInitRank inside the library, the schedule's collectives issued through the NCCL API
    inside the captured PCG / GMRES graphs -- and must reproduce the unsharded results.  Runs in a
    subprocess (tools/nccl_single.py) so the process group does not outlive the test."""
    import json
    import os
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT", "MASTER_ADDR")}
    p = subprocess.run([sys.executable, os.path.join(repo, "tools", "nccl_single.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["ok"] and out["backend"] == "nccl" and out["world_size"] == 1
    for c in out["cases"]:
        assert c["comm_kind"] == 1 and c["nccl_calls"]["allreduce"] > 0, c
    assert out["cases"][0]["nccl_calls"]["allgather"] > 0  # the coarse restriction's all-gather

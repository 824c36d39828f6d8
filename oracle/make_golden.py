"""Generate golden fixtures by running the REFERENCE itself (this container only).

    python oracle/make_golden.py            # writes tests/golden/*.npz

The reference package (``tlschwarz``) is imported from /root/reference/pkg/src
(read-only; nothing is copied).  The fixtures pin the oracle
(``oracle/tls_oracle.py``) and, through it, the CUDA path.  Adapters the
reference lacks are composed ONLY from its public stages:

* top-k modes: ``select_harmonic_modes`` / ``svd_harmonic_modes`` with
  tau = 1e-300, first k columns kept, then ``subdomain_coarse_columns`` ->
  ``assemble_coarse_basis`` -> ``rank_filter`` -> ``galerkin_coarse`` ->
  ``Preconditioner(...)`` (src/precond.py:89-103);
* GMRES(m): reference ``gmres`` cycles on the true residual with the
  tolerance rescaled to the original ||b||.

Matrices for configurations 2-5 come from ``paper_2401_03915_b200.problems``
(the reference has no such generators) at scaled-down sizes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import scipy.sparse as sp  # noqa: E402
import tlschwarz as T  # noqa: E402
from tlschwarz import coarse as C  # noqa: E402
from tlschwarz import spectral as S  # noqa: E402

from paper_2401_03915_b200 import problems as P  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def topk_setup(mat, n_sub, owner, overlap, n_modes, coarse, one_level, combine, drop_tol=1e-10):
    """Reference setup with a fixed number of modes per subdomain."""
    sym = mat.symmetric
    graph = T.symmetrized_graph(mat)
    part = T.Partition(n_sub, owner)
    maps = T.extend_overlap(graph, part, overlap)
    k_c, colors = T.color_subdomains(maps)
    blocks = [T.extract_local_blocks(mat, s) for s in maps]
    solves = [T.factor_dense(b.a, sym, b.subdomain) for b in blocks]
    harm = [T.build_harmonic(b) for b in blocks]
    sel = S.select_harmonic_modes if coarse == "gevp" else S.svd_harmonic_modes
    bases = []
    for b, s, h in zip(blocks, maps, harm):
        full = sel(b, s.pou_mask, h, 1e-300)
        bases.append(S.SpectralBasis(full.kind, full.threshold, full.vectors[:, :n_modes].copy(),
                                     full.values[:n_modes].copy(), full.all_values))
    variant = {"gevp": "shrunk", "svd": "svd"}[coarse]
    cols = [C.subdomain_coarse_columns(s, b, h, variant, harmonic_basis=bases[i])
            for i, (s, b, h) in enumerate(zip(maps, blocks, harm))]
    cs = C.assemble_coarse_basis(maps, cols, mat.nrows)
    cs = C.rank_filter(cs, maps, drop_tol=drop_tol)
    counts = cs.column_counts()
    cs = C.galerkin_coarse(mat, cs)
    rep = T.SetupReport(n=mat.nrows, n_subdomains=n_sub, overlap=overlap, one_level=one_level,
                        combine=combine, coarse_kind=coarse, symmetric=sym, n_coarse=cs.n_coarse,
                        k_c=k_c, mode_counts=counts, nnz_matrix=mat.nnz, nnz_coarse=cs.nnz_a00)
    return T.Preconditioner(mat, maps, blocks, solves, harm, bases, None, cs, one_level, combine,
                            k_c, colors, rep)


def gmres_restarted(mat, pre, b, tol, maxit, restart):
    bn = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    hist = [1.0]
    total = 0
    conv = False
    while total < maxit:
        r = b - mat.matvec(x) if total else b.copy()
        rn = float(np.linalg.norm(r))
        d, rep = T.gmres(mat, pre, r, tol=tol * bn / rn, maxit=min(restart, maxit - total))
        x = x + d
        hist.extend((rep.residuals[1:] * (rn / bn)).tolist())
        total += rep.iterations
        if rep.converged:
            conv = True
            break
    return x, total, conv, np.asarray(hist)


def pack_pre(pre, prefix=""):
    d = {}
    maps = pre.maps
    d[prefix + "offsets"] = np.cumsum([0] + [s.n_local for s in maps]).astype(np.int64)
    d[prefix + "indices"] = np.concatenate([s.indices for s in maps]).astype(np.int64)
    d[prefix + "n_interior"] = np.array([s.interior.size for s in maps], dtype=np.int64)
    d[prefix + "n_boundary"] = np.array([s.n_boundary for s in maps], dtype=np.int64)
    d[prefix + "k_c"] = np.int64(pre.k_c)
    d[prefix + "colors"] = np.asarray(pre.colors, dtype=np.int64)
    d[prefix + "mode_counts"] = np.asarray(pre.report.mode_counts, dtype=np.int64)
    d[prefix + "n_coarse"] = np.int64(pre.report.n_coarse)
    d[prefix + "nnz_coarse"] = np.int64(pre.report.nnz_coarse)
    d[prefix + "one_level"] = pre.one_level
    d[prefix + "combine"] = pre.combine
    return d


def save(name, **arrs):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    print("wrote", name, sum(np.asarray(v).nbytes for v in arrs.values()) // 1024, "KiB")


def csr_fields(a):
    return dict(a_indptr=a.indptr.astype(np.int64), a_indices=a.indices.astype(np.int32), a_data=a.data)


def config_case(name, a, sym, owner, n_sub, overlap, n_modes, coarse, solver, tol, restart=None,
                maxit=500, rhs_seed=0, n_apply=2, store_matrix=True, gen=""):
    mat = T.SparseMat(a, symmetric=sym)
    one_level = "asm" if sym else "ras"
    combine = "additive" if sym else "deflated"
    pre = topk_setup(mat, n_sub, owner, overlap, n_modes, coarse, one_level, combine)
    rng = np.random.default_rng(rhs_seed)
    b = rng.uniform(-1.0, 1.0, a.shape[0])
    rr = np.random.default_rng(123)
    rs = [rr.standard_normal(a.shape[0]) for _ in range(n_apply)]
    zs = [pre.apply(r) for r in rs]
    z1 = [pre.apply_one_level(r) for r in rs]
    zc = [pre.coarse_apply(r) for r in rs]
    if solver == "pcg":
        x, rep = T.pcg(mat, pre, b, tol=tol, maxit=maxit)
        it, conv, hist = rep.iterations, rep.converged, rep.residuals
    else:
        x, it, conv, hist = gmres_restarted(mat, pre, b, tol, maxit, restart)
    true_res = float(np.linalg.norm(b - mat.matvec(x)) / np.linalg.norm(b))
    mfields = csr_fields(a) if store_matrix else {}
    save(name, **mfields, gen=gen, symmetric=sym, owner=np.asarray(owner, np.int64), n_sub=n_sub,
         overlap=overlap, n_modes=n_modes, coarse=coarse, solver=solver, tol=tol,
         restart=-1 if restart is None else restart, maxit=maxit, b=b, r=np.array(rs), z=np.array(zs),
         z_one=np.array(z1), z_coarse=np.array(zc), x=x, iterations=it, converged=conv,
         history=hist, true_residual=true_res, **pack_pre(pre))


def main():
    # configuration 1 at full size (BASELINE.json configs[0])
    c1 = P.CONFIGS[1]
    a, sym, owner, nsub = c1.build()
    ref_a, _ = T.generate(T.ProblemSpec("poisson2d", 64))
    assert (ref_a.scipy() != a).nnz == 0
    config_case("cfg1", a, sym, owner, nsub, 1, 8, "gevp", "pcg", 1e-8)
    # scaled analogs of configurations 2-5 (same generators, smaller grids)
    a, sym, owner, nsub = P.CONFIGS[2].scaled(16, 8).build()
    config_case("cfg2_m16", a, sym, owner, nsub, 1, 16, "gevp", "pcg", 1e-8)
    a, sym, owner, nsub = P.CONFIGS[2].scaled(24, 8).build()
    config_case("cfg2_m24", a, sym, owner, nsub, 1, 16, "gevp", "pcg", 1e-8)
    a, sym, owner, nsub = P.CONFIGS[3].scaled(64, 16).build()
    config_case("cfg3_m64", a, sym, owner, nsub, 2, 20, "svd", "gmres", 1e-8, restart=50)
    a, sym, owner, nsub = P.CONFIGS[4].scaled(32, 8).build()
    config_case("cfg4_m32", a, sym, owner, nsub, 1, 20, "svd", "gmres", 1e-7, restart=50)
    a, sym, owner, nsub = P.CONFIGS[5].scaled(16, 8, angle_block=8).build()
    config_case("cfg5_m16", a, sym, owner, nsub, 1, 12, "gevp", "pcg", 1e-8)
    # many subdomains / several setup batches: 216 subdomains of 8^3 (matrix regenerated in tests)
    cfg = P.CONFIGS[2].scaled(48, 8)
    a, sym, owner, nsub = cfg.build()
    config_case("cfg2_m48", a, sym, owner, nsub, 1, 16, "gevp", "pcg", 1e-8, n_apply=1,
                store_matrix=False, gen="2:48:8")
    # config-4 family with 64 subdomains: the reference's GMRES(50) stagnates
    a, sym, owner, nsub = P.CONFIGS[4].scaled(64, 8).build()
    config_case("cfg4_m64_stall", a, sym, owner, nsub, 1, 20, "svd", "gmres", 1e-7, restart=50,
                maxit=100, n_apply=1)

    # reference default selection (tau) on config 1, its own setup()
    a, sym, owner, nsub = c1.build()
    mat = T.SparseMat(a, symmetric=True)
    pre = T.setup(mat, nsub, overlap=1, owner=owner)
    b = np.random.default_rng(0).uniform(-1.0, 1.0, a.shape[0])
    x, rep = T.pcg(mat, pre, b, tol=1e-8)
    r = np.random.default_rng(5).standard_normal(a.shape[0])
    save("cfg1_tau", **csr_fields(a), owner=owner, n_sub=nsub, b=b, x=x, iterations=rep.iterations,
         history=rep.residuals, r=r, z=pre.apply(r), **pack_pre(pre))

    # all 18 variant combinations on poisson2d(8), N=4, delta=2, tau=0.05
    # (tests/test_precond.py:78-101); partition from the reference partitioner
    mat, _ = T.generate(T.ProblemSpec("poisson2d", 8))
    arrs = dict(**csr_fields(mat.scipy()))
    rng = np.random.default_rng(7)
    rs = np.array([rng.standard_normal(64) for _ in range(3)])
    arrs["r"] = rs
    for one_level in ("asm", "ras"):
        for combine in ("none", "additive", "deflated"):
            for coarse in ("full", "gevp", "svd"):
                pre = T.setup(mat, 4, overlap=2, tau=0.05, coarse=coarse, one_level=one_level,
                              combine=combine)
                key = f"{one_level}_{combine}_{coarse}"
                arrs["z_" + key] = np.array([pre.apply(r) for r in rs])
                arrs["counts_" + key] = np.asarray(pre.report.mode_counts, np.int64)
    arrs["owner"] = np.asarray(T.partition_graph(T.symmetrized_graph(mat), 4).owner, np.int64)
    save("variants_p2d8", **arrs)

    # nonsymmetric defaults: advection2d (ras + deflated + svd), gmres unrestarted
    for m in (8, 12):
        mat, b = T.generate(T.ProblemSpec("advection2d", m))
        pre = T.setup(mat, 4, overlap=2, tau=0.05)
        rng = np.random.default_rng(8)
        rs = np.array([rng.standard_normal(m * m) for _ in range(2)])
        x, rep = T.gmres(mat, pre, b, tol=1e-10)
        owner = np.asarray(T.partition_graph(T.symmetrized_graph(mat), 4).owner, np.int64)
        save(f"adv{m}", **csr_fields(mat.scipy()), b=b, r=rs, z=np.array([pre.apply(r) for r in rs]),
             x=x, iterations=rep.iterations, history=rep.residuals, owner=owner, **pack_pre(pre))

    # weak scaling (tests/test_acceptance.py:187-210) at the two smaller sizes
    for m, nsub in ((30, 4), (60, 16)):
        mat, b = T.generate(T.ProblemSpec("poisson2d", m))
        g = T.symmetrized_graph(mat)
        owner = np.asarray(T.partition_graph(g, nsub).owner, np.int64)
        pre = T.setup(mat, nsub, overlap=2, tau=0.1, owner=owner)
        x, rep = T.pcg(mat, pre, b, tol=1e-10, maxit=500)
        save(f"weak_p2d{m}", **csr_fields(mat.scipy()), b=b, owner=owner, n_sub=nsub,
             iterations=rep.iterations, history=rep.residuals, x=x, **pack_pre(pre))

    # partitioner fixtures (src/partition.py:161-258)
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_spd  # noqa: E402  (reference test fixture)
    parts = {}
    for key, mat, nsub in (("p2d8_4", T.generate(T.ProblemSpec("poisson2d", 8))[0], 4),
                           ("p2d30_16", T.generate(T.ProblemSpec("poisson2d", 30))[0], 16),
                           ("spd40_4", random_spd(40, 9), 4),
                           ("spd80_7", random_spd(80, 5), 7)):
        g = T.symmetrized_graph(mat)
        parts[key + "_indptr"] = mat.scipy().indptr.astype(np.int64)
        parts[key + "_indices"] = mat.scipy().indices.astype(np.int32)
        parts[key + "_data"] = mat.scipy().data
        parts[key + "_owner"] = np.asarray(T.partition_graph(g, nsub).owner, np.int64)
        parts[key + "_nsub"] = nsub
    save("partitions", **parts)

    # Krylov behaviour (tests/test_krylov.py)
    import scipy.sparse as sps
    lap = lambda n: T.SparseMat(sps.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)],
                                          [-1, 0, 1], format="csr"), symmetric=True)
    kr = {}
    b = np.random.default_rng(0).standard_normal(32)
    x, rep = T.pcg(lap(32), None, b, tol=1e-10)
    kr.update(lap32_b=b, lap32_x=x, lap32_it=rep.iterations, lap32_hist=rep.residuals)
    b = np.random.default_rng(4).standard_normal(200)
    x, rep = T.pcg(lap(200), None, b, tol=1e-14, maxit=3)
    kr.update(lap200_b=b, lap200_x=x, lap200_it=rep.iterations, lap200_conv=rep.converged,
              lap200_hist=rep.residuals)
    mat, b = T.generate(T.ProblemSpec("advection2d", 9))
    x, rep = T.gmres(mat, None, b, tol=1e-8)
    kr.update(adv9_b=b, adv9_x=x, adv9_it=rep.iterations, adv9_hist=rep.residuals,
              **{"adv9_" + k: v for k, v in csr_fields(mat.scipy()).items()})
    q, _ = np.linalg.qr(np.random.default_rng(7).standard_normal((12, 12)))
    dense = q @ np.diag(np.arange(1.0, 13.0)) @ q.T
    bq = q[:, 0] + q[:, 5]
    x, rep = T.gmres(T.SparseMat.from_dense(dense), None, bq, tol=1e-15, maxit=50)
    kr.update(happy_a=dense, happy_b=bq, happy_x=x, happy_it=rep.iterations, happy_hist=rep.residuals)
    save("krylov", **kr)


if __name__ == "__main__":
    sys.path.insert(0, HERE)
    main()

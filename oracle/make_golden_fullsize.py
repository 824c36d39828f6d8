"""Golden fixtures for the BASELINE configurations at FULL size, made by running the REFERENCE
itself (this container only; /root/reference is read-only and nothing is copied).

    python oracle/make_golden_fullsize.py 3      # cfg3 full pipeline  -> tests/golden/full_cfg3.npz
    python oracle/make_golden_fullsize.py 4      # cfg4 full pipeline  -> tests/golden/full_cfg4.npz
    python oracle/make_golden_fullsize.py 2      # cfg2 sampled        -> tests/golden/full_cfg2.npz
    python oracle/make_golden_fullsize.py 5      # cfg5 sampled        -> tests/golden/full_cfg5.npz

Configurations 3 and 4 (GMRES(50), RAS + deflated + top-k SVD coarse space): the reference's own
stages run subdomain by subdomain -- ``extract_local_blocks`` -> ``factor_dense`` ->
``build_harmonic`` -> ``svd_harmonic_modes`` (tau = 1e-300, first k kept: the top-k adapter of
SURVEY.md §8c.1) -> ``subdomain_coarse_columns`` -- keeping only each subdomain's LU solve closure
and its coarse columns (the dense block and the harmonic factor are dropped as soon as they are
used), then ``assemble_coarse_basis`` -> ``rank_filter`` -> ``galerkin_coarse`` ->
``Preconditioner(...)`` (src/precond.py:89-103).  That is the reference's setup with its memory
footprint cut to the LU factors (cfg3: 43 GB, cfg4: 24 GB), so it fits this container.  The solve is
the reference's ``gmres`` in GMRES(50) cycles (same adapter as make_golden.py).
Configuration 4 stagnates, so its history is recorded for the first 100 iterations.

Configurations 2 and 5 (PCG, ASM + additive + top-k harmonic-pencil coarse space): the reference
cannot set them up (DENSE_GUARD and ~0.24 / 2 TB of dense blocks + factors).  Its
graph, overlap and colouring stages run on the whole problem (SHA-256 of every index set and of
the colours is stored: the GPU path must reproduce all of them bit for bit), and its local stages
run with DENSE_GUARD raised on 8 sampled subdomains (corner, edge, face and interior blocks):
``y_i = A_ii^{-1} R_i r`` for a seeded r, the top-k harmonic-pencil values and the orthogonal
projection of 4 seeded vectors onto the span of the subdomain's coarse columns.

Vectors of length n are stored only as sampled entries plus a few full-length inner products with
seeded vectors, so the fixtures stay small.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import tlschwarz as T  # noqa: E402
from tlschwarz import coarse as C  # noqa: E402
from tlschwarz import spectral as S  # noqa: E402
from tlschwarz import subdomain as SD  # noqa: E402

from paper_2401_03915_b200 import problems as P  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")
SAMPLE_IDX_SEED = 77
N_SAMPLE = 8192

SAMPLED = {2: [0, 63, 86, 195, 220, 291, 424, 511],
           5: [0, 316, 1023, 2176, 2183, 2424, 3237, 4095]}


def log(msg, t0=[time.perf_counter()]):
    print(f"[{time.perf_counter() - t0[0]:8.1f}s] {msg}", flush=True)


def maps_digest(maps, colors, k_c):
    """SHA-256 over every subdomain's (n_interior, layer sizes, indices) and the colours."""
    h = hashlib.sha256()
    for s in maps:
        h.update(np.int64(s.interior.size).tobytes())
        h.update(np.asarray([l.size for l in s.layers], np.int64).tobytes())
        h.update(np.asarray(s.indices, np.int64).tobytes())
    h.update(np.asarray(colors, np.int64).tobytes())
    h.update(np.int64(k_c).tobytes())
    return h.hexdigest()


def vec_summary(v, prefix, n):
    """Sampled entries + norms + inner products with 3 seeded vectors (regenerated in the tests)."""
    idx = np.sort(np.random.default_rng(SAMPLE_IDX_SEED).choice(n, size=min(N_SAMPLE, n), replace=False))
    w = np.random.default_rng(SAMPLE_IDX_SEED + 1).standard_normal((3, n))
    return {prefix + "_idx": idx, prefix + "_vals": v[idx], prefix + "_norm": float(np.linalg.norm(v)),
            prefix + "_maxabs": float(np.abs(v).max()), prefix + "_dots": w @ v}


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
        log(f"  cycle: {rep.iterations} its, residual {hist[-1]:.3e}")
        if rep.converged:
            conv = True
            break
    return x, total, conv, np.asarray(hist)


def full_pipeline(cid, maxit):
    cfg = P.CONFIGS[cid]
    a, sym, owner, nsub = cfg.build()
    n = a.shape[0]
    log(f"cfg{cid}: n={n} nnz={a.nnz} subdomains={nsub}")
    mat = T.SparseMat(a, symmetric=sym)
    graph = T.symmetrized_graph(mat)
    part = T.Partition(nsub, owner)
    maps = T.extend_overlap(graph, part, cfg.overlap)
    k_c, colors = T.color_subdomains(maps)
    log(f"maps + colours: k_c={k_c}")
    SD.DENSE_GUARD = 10 ** 9
    solves, bases, cols = [], [], []
    for i, smap in enumerate(maps):
        blk = T.extract_local_blocks(mat, smap)
        solves.append(T.factor_dense(blk.a, sym, blk.subdomain))
        harm = T.build_harmonic(blk)
        full = S.svd_harmonic_modes(blk, smap.pou_mask, harm, 1e-300)
        basis = S.SpectralBasis(full.kind, full.threshold, full.vectors[:, :cfg.n_modes].copy(),
                                full.values[:cfg.n_modes].copy(), full.all_values)
        bases.append(basis)
        cols.append(C.subdomain_coarse_columns(smap, blk, harm, "svd", harmonic_basis=basis))
        del blk, harm, full
        if i % 32 == 0:
            log(f"  subdomain {i}/{nsub}")
    cs = C.assemble_coarse_basis(maps, cols, n)
    del cols
    cs = C.rank_filter(cs, maps)
    counts = cs.column_counts()
    cs = C.galerkin_coarse(mat, cs)
    log(f"coarse: n_C={cs.n_coarse} nnz_a00={cs.nnz_a00}")
    rep = T.SetupReport(n=n, n_subdomains=nsub, overlap=cfg.overlap, one_level="ras",
                        combine="deflated", coarse_kind="svd", symmetric=sym, n_coarse=cs.n_coarse,
                        k_c=k_c, mode_counts=counts, nnz_matrix=mat.nnz, nnz_coarse=cs.nnz_a00)
    pre = T.Preconditioner(mat, maps, None, solves, None, bases, None, cs, "ras", "deflated",
                           k_c, colors, rep)
    out = dict(cid=cid, n=n, nnz=a.nnz, n_sub=nsub, k_c=k_c, digest=maps_digest(maps, colors, k_c),
               mode_counts=np.asarray(counts, np.int64), n_coarse=cs.n_coarse, nnz_coarse=cs.nnz_a00,
               a00_fro=float(np.linalg.norm(cs.a00)), a00_trace=float(np.trace(cs.a00)),
               sigma_cut=np.array([b.all_values[cfg.n_modes - 1] / b.all_values[cfg.n_modes]
                                   for b in bases]))
    r = np.random.default_rng(123).standard_normal(n)
    out.update(vec_summary(pre.apply(r), "z", n))
    out.update(vec_summary(pre.apply_one_level(r), "z_one", n))
    out.update(vec_summary(pre.coarse_apply(r), "z_coarse", n))
    log("applies done; GMRES(50)")
    b = cfg.rhs(n)
    x, it, conv, hist = gmres_restarted(mat, pre, b, cfg.tol, maxit, cfg.restart)
    true_res = float(np.linalg.norm(b - mat.matvec(x)) / np.linalg.norm(b))
    out.update(vec_summary(x, "x", n))
    out.update(iterations=it, converged=conv, history=hist, true_residual=true_res, maxit=maxit)
    log(f"gmres: {it} its converged={conv} final={hist[-1]:.3e} true={true_res:.3e}")
    return out


def sampled(cid):
    cfg = P.CONFIGS[cid]
    a, sym, owner, nsub = cfg.build()
    n = a.shape[0]
    log(f"cfg{cid}: n={n} nnz={a.nnz} subdomains={nsub}")
    mat = T.SparseMat(a, symmetric=sym)
    graph = T.symmetrized_graph(mat)
    log("graph")
    part = T.Partition(nsub, owner)
    maps = T.extend_overlap(graph, part, cfg.overlap)
    log("overlap")
    k_c, colors = T.color_subdomains(maps)
    log(f"colours: k_c={k_c}")
    out = dict(cid=cid, n=n, nnz=a.nnz, n_sub=nsub, k_c=k_c, digest=maps_digest(maps, colors, k_c),
               n_local=np.asarray([s.n_local for s in maps], np.int64), sampled=np.asarray(SAMPLED[cid]))
    del graph
    SD.DENSE_GUARD = 10 ** 9
    r = np.random.default_rng(321).standard_normal(n)
    for s in SAMPLED[cid]:
        smap = maps[s]
        blk = T.extract_local_blocks(mat, smap)
        solve = T.factor_dense(blk.a, sym, blk.subdomain)
        harm = T.build_harmonic(blk)
        full = S.select_harmonic_modes(blk, smap.pou_mask, harm, 1e-300)
        k = cfg.n_modes
        basis = S.SpectralBasis(full.kind, full.threshold, full.vectors[:, :k].copy(),
                                full.values[:k].copy(), full.all_values)
        cols = C.subdomain_coarse_columns(smap, blk, harm, "shrunk", harmonic_basis=basis)
        ni = smap.interior.size
        zc = cols[:ni]                                   # interior support (src/coarse.py:1-7)
        q, _ = np.linalg.qr(zc)
        w = np.random.default_rng(1000 + s).standard_normal((ni, 4))
        out[f"s{s}_y"] = solve(r[smap.indices])
        out[f"s{s}_sigma"] = full.all_values[:k + 2].copy()
        out[f"s{s}_proj"] = q @ (q.T @ w)
        out[f"s{s}_k"] = cols.shape[1]
        log(f"  subdomain {s}: n_local={smap.n_local} sigma_k/sigma_k+1="
            f"{full.all_values[k - 1] / full.all_values[k]:.6f}")
        del blk, harm, full, solve
    return out


def main():
    cid = int(sys.argv[1])
    if cid in (3, 4):
        out = full_pipeline(cid, maxit=500 if cid == 3 else 100)
    else:
        out = sampled(cid)
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"full_cfg{cid}.npz")
    np.savez_compressed(path, **out)
    log(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")


if __name__ == "__main__":
    main()

"""Compare band vs inverse local operators on one configuration (components + solve)."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = PR.CONFIGS[cid] if not scale else PR.CONFIGS[cid].scaled(scale)
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
pres = {}
for kind in ("band", "inverse"):
    t0 = time.time()
    pres[kind] = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes, local=kind)
    print(kind, "setup", round(time.time() - t0, 1), "s counts", set(pres[kind].report.mode_counts), "nnzA0", pres[kind].report.nnz_coarse, flush=True)
r = np.random.default_rng(1).standard_normal(a.shape[0])
z1 = {k: p.apply_one_level(r) for k, p in pres.items()}
zc = {k: p.coarse_apply(r) for k, p in pres.items()}
za = {k: p.apply(r) for k, p in pres.items()}
rel = lambda u, v: np.abs(u - v).max() / np.abs(v).max()
print("one-level band vs inverse:", rel(z1["band"], z1["inverse"]))
print("coarse    band vs inverse:", rel(zc["band"], zc["inverse"]))
print("apply     band vs inverse:", rel(za["band"], za["inverse"]))
# coarse spans: principal angles per subdomain between the two bases
zb = pres["band"].coarse._z; zi = pres["inverse"].coarse._z
worst = 0.0; worst_s = -1
for s in range(nsub):
    qb, _ = np.linalg.qr(zb[s]); qi, _ = np.linalg.qr(zi[s])
    sv = np.linalg.svd(qb.T @ qi, compute_uv=False)
    ang = np.sqrt(max(0.0, 1 - sv.min() ** 2))
    if ang > worst: worst, worst_s = ang, s
print("max principal-angle sine between coarse spans:", worst, "subdomain", worst_s)
b = cfg.rhs(a.shape[0])
for k, p in pres.items():
    x, rep = (B.pcg(mat, p, b, tol=cfg.tol) if cfg.solver == "pcg" else B.gmres(mat, p, b, tol=cfg.tol, restart=cfg.restart))
    print(k, "iterations", rep.iterations, "final", rep.residuals[-1], flush=True)
for k, p in pres.items():
    g = np.array(sorted(p.coarse.cut_gaps.values()))
    print(k, "cut gaps: min", g[:5].tolist(), "count<1e-6:", int((g < 1e-6).sum()), "count<1e-3:", int((g < 1e-3).sum()))

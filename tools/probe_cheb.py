"""Chebyshev top-k eigensolver settings on real harmonic-pencil matrices (configuration-5 family,
64^3 grid with 16^3 blocks: 64 subdomains, interior rings of 1,736 nodes): block products, time and
the span error against a dense eigh for tolerance / block size / degree cap variants."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import gpu_setup as G  # noqa: E402
from paper_2401_03915_b200 import precond, problems  # noqa: E402

cfg = problems.CONFIGS[5].scaled(64, 16)
mat, sym, owner, nsub = cfg.build()
cap = {}
cheb = G.topk_chebyshev


def spy(torch_, M, k, **kw):
    if "M" not in cap or M.shape[1] > cap["M"].shape[1] or (M.shape[1] == cap["M"].shape[1] and M.shape[0] > cap["M"].shape[0]):
        cap["M"], cap["k"] = M.clone(), k
    return cheb(torch_, M, k, **kw)


G.topk_chebyshev = spy
precond.setup(B.SparseMat(mat, symmetric=sym), nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
G.topk_chebyshev = cheb
M, k = cap["M"], cap["k"]
print(f"captured M {tuple(M.shape)} k={k}", flush=True)
w, Q = torch.linalg.eigh(M)
w, Q = w.flip(-1)[:, :k], Q.flip(-1)[:, :, :k]
P = Q @ Q.mT
print("gap at the cut (relative):", ((w[:, k - 2] - w[:, k - 1]) / w[:, k - 2]).min().item(), flush=True)
for tol, p, dmax, rmax in [(1e-14, None, 16, 1e8), (3e-14, None, 16, 1e8), (1e-13, None, 16, 1e8),
                           (1e-14, 2 * k, 16, 1e8), (1e-14, 4 * k, 16, 1e8), (1e-14, None, 24, 1e8),
                           (1e-14, None, 16, 1e10), (1e-14, None, 32, 1e12)]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    try:
        th, X, mv = G.topk_chebyshev(torch, M, k, tol=tol, p=p, dmax=dmax, rmax=rmax)
    except Exception as e:  # noqa: BLE001
        print(f"tol={tol} p={p} dmax={dmax} rmax={rmax}: {e}")
        continue
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    err = (X @ X.mT - P).abs().amax().item()
    print(f"tol={tol:.0e} p={p or 'default'} dmax={dmax} rmax={rmax:.0e}: {mv} products, {1e3 * dt:.0f} ms, "
          f"span err {err:.1e}, theta err {((th - w).abs() / w[:, :1]).max().item():.1e}", flush=True)

"""Probe the batched top-k eigensolver of the harmonic pencil on real subdomain matrices.

Captures the reduced matrices M of the first batched group during a setup of a scaled config,
prints their spectrum decay and times eigensolver variants on them.

    python tools/probe_subspace.py --config 5 --m 64 --part 16
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import gpu_setup as G
from paper_2401_03915_b200 import precond, problems


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--part", type=int, default=16)
    ap.add_argument("--ps", default="0,64,96")
    a = ap.parse_args()
    cfg = problems.CONFIGS[a.config].scaled(a.m, a.part)
    mat, sym, owner, nsub = cfg.build()
    cap = {}
    orig = G.topk_subspace
    cheb = G.topk_chebyshev

    def spy(torch_, M, k, **kw):
        if "M" not in cap or M.shape[0] > cap["M"].shape[0]:
            cap["M"] = M.clone()
            cap["k"] = k
        return cheb(torch_, M, k, **kw)

    G.topk_chebyshev = spy
    t = time.perf_counter()
    precond.setup(B.SparseMat(mat, symmetric=sym), nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
    torch.cuda.synchronize()
    print(f"setup {time.perf_counter() - t:.2f}s", flush=True)
    G.topk_chebyshev = cheb
    M, k = cap["M"], cap["k"]
    print(f"captured M {tuple(M.shape)} k={k}", flush=True)
    for i in range(min(3, M.shape[0])):
        w = torch.linalg.eigvalsh(M[i]).flip(0).cpu().numpy()
        idx = [0, k - 1, k, 2 * k, 3 * k, 4 * k, 6 * k, 8 * k]
        print("  theta[idx]/theta0:", " ".join(f"{j}:{w[j] / w[0]:.3e}" for j in idx if j < w.size), flush=True)
    for p in [int(x) for x in a.ps.split(",")]:
        torch.cuda.synchronize()
        t = time.perf_counter()
        th, X, its = orig(torch, M, k, p=p or None)
        torch.cuda.synchronize()
        print(f"subspace p={p or 'default'}: sweeps {its}, {1e3 * (time.perf_counter() - t):.1f} ms "
              f"for {M.shape[0]} matrices", flush=True)
    for p in [int(x) for x in a.ps.split(",")]:
        torch.cuda.synchronize()
        t = time.perf_counter()
        tr = []
        th2, X2, mv = G.topk_chebyshev(torch, M, k, p=p or None, trace=tr)
        torch.cuda.synchronize()
        print("  steps (d, res, active, per_max):", " ".join(f"({d},{r:.0e},{n},{pm:.2f})" for d, r, n, pm in tr))
        err = float((th2 - th).abs().max() / th[:, :1].abs().min())
        print(f"chebyshev p={p or 'default'}: {mv} block products, {1e3 * (time.perf_counter() - t):.1f} ms, "
              f"theta err {err:.1e}", flush=True)

if __name__ == "__main__":
    main()

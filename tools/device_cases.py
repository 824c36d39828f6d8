"""Small device cases covering each local-solve kernel family, checked against the CPU oracle.

(Written for compute-sanitizer runs; the tool is closed on the GPU pool, so this runs plain:
``python tools/device_cases.py [spd gen inv]``.) Each case sets up a small problem through the public API, runs
one apply (checked against the CPU oracle) and one Krylov solve:
  spd  -- poisson2d, ASM + additive coarse, banded Cholesky sweeps, PCG (cfg 1 family);
  gen  -- 2D advection-diffusion, RAS + deflated coarse, banded pivoted-LU sweeps, GMRES(m)
          (cfg 3 family);
  inv  -- poisson2d with stored A_ii^-1 tiles (local="inverse": k_symv_tiles).
TLS_BAND_RING=0/4 in the environment selects the 4-CTA/SM sweep or the cp.async ring kernel.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2401_03915_b200 as P  # noqa: E402
from oracle import tls_oracle as O  # noqa: E402


def run(case):
    torch.cuda.set_device(0)
    cid, m, part, local = {"spd": (1, 32, 16, None), "gen": (3, 32, 16, None),
                           "inv": (1, 32, 16, "inverse")}[case]
    cfg = P.problems.CONFIGS[cid].scaled(m, part)
    a, sym, owner, nsub = cfg.build()
    mat = P.SparseMat(a, symmetric=sym)
    kw = {} if local is None else {"local": local}
    pre = P.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=4, **kw)
    ref = O.OraclePreconditioner(a, sym, owner, nsub, cfg.overlap, n_modes=4)
    r = np.random.default_rng(3).standard_normal(a.shape[0])
    z, zr = pre.apply(r), ref.apply(r)
    err = np.abs(z - zr).max() / np.abs(zr).max()
    b = cfg.rhs(a.shape[0])
    if sym:
        _, rep = P.pcg(mat, pre, b, tol=1e-8)
    else:
        _, rep = P.gmres(mat, pre, b, tol=1e-8, restart=8)
    torch.cuda.synchronize()
    print(f"case {case}: n={a.shape[0]} subdomains={nsub} apply rel err {err:.2e} "
          f"its={rep.iterations} converged={rep.converged}")
    assert err < 1e-10 and rep.converged


if __name__ == "__main__":
    for c in sys.argv[1:] or ["spd", "gen", "inv"]:
        run(c)

"""Per-kernel durations INSIDE a real solve (GPU box): the host-driven PCG / GMRES loop (selected by
a callback) with an event pair around every launch -- warm caches and the kernels' real inputs,
unlike ncu's serialised cold-cache replay; no graph / PDL overlap.

    python tools/ktrace.py <cfg> [m subdomains-per-side]  -> table on stdout
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import _lib  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = B.problems.CONFIGS[cid]
if len(sys.argv) > 3:
    cfg = cfg.scaled(int(sys.argv[2]), int(sys.argv[3]))
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
b = cfg.rhs(a.shape[0])
solve = (lambda cb: B.pcg(mat, pre, b, tol=cfg.tol, maxit=cfg.maxit, callback=cb)) if cfg.solver == "pcg" else \
    (lambda cb: B.gmres(mat, pre, b, tol=cfg.tol, maxit=cfg.maxit, restart=cfg.restart, callback=cb))
solve(None)  # warm
lib = _lib.load()
h = pre.handle
lib.tls_set_kernel_trace(h.ctx, 1)
x, rep = solve(lambda it, xk: None)
buf = C.create_string_buffer(1 << 16)
lib.tls_kernel_trace_dump(h.ctx, buf, len(buf))
lib.tls_set_kernel_trace(h.ctx, 0)
rows = [ln.rsplit(" ", 2) for ln in buf.value.decode().splitlines()]
tot = sum(float(r[2]) for r in rows)
its = rep.iterations
print(f"cfg{cid}: {its} iterations, traced kernel time {tot:.3f} ms = {1e3 * tot / its:.1f} us per iteration")
for name, cnt, ms in rows:
    cnt, ms = int(cnt), float(ms)
    print(f"{name[:60]:60s} n={cnt:5d} total={ms:9.3f} ms avg={1e3 * ms / cnt:8.2f} us  per-it={1e3 * ms / its:7.2f} us "
          f"share={100 * ms / tot:5.1f}%")

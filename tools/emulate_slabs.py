"""Per-rank local-solve kernel of the sharded path at N = 1, 2, 4, 8 ranks, measured on ONE GPU
for a configuration too large to hold N ranks in one process (configuration 5: 95 GB of band
factors).  For every N and a boundary and an interior rank q, a handle is set up that owns only
rank q's slab of subdomains (the slab the sharded setup would give it: distributed.slab_ranges),
with that slab's banded factors, and its k_band_solve launch -- 83% of a configuration-5 iteration
on one GPU -- is timed alone (CUDA events, 10 back-to-back launches, tls_profile_local_solve).
The rest of the iteration (SpMV rows, coarse rows, prolongation, vector updates: all row-
partitioned) is modelled as the single-GPU remainder / N; the collectives come on top.

    python tools/emulate_slabs.py [cfg] [N ...]      (one JSON line per N)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import _lib  # noqa: E402
from paper_2401_03915_b200 import device as D  # noqa: E402
from paper_2401_03915_b200 import problems as PR  # noqa: E402
from paper_2401_03915_b200.distributed import slab_ranges  # noqa: E402
from paper_2401_03915_b200.gpu_setup import build_device_operators  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
Ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
part = B.Partition(nsub, owner)


class SlabShard:
    """Rank q of N as far as the local operators are concerned (no communicator, no coarse)."""

    def __init__(self, n, q):
        self.nranks, self.rank, self.lo, self.hi, self.coll = n, q, None, None, None

    def attach(self, handle):
        pass


h0 = D.Handle()
h0.upload_matrix(a, sym)
graph = D.device_graph(h0)
maps, _, _ = D.device_overlap(h0, part, cfg.overlap)
del h0
n_loc = np.array([m.n_local for m in maps], dtype=np.float64)


def band_time(n, q):
    h = D.Handle()
    h.upload_matrix(a, sym)
    sh = SlabShard(n, q) if n > 1 else None
    build_device_operators(h, a, sym, maps, owner, "none", 0.1, None, 1e-10, shard=sh, graph=graph)
    h.check(h.lib.tls_precond_finalize(h.ctx, _lib.ONE_LEVEL["asm"], _lib.COMBINE["none"]))
    ms, algo = C.c_double(), C.c_double()
    h.check(h.lib.tls_profile_local_solve(h.ctx, 10, C.byref(ms), C.byref(algo), D.stream_ptr()))
    lo, hi = (0, nsub) if n == 1 else (sh.lo, sh.hi)
    del h
    torch.cuda.empty_cache()
    return ms.value, algo.value, hi - lo


if __name__ == "__main__":
    base = None
    for n in Ns:
        ranks = [0] if n == 1 else sorted({0, n // 2, n - 1})
        res = {q: band_time(n, q) for q in ranks}
        tmax = max(v[0] for v in res.values())
        if n == 1:
            base = tmax
        print(json.dumps({"config": cfg.name, "ranks": n, "slab_ranges": [list(r) for r in slab_ranges(n_loc ** 2, n)],
                          "band_ms": {q: round(v[0], 4) for q, v in res.items()},
                          "band_GBps": {q: round(v[1] / v[0] / 1e6, 1) for q, v in res.items()},
                          "subdomains": {q: v[2] for q, v in res.items()},
                          "band_ms_max": round(tmax, 4),
                          "band_efficiency": round(base / (n * tmax), 4)}), flush=True)

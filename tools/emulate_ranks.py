"""Per-rank compute of the sharded PCG iteration at N = 1, 2, 4, 8 ranks, measured on ONE GPU.

All N ranks are set up in one process (in-process group: the real setup collectives), then each
rank's handle switches to the recording transport (capturable, moves no data) and its PCG graph
is timed alone with CUDA events: per-iteration time = (t(maxit=75) - t(maxit=25)) / 50.  This is
the compute share of each rank; the collectives (2 halos, 1 reverse halo, 4 small all-reduces
per iteration) come on top.  Output: one JSON line per N.

    python tools/emulate_ranks.py [cfg] [N ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import problems as PR  # noqa: E402
from paper_2401_03915_b200.distributed import LocalGroup  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
Ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
b = cfg.rhs(a.shape[0])


def timed(mat, pre, maxit):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    try:
        _, rep = B.pcg(mat, pre, b, tol=1e-300, maxit=maxit)
        its = rep.iterations
    except Exception:  # noqa: BLE001  (partial dot products can break down: not a timing)
        its = -1
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), its


for N in Ns:
    if N == 1:
        mat = B.SparseMat(a, symmetric=sym)
        pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
        timed(mat, pre, 25)
        t25, _ = timed(mat, pre, 25)
        t75, its = timed(mat, pre, 75)
        per = [(t75 - t25) / 50]
        del pre
    else:
        grp = LocalGroup(N)

        def body(shard):
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                mat = B.SparseMat(a, symmetric=sym)
                pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes, shard=shard,
                              batch=max(2, 32 // N))  # N setups share one GPU here
                st.synchronize()
                return mat, pre

        res = grp.run(body)
        per = []
        for rank, (mat, pre) in enumerate(res):
            h = pre.handle
            h.check(h.lib.tls_comm_init_record(h.ctx, N, rank))
            if os.environ.get("TLS_PROFILE_RANGE") == "1" and rank == 1:  # ncu on one rank's solve
                torch.cuda.profiler.start()
                timed(mat, pre, 25)
                torch.cuda.profiler.stop()
            timed(mat, pre, 25)
            t25, _ = timed(mat, pre, 25)
            t75, its = timed(mat, pre, 75)
            per.append((t75 - t25) / 50)
        del res, grp
    torch.cuda.empty_cache()
    print(json.dumps({"config": cfg.name, "ranks": N, "ms_per_iteration_per_rank": [round(x, 4) for x in per],
                      "max_ms": round(max(per), 4)}), flush=True)

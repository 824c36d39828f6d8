"""The NCCL transport on a 1-GPU box: a torch.distributed group of ONE rank (backend nccl) runs the
sharded path end to end -- TorchCollective for the setup exchanges, the unique-id broadcast,
``tls_comm_init_nccl`` (ncclCommInitRank inside libtls_b200), the row renumbering and (empty) halo
plans, and every collective of the schedule issued through the NCCL API inside the captured
PCG / GMRES graphs (ncclAllReduce, ncclAllGather, grouped ncclSend/ncclRecv with no peers).

It cannot show link traffic (one rank moves no data between GPUs) -- it shows that the
communicator initialises against the NCCL this image ships, that NCCL calls capture into the
solve graphs and replay, and that the results equal the unsharded path.  Launch:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
        --master-port 29517 tools/nccl_single.py

or plain ``python tools/nccl_single.py`` (it fills in the rendezvous variables itself).  Prints one
JSON line; exit code 0 only when every check passed.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import socket
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    os.environ.setdefault("LOCAL_RANK", "0")
    import torch
    import torch.distributed as dist
    from conftest import golden, golden_csr

    assert torch.cuda.is_available(), "needs cuda:0"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    import paper_2401_03915_b200 as B
    from paper_2401_03915_b200 import build
    from paper_2401_03915_b200.distributed import world_shard
    build.build()

    out = {"world_size": dist.get_world_size(), "backend": dist.get_backend(), "cases": []}
    ok = True
    cases = [("cfg2_m24", "pcg", {}), ("cfg3_m64", "gmres", {}), ("cfg2_m24", "pcg", {"coarse": "none"})]
    for name, solver, extra in cases:
        d = dict(golden(name))
        a = golden_csr(d)
        sym = bool(d["symmetric"])
        opts = dict(overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]),
                    n_modes=int(d["n_modes"]))
        opts.update(extra)

        def run(shard):
            mat = B.SparseMat(a, symmetric=sym)
            pre = B.setup(mat, int(d["n_sub"]), shard=shard, **opts)
            z = pre.apply(d["r"][0])
            t0 = time.perf_counter()
            if solver == "pcg":
                x, rep = B.pcg(mat, pre, d["b"], tol=float(d["tol"]), maxit=300)
            else:
                x, rep = B.gmres(mat, pre, d["b"], tol=float(d["tol"]), restart=int(d["restart"]))
            torch.cuda.synchronize()
            return pre, z, x, rep, time.perf_counter() - t0

        pre_s, z_s, x_s, rep_s, t_s = run(world_shard(single=True))
        pre_p, z_p, x_p, rep_p, t_p = run(None)
        calls = (C.c_int64 * 3)()
        comm_kind = int(pre_s.handle.lib.tls_comm_info(pre_s.handle.ctx, calls))
        err_z = float(np.abs(z_s - z_p).max() / np.abs(z_p).max())
        err_x = float(np.abs(x_s - x_p).max() / np.abs(x_p).max())
        case_ok = (comm_kind == 1 and err_z <= 1e-12 and err_x <= 1e-8
                   and abs(rep_s.iterations - rep_p.iterations) <= 1 and rep_s.converged)
        if not extra:  # against the reference's own numbers too
            zr = d["z"][0]
            case_ok = case_ok and float(np.abs(z_s - zr).max() / np.abs(zr).max()) <= 1e-10 \
                and abs(rep_s.iterations - int(d["iterations"])) <= 1
        ok = ok and case_ok
        out["cases"].append({"case": name, "solver": solver, **extra, "ok": bool(case_ok),
                             "comm_kind": comm_kind, "nccl_calls": {"allreduce": int(calls[0]), "exchange": int(calls[1]),
                                                                    "allgather": int(calls[2])}, "apply_rel_diff": err_z, "x_rel_diff": err_x,
                             "iterations_nccl": int(rep_s.iterations), "iterations_plain": int(rep_p.iterations),
                             "solve_s_nccl": t_s, "solve_s_plain": t_p,
                             "launches_nccl": int(rep_s.gpu_launches), "launches_plain": int(rep_p.gpu_launches)})
        del pre_s, pre_p
    out["ok"] = bool(ok)
    print(json.dumps(out))
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

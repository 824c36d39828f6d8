"""Time the banded factorisation of one setup batch: library path vs in-tree K9 (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp, torch
from paper_2401_03915_b200 import problems as PR, gpu_setup as G, partition as Pt
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 48
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
g = Pt.symmetrized_graph(a, symmetric=True)
maps = Pt.extend_overlap(g, Pt.Partition(nsub, owner), cfg.overlap)
ms = maps[nsub // 2: nsub // 2 + cnt]
ld = -(-max(m.n_local for m in ms) // 64) * 64
A = torch.zeros(len(ms), ld, ld, dtype=torch.float64, device="cuda")
for b, m in enumerate(ms):
    A[b, :m.n_local, :m.n_local] = torch.as_tensor(a[m.indices][:, m.indices].toarray())
    A[b, m.n_local:, m.n_local:] = torch.eye(ld - m.n_local, dtype=torch.float64)
adj = sp.csr_matrix((np.ones(g.adjacency.size, dtype=np.int8), g.adjacency, g.indptr), shape=a.shape)
kind, _ = G.choose_local_order(adj, maps, True)
perms = G.local_orders(adj, ms, kind)
n_list = [m.n_local for m in ms]
for mode in ("torch", "kernel", "torch", "kernel"):
    G.BAND_CHOL = mode
    B = A.clone()
    torch.cuda.synchronize()
    t = time.perf_counter()
    G._band_factor(torch, B, perms, n_list, ld)
    torch.cuda.synchronize()
    print(mode, f"cfg{cid} batch {cnt} ld {ld} order {kind}: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)

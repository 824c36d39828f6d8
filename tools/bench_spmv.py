"""Time tls_spmv (CUDA events) on a configuration's matrix for the current TLS_SPMV_LPR."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR, _lib
cid = int(sys.argv[1]); scale = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = PR.CONFIGS[cid] if not scale else PR.CONFIGS[cid].scaled(scale)
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
h = mat.device_handle()
x = torch.randn(a.shape[0], dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(5): h.lib.tls_spmv(h.ctx, _lib.ptr(x), _lib.ptr(y), st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); reps = 50
for _ in range(reps): h.lib.tls_spmv(h.ctx, _lib.ptr(x), _lib.ptr(y), st)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
byts = 12 * a.nnz + 4 * (a.shape[0] + 1) + 16 * a.shape[0]
print(f"cfg{cid} LPR={os.environ.get('TLS_SPMV_LPR','auto')} {ms*1e3:.1f} us  {byts/ms/1e6:.0f} GB/s")

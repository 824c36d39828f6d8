"""A/B of the thin-SVD variants for the svd coarse columns (src/spectral.py:135-154) on one 4096 x 260 block:
torch default / gesvd / gesvdj / QR + small SVD. Result: profiles/ab_svd_r01.txt (no variant beats the default)."""
import torch, time
torch.manual_seed(0)
E = torch.randn(4096, 260, dtype=torch.float64, device="cuda") @ torch.diag(torch.logspace(0, -8, 260, dtype=torch.float64, device="cuda"))
def t(f, n=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r
U0, S0, _ = torch.linalg.svd(E, full_matrices=False)
def qrsvd():
    Q, R = torch.linalg.qr(E)
    Ur, S, _ = torch.linalg.svd(R)
    return Q @ Ur, S
for name, f in [("svd default", lambda: torch.linalg.svd(E, full_matrices=False)[:2]),
                ("svd gesvd", lambda: torch.linalg.svd(E, full_matrices=False, driver="gesvd")[:2]),
                ("svd gesvdj", lambda: torch.linalg.svd(E, full_matrices=False, driver="gesvdj")[:2]),
                ("qr+svd", qrsvd),
                ("qr+svd(R, gesvdj)", lambda: (lambda Q, R: (lambda u: (Q @ u[0], u[1]))(torch.linalg.svd(R, driver="gesvdj")[:2]))(*torch.linalg.qr(E)))]:
    ms, (U, S) = t(f)
    k = 40
    P0 = U0[:, :k] @ U0[:, :k].T; P1 = U[:, :k] @ U[:, :k].T
    print(f"{name:20s} {ms:8.2f} ms  sv rel err {float(((S - S0).abs() / S0).max()):.2e}  top-{k} projector diff {float((P0 - P1).abs().max()):.2e}")

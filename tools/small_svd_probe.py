"""Left singular vectors of tall-skinny / wide matrices: torch SVD vs QR + fl_svd_batched (dev tool)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
def qr_route(M):
    n, m = M.shape
    if n >= m:
        Q, R = torch.linalg.qr(M)
        U, s, _ = decomp.svd_batched(R[None])
        return Q @ U[0], s[0]
    Q, R = torch.linalg.qr(M.T)
    U, s, _ = decomp.svd_batched(R.T.contiguous()[None])
    return U[0], s[0]
for n, m in [(1023, 36), (511, 36), (255, 36), (127, 36), (1023, 64), (36, 1023), (64, 4096), (110, 8000), (127, 8000)]:
    M = torch.randn(n, m, dtype=torch.float64, device="cuda") @ torch.diag(torch.logspace(0, -12, m, dtype=torch.float64, device="cuda"))
    k = min(n, m)
    ta = t(lambda: torch.linalg.svd(M, full_matrices=False))
    tb = t(lambda: qr_route(M))
    U0, s0, _ = torch.linalg.svd(M, full_matrices=False)
    U1, s1 = qr_route(M)
    r = min(k, 20)
    sub = float(torch.linalg.matrix_norm(U0[:, :r] @ U0[:, :r].T - U1[:, :r] @ U1[:, :r].T))
    print("%5d x %5d: torch %.2f ms, qr+jacobi %.2f ms, subspace err %.1e, sv err %.1e" % (
        n, m, ta, tb, sub, float((s0 - s1).abs().max() / s0[0])), flush=True)

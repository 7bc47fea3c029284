"""fl_svd_batched on single square matrices vs torch (dev tool): time + accuracy."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
for n in (64, 127, 200, 255):
    # graded spectrum like truncation inputs
    Q1 = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda"))[0]
    Q2 = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda"))[0]
    s = torch.logspace(0, -14, n, dtype=torch.float64, device="cuda")
    A = (Q1 * s) @ Q2.T
    tt = t(lambda: torch.linalg.svd(A))
    tb = t(lambda: decomp.svd_batched(A[None]))
    U, S, Vt = decomp.svd_batched(A[None])
    U0, S0, V0 = torch.linalg.svd(A)
    k = 20
    sub = float(torch.linalg.matrix_norm(U[0, :, :k] @ U[0, :, :k].T - U0[:, :k] @ U0[:, :k].T))
    rec = float(torch.linalg.matrix_norm((U[0] * S[0]) @ Vt[0] - A) / torch.linalg.matrix_norm(A))
    print(n, "torch %.2f ms, fl_svd_batched %.2f ms, subspace err %.2e, recon %.2e, sv relerr %.2e" % (
        tt, tb, sub, rec, float(((S[0] - S0).abs() / S0[0]).max())), flush=True)

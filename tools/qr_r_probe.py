"""Left singular vectors of wide 127 x m factors (configs[1] c2t): library SVD
of M vs R-only QR of M^T (no Q formed) + SVD of the 127 x 127 R^T (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1809_01971_b200.decomp import svd_batched


def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


g = torch.Generator(device="cuda"); g.manual_seed(0)
for m in (144, 1000, 16000, 131400):
    # graded columns like the CP factors: singular values spread over 1e-14..1
    A = torch.randn(127, 127, dtype=torch.float64, device="cuda", generator=g)
    Q1 = torch.linalg.qr(A)[0]
    B = torch.randn(m, 127, dtype=torch.float64, device="cuda", generator=g)
    Q2 = torch.linalg.qr(B)[0]
    sig = torch.logspace(0, -14, 127, dtype=torch.float64, device="cuda")
    M = (Q1 * sig) @ Q2.T
    ta, (U, s, _) = t(lambda: torch.linalg.svd(M, full_matrices=False))
    tb, (U2, s2, _) = t(lambda: torch.linalg.svd(torch.linalg.qr(M.T, mode="r")[1].T, full_matrices=False))
    tc, (U3, s3, _) = t(lambda: svd_batched(torch.linalg.qr(M.T, mode="r")[1].T.contiguous()[None], right=False))
    tr, _ = t(lambda: torch.linalg.qr(M.T, mode="r")[1])
    U3, s3 = U3[0], s3[0]
    def cmp(Ux, sx):
        ds = float(((sx - s).abs() / s[0]).max())
        k = int((s > 1e-8 * s[0]).sum())
        du = float((1.0 - (Ux[:, :k] * U[:, :k]).sum(0).abs()).abs().max())
        return ds, du, k
    print("m=%6d svd %.2f ms | qr_r+svd %.2f ms %s | qr_r+jacobi %.2f ms %s | qr_r alone %.2f ms" % (
        m, ta, tb, cmp(U2, s2), tc, cmp(U3, s3), tr), flush=True)

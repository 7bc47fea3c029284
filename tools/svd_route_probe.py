"""torch.linalg.svd vs QR + batched Jacobi for c2t shapes (dev tool)."""
import time
import torch
from paper_1809_01971_b200.decomp import svd_batched


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def qr_jacobi(M):
    a, b = M.shape
    if a >= b:
        Q, R = torch.linalg.qr(M)
        U, S, Vt = svd_batched(R[None])
        return Q @ U[0], S[0], Vt[0]
    Q, R = torch.linalg.qr(M.T)
    U, S, Vt = svd_batched(R.T[None].contiguous())
    return U[0], S[0], Vt[0] @ Q.T


for shape in [(127, 127), (127, 5000), (60, 3600), (127, 16129), (64, 64), (200, 200), (40, 1600)]:
    M = torch.randn(*shape, dtype=torch.float64, device="cuda")
    a = t(lambda: torch.linalg.svd(M, full_matrices=False))
    b = t(lambda: qr_jacobi(M))
    U, S, Vt = qr_jacobi(M)
    err = float(torch.linalg.matrix_norm(U * S @ Vt - M) / torch.linalg.matrix_norm(M))
    s_ref = torch.linalg.svdvals(M)
    print(shape, "torch %.2f ms  qr+jacobi %.2f ms  rec err %.1e  sv err %.1e" % (a, b, err, float((S - s_ref).abs().max() / s_ref[0])))

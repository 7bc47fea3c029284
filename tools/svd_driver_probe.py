"""SVD route timings for _left_sv shapes (dev tool)."""
import time, torch
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
for n, m in [(127, 400), (127, 2500), (127, 10000), (127, 40000), (255, 10000)]:
    M = torch.randn(n, m, dtype=torch.float64, device="cuda")
    res = {}
    for drv in (None, "gesvd", "gesvdj", "gesvda"):
        try:
            res[str(drv)] = round(t(lambda: torch.linalg.svd(M, full_matrices=False, driver=drv)), 2)
        except Exception as e:
            res[str(drv)] = "err"
    def qr_route():
        R = torch.linalg.qr(M.T, mode="r")[1]       # M^T = Q R, M = R^T Q^T
        U, s, _ = torch.linalg.svd(R.T)
        return U
    res["qr+svd"] = round(t(qr_route), 2)
    def qr_route_j():
        R = torch.linalg.qr(M.T, mode="r")[1]
        U, s, _ = torch.linalg.svd(R.T, driver="gesvdj")
        return U
    res["qr+svdj"] = round(t(qr_route_j), 2)
    # accuracy of leading subspace vs default
    U0 = torch.linalg.svd(M, full_matrices=False)[0][:, :20]
    R = torch.linalg.qr(M.T, mode="r")[1]; U1 = torch.linalg.svd(R.T)[0][:, :20]
    res["qr_subspace_err"] = float(torch.linalg.matrix_norm(U0 @ U0.T - U1 @ U1.T))
    print(n, m, res, flush=True)

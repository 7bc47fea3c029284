"""Left singular vectors of wide 127 x m matrices: route timings (dev tool)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))



def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


def sub_err(U, Uref, r):
    # distance between leading r-subspaces
    P = U[:, :r].T @ Uref[:, :r]
    s = np.linalg.svd(P, compute_uv=False)
    return float(np.sqrt(max(0.0, r - np.sum(s ** 2))))


rng = np.random.default_rng(0)
for m in (144, 2112, 131400):
    # decaying spectrum like the truncation inputs
    n = 127
    A = rng.standard_normal((n, n)) @ np.diag(np.logspace(0, -14, n)) @ np.linalg.qr(rng.standard_normal((m, n)))[0].T
    M = torch.tensor(A, device="cuda")
    Uref = np.linalg.svd(A, full_matrices=False)[0]
    res = {}
    for drv in (None, "gesvd", "gesvdj", "gesvda"):
        try:
            ms, out = t(lambda: torch.linalg.svd(M, full_matrices=False, driver=drv))
            res["svd[%s]" % drv] = (ms, sub_err(out[0].cpu().numpy(), Uref, 40))
        except Exception as e:
            res["svd[%s]" % drv] = str(e)[:60]

    def qr_route(drv=None):
        R = torch.linalg.qr(M.T)[1]
        return torch.linalg.svd(R.T, full_matrices=False, driver=drv)[0]
    for drv in (None, "gesvd", "gesvdj"):
        ms, U = t(lambda: qr_route(drv))
        res["qr+svd[%s]" % drv] = (ms, sub_err(U.cpu().numpy(), Uref, 40))

    def cpu_route():
        R = torch.linalg.qr(M.T)[1]
        u = np.linalg.svd(R.T.cpu().numpy())[0]
        return torch.tensor(u, device="cuda")
    ms, U = t(cpu_route)
    res["qr+cpu"] = (ms, sub_err(U.cpu().numpy(), Uref, 40))

    def gram():
        w, V = torch.linalg.eigh(M @ M.T)
        return V.flip(1)
    ms, U = t(gram)
    res["gram+eigh"] = (ms, sub_err(U.cpu().numpy(), Uref, 40))
    ms, _ = t(lambda: torch.linalg.qr(M.T)[1])
    res["qr only"] = (ms, 0)
    from paper_1809_01971_b200.decomp import svd_batched

    def jac():
        R = torch.linalg.qr(M.T)[1]
        U, s, _ = svd_batched(R.T.contiguous()[None])
        return U[0], s[0]
    ms, (U, s) = t(jac)
    sref = np.linalg.svd(A, compute_uv=False)
    res["qr+jacobi"] = (ms, sub_err(U.cpu().numpy(), Uref, 40))
    print("   jacobi sigma rel err (top 60): %.1e" % np.max(np.abs(s.cpu().numpy()[:60] - sref[:60]) / sref[:60]))
    Rt = torch.linalg.qr(M.T)[1].T.contiguous()
    ms, _ = t(lambda: svd_batched(Rt[None]))
    res["jacobi only"] = (ms, 0)
    ms, (U2, s2, _) = t(lambda: svd_batched(Rt[None], right=False))
    res["jacobi left"] = (ms, float(torch.max(torch.abs(U2[0] - U.cpu().cuda() if False else U2[0] - jac()[0]))))
    ms, _ = t(lambda: torch.linalg.svdvals(M))
    res["svdvals"] = (ms, 0)
    ms, _ = t(lambda: torch.linalg.svdvals(torch.linalg.qr(M.T)[1]))
    res["qr+svdvals"] = (ms, 0)
    print(m, flush=True)
    for k, v in res.items():
        print("   %-16s %s" % (k, v if isinstance(v, str) else "%.2f ms  subspace err %.1e" % v), flush=True)

"""configs[0] setup breakdown and small-SVD routes (dev tool)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import fullsolve, fracop, decomp
from paper_1809_01971_b200.fracop import dense_core_dev


def tm(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print("%-40s %8.3f ms (min %8.3f)" % (label, 1e3 * sum(ts) / len(ts), 1e3 * min(ts)), flush=True)
    return out


n = 255
spec = fl.laplacian_spectrum(n, 2)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-3, eps=1e-10, precond_rank=6, residual_tol=1e-8, k_max=100)
kind = fullsolve._control_kind(cfg)
tm("control_cores total", lambda: fullsolve.control_cores(cfg, spec))
tm("dense_core (A)", lambda: fullsolve.dense_core(kind, spec))
tm("kronecker_preconditioner", lambda: fullsolve.kronecker_preconditioner(cfg, spec))
G = dense_core_dev(kind, spec, True)
tm("dense_core_dev reciprocal", lambda: dense_core_dev(kind, spec, True))
tm("torch.linalg.svd 255x255", lambda: torch.linalg.svd(G, full_matrices=False))
tm("torch.linalg.svdvals 255x255", lambda: torch.linalg.svdvals(G))
tm("svd_batched (Jacobi) 255x255", lambda: decomp.svd_batched(G[None]))
tm("eigh(G G^T)", lambda: torch.linalg.eigh(G @ G.T))
U, S, Vt = torch.linalg.svd(G, full_matrices=False)
U2, S2, V2 = decomp.svd_batched(G[None])
print("sv rel diff jacobi vs lib:", float(((S2[0] - S).abs() / S).max()))
for m in (127, 63):
    Gm = G[:m, :m].contiguous()
    tm("torch.linalg.svd %dx%d" % (m, m), lambda: torch.linalg.svd(Gm, full_matrices=False))
    tm("svd_batched %dx%d" % (m, m), lambda: decomp.svd_batched(Gm[None]))
for shape in ((127, 1600), (127, 20000), (127, 131400)):
    M = torch.randn(shape, dtype=torch.float64, device="cuda")
    tm("left_sv %s lib svd" % (shape,), lambda: torch.linalg.svd(M, full_matrices=False), reps=3)
    tm("left_sv %s qr(M^T) r-only" % (shape,), lambda: torch.linalg.qr(M.T, mode="r"), reps=3)
    tm("left_sv %s gram" % (shape,), lambda: M @ M.T, reps=3)

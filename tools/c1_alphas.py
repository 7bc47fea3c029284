"""configs[1] at the three alphas, build included (dev tool): seconds, iterations, rank."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
n = 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
out = []
for alpha in (0.25, 0.5, 0.75):
    cfg = fl.SolverConfig(alpha=alpha, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
    fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u, rep = fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize()
    out.append("alpha %.2f: %.3f s, %d its, rank %d, res %.3e" % (alpha, time.perf_counter() - t0, rep.iterations, u.rank, rep.residuals[-1]))
print("FL_KR_FUSED=%s | " % os.environ.get("FL_KR_FUSED", "1") + " | ".join(out))

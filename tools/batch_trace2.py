"""Residual / rank history of one configs[4] problem (dev tool): python tools/batch_trace2.py N PROBLEM [k_max]"""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, solver, spectral
import paper_1809_01971_b200 as fl
n, i = int(sys.argv[1]), int(sys.argv[2])
kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 25
spec = spectral.laplacian_spectrum(n, 3)
y, cfg = batch.problem(i, n)
cfg = fl.SolverConfig(alpha=cfg.alpha, beta=cfg.beta, eps=cfg.eps, precond_rank=cfg.precond_rank,
                      residual_tol=cfg.residual_tol, k_max=kmax)
print("problem %d n=%d alpha %.4f beta %.3e" % (i, n, cfg.alpha, cfg.beta), flush=True)
orig_tr = solver.trunc
def tr(x, spec_, **kw):
    t0 = time.perf_counter()
    out = orig_tr(x, spec_, **kw)
    torch.cuda.synchronize()
    print("    trunc %s rank %d -> %d  %.2f s" % (type(x).__name__, x.rank, out.rank, time.perf_counter() - t0), flush=True)
    return out
solver.trunc = tr
orig_inner = solver.cp_inner_dev
def inner(a, b):
    v = orig_inner(a, b)
    print("    inner %.6e" % float(v), flush=True)
    return v
solver.cp_inner_dev = inner
t0 = time.perf_counter()
try:
    u, rep = batch.solve_control_large(y, cfg, spec)
    print("done: its %d converged %s residuals %s" % (rep.iterations, rep.converged, ["%.2e" % r for r in rep.residuals]))
except Exception as e:
    print("FAILED %s: %s" % (type(e).__name__, str(e)[:300]))
print("%.1f s" % (time.perf_counter() - t0))

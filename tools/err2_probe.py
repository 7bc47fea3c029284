"""The values c2t's rank-growth test sees at configs[1] (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp
orig = decomp._c2t_at_ranks
log = []
def traced(an, ranks, sweeps, left=None):
    tt = orig(an, ranks, sweeps, left)
    nrm = decomp.cp_norm(an)
    c2 = float(torch.sum(tt.core * tt.core))
    # the true error through the dense expansion when it is affordable
    log.append((an.dims, an.rank, ranks, (nrm * nrm - c2) / (nrm * nrm)))
    return tt
decomp._c2t_at_ranks = traced
n = 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
for alpha in (0.25, 0.5, 0.75):
    cfg = fl.SolverConfig(alpha=alpha, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
    log.clear()
    fl.solve_control(y, cfg, spec)
    print("alpha", alpha, "attempts", len(log))
    for dims, R, ranks, rel in log:
        print("   dims %s R %d ranks %s  (nrm^2 - core^2)/nrm^2 = %+.3e   (tol^2 = 2.5e-17)" % (dims, R, ranks, rel))

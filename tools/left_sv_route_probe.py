"""configs[1] solve time and result for two _left_sv Jacobi size caps (dev tool)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp
from paper_1809_01971_b200.tensor import cp_inner, cp_norm
n = 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
caps = [int(v) for v in sys.argv[1:]] or [64, 128]
outs = {}
for cap in caps + caps:
    decomp._JACOBI_LEFT_SV_MAX = cap
    fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize()
    outs[cap] = u
    print("cap %d: %.3f s, %d its, rank %d, residuals %s" % (cap, time.perf_counter() - t0, rep.iterations, u.rank,
          ["%.2e" % r for r in rep.residuals][-2:]), flush=True)
a, b = outs[caps[0]], outs[caps[-1]]
na, nb = cp_norm(a), cp_norm(b)
print("relative difference of the controls: %.2e" % (max(0.0, na ** 2 + nb ** 2 - 2 * cp_inner(a, b)) ** 0.5 / na))

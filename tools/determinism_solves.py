"""Bitwise determinism of the solves (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import fullsolve, full
def same(a, b):
    if isinstance(a, torch.Tensor):
        return torch.equal(a, b)
    return all(torch.equal(x, y) for x, y in zip([a.weights] + list(a.factors), [b.weights] + list(b.factors)))
# full-format 2D (configs[0]-like) and 3D n=255 spectral PCG
for dims in ((255, 255), (127, 127, 127)):
    n = dims[0]
    spec = fl.laplacian_spectrum(n, len(dims))
    cfg = fl.SolverConfig(alpha=0.5, beta=1e-3, residual_tol=1e-8)
    y = full.cp_dense(fl.gaussian_bumps(n, len(dims), 4, seed=1))
    cores = fullsolve.control_cores(cfg, spec)
    u1, r1 = fullsolve.solve_control_full(y, cfg, spec, cores=cores)
    u2, r2 = fullsolve.solve_control_full(y, cfg, spec, cores=cores)
    cores2 = fullsolve.control_cores(cfg, spec)
    print(dims, "solve bitwise equal:", torch.equal(u1, u2), r1.iterations, r2.iterations,
          "| cores rebuilt equal:", torch.equal(cores[0], cores2[0]), torch.equal(cores[1], cores2[1]), flush=True)
# canonical 3D n=31
spec = fl.laplacian_spectrum(31, 3)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8)
y = fl.gaussian_bumps(31, 3, 8, seed=11)
u1, r1 = fl.solve_control(y, cfg, spec)
u2, r2 = fl.solve_control(y, cfg, spec)
print("canonical n=31:", same(u1, u2), r1.iterations, r2.iterations, u1.rank, u2.rank, flush=True)

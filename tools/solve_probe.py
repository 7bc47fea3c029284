"""Timing/profile probe for the solvers (development tool)."""
import cProfile, pstats, sys, time
import numpy as np
import torch
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import fullsolve

which = sys.argv[1]
if which == "canon":
    n = int(sys.argv[2]); alpha = float(sys.argv[3])
    spec = fl.laplacian_spectrum(n, 3)
    y = fl.gaussian_bumps(n, 3, 8, seed=11)
    cfg = fl.SolverConfig(alpha=alpha, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
    import paper_1809_01971_b200.decomp as dec
    orig = dec.trunc
    def traced(x, spec):
        out = orig(x, spec); print("  trunc rank %d -> %d" % (x.rank, out.rank)); return out
    import paper_1809_01971_b200.solver as sol
    sol.trunc = traced
    pr = cProfile.Profile(); t0 = time.time(); pr.enable()
    u, rep = fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize(); pr.disable()
    print("canonical n=%d alpha=%g: %d its, rank %d, %.2fs, per-it %.3fs" % (n, alpha, rep.iterations, u.rank, time.time() - t0, rep.seconds_per_iteration))
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)
else:
    n = int(sys.argv[2])
    spec = fl.laplacian_spectrum(n, 3)
    w, f = fl.gaussian_bumps(n, 3, 16, seed=7).numpy()
    yc = fl.CpTensor(w, f)
    y = fl.cp_to_dense(yc) if n ** 3 <= 2 ** 24 else None
    if y is None:
        from paper_1809_01971_b200 import full
        y = full.cp_dense(yc)
    y.add_(1e-3 * torch.randn_like(y))
    cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, precond_rank=6, residual_tol=1e-8, k_max=100)
    torch.cuda.synchronize(); t0 = time.time()
    cores = fullsolve.control_cores(cfg, spec)
    torch.cuda.synchronize(); t1 = time.time()
    u, rep = fullsolve.solve_control_full(y, cfg, spec, cores=cores)
    torch.cuda.synchronize(); t2 = time.time()
    print("full n=%d: setup %.2fs solve %.3fs its %d per-it %.2f ms res %.2e mem %.1f GB" % (n, t1 - t0, t2 - t1, rep.iterations, 1e3 * rep.seconds_per_iteration, rep.residuals[-1], torch.cuda.max_memory_allocated() / 1e9))

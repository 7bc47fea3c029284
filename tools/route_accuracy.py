"""Solution error vs the exact optimality solve for the canonical routes at
full size (dev tool):
  python tools/route_accuracy.py c1 ALPHA        configs[1] n=127: compressed vs uncompressed truncation
  python tools/route_accuracy.py c4 N I          configs[4]: large-grid route vs reference-shaped route"""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import batch, decomp, full
from paper_1809_01971_b200.full import cp_dense


def err(spec, cfg, u, y):
    kind = fl.CoreFunctionKind("g2", cfg.alpha, coeff_minus=float(cfg.beta), coeff_plus=float(cfg.gamma) / float(cfg.beta))
    inv = full.FullOperator.from_kind(kind, spec, reciprocal=True)
    yd = cp_dense(y)
    us = inv(yd)
    ud = cp_dense(u)
    return float(torch.linalg.vector_norm(ud - us) / torch.linalg.vector_norm(us))


mode = sys.argv[1]
if mode == "c1":
    alpha = float(sys.argv[2])
    n = 127
    spec = fl.laplacian_spectrum(n, 3)
    y = fl.gaussian_bumps(n, 3, 8, seed=11)
    for label, cmin, eps in (("compressed", 100, 1e-8), ("uncompressed", 1 << 30, 1e-8), ("compressed eps1e-10", 100, 1e-10)):
        decomp._COMPRESS_MIN_N = cmin
        cfg = fl.SolverConfig(alpha=alpha, beta=1e-2, eps=eps, precond_rank=6, residual_tol=1e-6, k_max=60)
        t0 = time.perf_counter()
        u, rep = fl.solve_control(y, cfg, spec)
        print("c1 alpha %.2f %-20s its %d rank %d err vs exact %.3e (%.1f s)" % (alpha, label, rep.iterations, u.rank,
              err(spec, cfg, u, y), time.perf_counter() - t0), flush=True)
else:
    n, i = int(sys.argv[2]), int(sys.argv[3])
    spec = fl.laplacian_spectrum(n, 3)
    y, cfg = batch.problem(i, n)
    t0 = time.perf_counter()
    u, rep = batch.solve_control_large(y, cfg, spec)
    print("c4 n=%d problem %d large route: its %d rank %d err %.3e (%.1f s)" % (n, i, rep.iterations, u.rank,
          err(spec, cfg, u, y), time.perf_counter() - t0), flush=True)
    for label, c in (("tol 1e-8 large route", fl.SolverConfig(alpha=cfg.alpha, beta=cfg.beta, eps=1e-8, precond_rank=6,
                                                               residual_tol=1e-6, k_max=60)),):
        t0 = time.perf_counter()
        u, rep = batch.solve_control_large(y, c, spec)
        print("c4 n=%d problem %d %s: its %d rank %d err %.3e (%.1f s)" % (n, i, label, rep.iterations, u.rank,
              err(spec, c, u, y), time.perf_counter() - t0), flush=True)
    t0 = time.perf_counter()
    with decomp.dense_budget(n ** 3):
        u, rep = fl.solve_control(y, cfg, spec)
    print("c4 n=%d problem %d reference-shaped route: its %d rank %d err %.3e (%.1f s)" % (n, i, rep.iterations, u.rank,
          err(spec, cfg, u, y), time.perf_counter() - t0), flush=True)

"""Trace one configs[4] problem (dev tool): python tools/batch_trace.py N i
prints every cp_norm the PCG takes (relative residual trail) and the ranks."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, spectral, solver
n, i = int(sys.argv[1]), int(sys.argv[2])
orig_norm = solver.cp_norm
orig_tr = solver.trunc
t0 = time.perf_counter()


def norm(x):
    v = orig_norm(x)
    print("  %7.2fs cp_norm rank %6d -> %.6e" % (time.perf_counter() - t0, x.rank, v), flush=True)
    return v


def tr(x, spec, overwrite_input=False):
    out = orig_tr(x, spec, overwrite_input)
    print("  %7.2fs trunc %d -> %d" % (time.perf_counter() - t0, x.rank, out.rank), flush=True)
    return out


solver.cp_norm = norm
solver.trunc = tr
spec = spectral.laplacian_spectrum(n, 3)
y, cfg = batch.problem(i, n)
print("n=%d problem %d alpha %.4f beta %.3e" % (n, i, cfg.alpha, cfg.beta), flush=True)
u, rep = batch.solve_control_large(y, cfg, spec)
print("its", rep.iterations, "conv", rep.converged, "rank", u.rank, "%.1fs" % (time.perf_counter() - t0))

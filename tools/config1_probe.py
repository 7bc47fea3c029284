"""Where configs[1] (3D canonical control solve, n=127) spends its time (dev tool)."""
import os
import sys
import time
import collections
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp, fracop, solver

stats = collections.defaultdict(lambda: [0, 0.0])


def wrap(mod, name, label):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize()
        stats[label][0] += 1
        stats[label][1] += time.perf_counter() - t0
        return out
    setattr(mod, name, g)


if os.environ.get("FL_COMPRESS_MIN_N"):
    decomp._COMPRESS_MIN_N = int(os.environ["FL_COMPRESS_MIN_N"])
for nm in ("trunc", "c2t", "t2c", "_merge_collinear", "rhosvd", "_pick_ranks", "_svd", "_left_sv", "_kr_contract",
           "_cp_project_core", "_range_basis_gen", "cp_norm", "multigrid_tucker", "_core_cp_als", "tucker_als"):
    if hasattr(decomp, nm):
        wrap(decomp, nm, "decomp." + nm)
for nm in ("build_core", "reciprocal_core", "apply", "apply_compressed", "_probe_error"):
    wrap(fracop, nm, "fracop." + nm)
for nm in ("trunc", "apply", "apply_compressed", "build_preconditioner", "cp_inner", "cp_norm"):
    if hasattr(solver, nm):
        wrap(solver, nm, "solver." + nm)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
fl.solve_control(y, cfg, spec)  # warm
stats.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
u, rep = fl.solve_control(y, cfg, spec)
torch.cuda.synchronize()
print("n=%d total %.2f s, %d its, rank %d, per-iter %s" % (n, time.perf_counter() - t0, rep.iterations, u.rank,
      [round(v, 2) for v in rep.iteration_seconds]))
for k, (c, t) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print("  %-28s %4d calls %8.3f s" % (k, c, t))

"""Time breakdown of one configs[4] problem (dev tool): python tools/batch_profile.py N"""
import os, sys, time, collections, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, decomp, fracop, solver
stats = collections.defaultdict(lambda: [0, 0.0])
def wrap(mod, name, label):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = f(*a, **k); torch.cuda.synchronize()
        stats[label][0] += 1; stats[label][1] += time.perf_counter() - t0; return out
    setattr(mod, name, g)
for nm in ("trunc", "c2t", "t2c", "_merge_collinear", "rhosvd", "_pick_ranks", "_svd", "_left_sv", "_kr_contract",
           "_cp_project_core", "_range_basis_gen", "cp_norm", "svd_batched", "_core_cp_als", "tucker_als", "multigrid_tucker"):
    if hasattr(decomp, nm): wrap(decomp, nm, "decomp." + nm)
for nm in ("apply", "apply_compressed", "build_core", "reciprocal_core"):
    if hasattr(fracop, nm): wrap(fracop, nm, "fracop." + nm)
for nm in ("apply", "apply_compressed", "build_preconditioner", "trunc", "cp_inner"):
    if hasattr(solver, nm): wrap(solver, nm, "solver." + nm)
for nm in ("control_core_expsum", "preconditioner_coarse", "pcg", "trunc", "multigrid_tucker", "t2c"):
    wrap(batch, nm, "batch." + nm)
n = int(sys.argv[1])
list(batch.solve_batch(n, 1))  # warm-up
stats.clear()
t0 = time.perf_counter()
recs = list(batch.solve_batch(n, 1))
print("n=%d total %.2f s" % (n, time.perf_counter() - t0), recs[0].get("iterations"), flush=True)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:22]:
    print("  %-28s %5d calls %8.3f s" % (k, v[0], v[1]))

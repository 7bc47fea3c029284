"""Where the configs[3] setup (n=1023 Kronecker preconditioner + dense cores) spends its time (dev tool)."""
import os, sys, time, collections, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp, fracop, fullsolve, full
stats = collections.defaultdict(lambda: [0, 0.0])
def wrap(mod, name, label):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = f(*a, **k); torch.cuda.synchronize()
        stats[label][0] += 1; stats[label][1] += time.perf_counter() - t0; return out
    setattr(mod, name, g)
for nm in ("multigrid_tucker", "tucker_als", "hosvd", "t2c", "c2t", "trunc", "_svd", "_left_sv", "svd_batched", "rhosvd", "cp_norm", "_merge_collinear"):
    if hasattr(decomp, nm): wrap(decomp, nm, "decomp." + nm)
for nm in ("reciprocal_core", "build_core", "_dense_core"):
    if hasattr(fracop, nm): wrap(fracop, nm, "fracop." + nm)
wrap(full, "dense_core", "full.dense_core"); wrap(full, "cp_dense", "full.cp_dense")
n = 1023
spec = fl.laplacian_spectrum(n, 3)
cfg = fl.SolverConfig(alpha=0.75, beta=1e-4)
fullsolve.control_cores(cfg, spec)  # warm-up
stats.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
fullsolve.control_cores(cfg, spec)
torch.cuda.synchronize()
print("control_cores %.3f s" % (time.perf_counter() - t0))
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print("  %-28s %4d calls %7.3f s" % (k, v[0], v[1]))

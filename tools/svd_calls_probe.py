"""Shapes and times of the SVD calls of the configs[1] solve (dev tool)."""
import collections, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp

rec = collections.defaultdict(lambda: [0, 0.0])
depth = [0]


def wrap(name):
    f = getattr(decomp, name)

    def g(M, *a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        depth[0] += 1
        out = f(M, *a, **k)
        depth[0] -= 1
        torch.cuda.synchronize()
        key = (name, depth[0], tuple(M.shape), k.get("compute_uv", a[0] if a and name == "_svd" else True))
        rec[key][0] += 1
        rec[key][1] += time.perf_counter() - t0
        return out
    setattr(decomp, name, g)


wrap("_left_sv")
wrap("_svd")
n = 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
fl.solve_control(y, cfg, spec)
rec.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
fl.solve_control(y, cfg, spec)
torch.cuda.synchronize()
print("total %.2f s" % (time.perf_counter() - t0))
for k, (c, t) in sorted(rec.items(), key=lambda kv: -kv[1][1])[:30]:
    print("  %-50s %4d calls %8.3f s (%.2f ms each)" % (k, c, t, 1e3 * t / c))

import collections, time, torch
import paper_1809_01971_b200 as fl
stats = collections.defaultdict(lambda: [0, 0.0])
orig_svd, orig_vals = torch.linalg.svd, torch.linalg.svdvals
def wrap(fn, tag):
    def f(A, *a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = fn(A, *a, **k); torch.cuda.synchronize()
        key = (tag, tuple(A.shape)[-2:] if A.ndim >= 2 else tuple(A.shape), A.ndim)
        bucket = (tag, "x".join(str(min(s, 10**6)) for s in key[1]) if max(key[1]) < 200 else "%s:big(%s)" % (tag, "x".join(map(str, key[1]))))
        stats[(tag, key[1][0] if len(key[1]) else 0, key[1][1] >= 1000 if len(key[1]) > 1 else False)][0] += 1
        stats[(tag, key[1][0] if len(key[1]) else 0, key[1][1] >= 1000 if len(key[1]) > 1 else False)][1] += time.perf_counter() - t
        return r
    return f
torch.linalg.svd = wrap(orig_svd, "svd"); torch.linalg.svdvals = wrap(orig_vals, "svdvals")
spec = fl.laplacian_spectrum(127, 3)
y = fl.gaussian_bumps(127, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
u, rep = fl.solve_control(y, cfg, spec)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:12]:
    print(k, v[0], "%.3f s" % v[1])

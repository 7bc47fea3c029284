"""A/B of trunc with and without the hand-written wide factorisations on the
compression test's case (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp


def smooth_cp(dims, R, seed):
    rng = np.random.default_rng(seed)
    fs = []
    for n in dims:
        x = (np.arange(n) + 1.0) / (n + 1.0)
        c = rng.uniform(0.2, 0.8, R); s = rng.uniform(0.05, 0.2, R)
        fs.append(np.exp(-((x[:, None] - c[None, :]) / s[None, :]) ** 2))
    return fl.CpTensor(rng.standard_normal(R), fs)


orig = decomp._c2t_at_ranks
def traced(an, ranks, sweeps, left=None):
    tt = orig(an, ranks, sweeps, left)
    print("    c2t_at_ranks dims", an.dims, "ranks", ranks, "core^2 %.17g" % float(torch.sum(tt.core * tt.core)))
    return tt
decomp._c2t_at_ranks = traced
for dims, R, tol in [((255, 255, 255), 1200, 1e-6), ((255, 63, 191), 250, 1e-6), ((127, 127, 127), 400, 1e-8)]:
    x = smooth_cp(dims, R, seed=R)
    spec = decomp.TruncationSpec(tolerance=tol)
    dx = fl.cp_norm(x)
    res = {}
    for wide in (False, True):
        for comp in (False, True):
            decomp._WIDE_ENABLED = wide
            decomp._COMPRESS_MIN_N = 16 if comp else 1 << 30
            print("  wide", wide, "compressed", comp)
            res[(wide, comp)] = decomp.trunc(x, spec)
    keys = list(res)
    for a in range(len(keys)):
        for b in range(a + 1, len(keys)):
            d = fl.cp_norm(fl.cp_add(res[keys[a]], fl.cp_scale(res[keys[b]], -1.0)))
            print(dims, keys[a], keys[b], "ranks", res[keys[a]].rank, res[keys[b]].rank, "diff/(tol dx) %.3e" % (d / (tol * dx)))
    for kk in keys:
        e = fl.cp_norm(fl.cp_add(res[kk], fl.cp_scale(x, -1.0)))
        print(dims, kk, "err/(tol dx) %.3f" % (e / (tol * dx)))

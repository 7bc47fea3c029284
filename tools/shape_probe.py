"""Histogram of the factorisation shapes the canonical solves issue (dev tool):
python tools/shape_probe.py c1|c4 [n]"""
import os, sys, collections, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import batch, decomp

hist = collections.defaultdict(lambda: [0, 0.0])


def wrap(mod, name, key):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize()
        h = hist[key(*a, **k)]; h[0] += 1; h[1] += time.perf_counter() - t0
        return out
    setattr(mod, name, g)


def bucket(v, q=16):
    return (int(v) + q - 1) // q * q


wrap(decomp, "_left_sv", lambda M, r, *a: ("left_sv", bucket(min(M.shape)), bucket(max(M.shape), 512), "wide" if M.shape[0] <= M.shape[1] else "tall"))
wrap(decomp, "_svdvals", lambda M: ("svdvals", bucket(min(M.shape)), bucket(max(M.shape), 512)))
wrap(decomp, "_svd", lambda M, compute_uv=True: ("lib_svd", bucket(min(M.shape)), bucket(max(M.shape), 512)))
wrap(decomp, "_range_basis_gen", lambda block, n, R, w, *a, **k: ("range", n, bucket(R, 4096)))
_qr, _sv = torch.linalg.qr, torch.linalg.svd


def qr(A, mode="reduced"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = _qr(A, mode=mode)
    torch.cuda.synchronize()
    h = hist[("qr_" + mode, bucket(A.shape[1]), bucket(A.shape[0], 512))]; h[0] += 1; h[1] += time.perf_counter() - t0
    return out


def sv(A, full_matrices=True):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = _sv(A, full_matrices=full_matrices)
    torch.cuda.synchronize()
    h = hist[("linalg_svd", bucket(min(A.shape[-2:])), bucket(max(A.shape[-2:]), 512))]; h[0] += 1; h[1] += time.perf_counter() - t0
    return out


torch.linalg.qr, torch.linalg.svd = qr, sv
which = sys.argv[1]
if which == "c1":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 127
    spec = fl.laplacian_spectrum(n, 3)
    y = fl.gaussian_bumps(n, 3, 8, seed=11)
    cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
    run = lambda: fl.solve_control(y, cfg, spec)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1023
    cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    run = lambda: list(batch.solve_batch(n, cnt))
run()
hist.clear()
t0 = time.perf_counter()
run()
print("%s n=%d total %.2f s" % (which, n, time.perf_counter() - t0))
tot = collections.defaultdict(float)
for k, (c, t) in sorted(hist.items(), key=lambda kv: (kv[0][0], -kv[1][1])):
    print("  %-44s %5d calls %8.3f s  (%.2f ms)" % (k, c, t, 1e3 * t / c))
    tot[k[0]] += t
print({k: round(v, 3) for k, v in tot.items()})

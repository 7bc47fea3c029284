"""k_jacobi_small timing on random / graded / real configs[1] factors (dev tool)."""
import os, sys, time, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp


def tm(label, fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print("%-44s %8.3f ms" % (label, (time.perf_counter() - t0) / reps * 1e3), flush=True)
    return out


rng = np.random.default_rng(0)
for k in (64, 127, 128):
    A = torch.tensor(rng.standard_normal((k, k)), device="cuda")
    tm("jacobi_small random %dx%d" % (k, k), lambda: decomp.svd_batched(A[None], right=False))
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k))); Q2, _ = np.linalg.qr(rng.standard_normal((k, k)))
    G = torch.tensor((Q1 * 10.0 ** (-18 * np.arange(k) / (k - 1))) @ Q2.T, device="cuda")
    tm("jacobi_small graded 1e-18 %dx%d" % (k, k), lambda: decomp.svd_batched(G[None], right=False))
p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tmpdata", "leftsv_samples.npz")
if os.path.exists(p):
    d = np.load(p)
    for key in d.files[:3]:
        M = torch.tensor(d[key], device="cuda")
        tm("real %s qr r-only" % (tuple(M.shape),), lambda: torch.linalg.qr(M.T, mode="r"))
        _, X = decomp._small_factor(M)
        tm("real %s jacobi on R^T" % (tuple(M.shape),), lambda: decomp.svd_batched(X[None], right=False))
        tm("real %s _left_sv" % (tuple(M.shape),), lambda: decomp._left_sv(M, 40))
        tm("real %s lib svd" % (tuple(M.shape),), lambda: torch.linalg.svd(M, full_matrices=False))
# pivoted route (column-pivoted QR + Jacobi on R^T)
for k in (64, 127):
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k))); Q2, _ = np.linalg.qr(rng.standard_normal((k, k)))
    G = torch.tensor((Q1 * 10.0 ** (-18 * np.arange(k) / (k - 1))) @ Q2.T, device="cuda")
    tm("pivoted graded 1e-18 %dx%d" % (k, k), lambda: decomp.svd_left_pivoted(G))
if os.path.exists(p):
    for key in d.files[:3]:
        M = torch.tensor(d[key], device="cuda")
        R = torch.linalg.qr(M.T, mode="r")[1]
        tm("real %s pivoted on R^T" % (tuple(M.shape),), lambda: decomp.svd_left_pivoted(R.T))
        tm("real %s _left_sv (pivoted route)" % (tuple(M.shape),), lambda: decomp._left_sv(M, 40))

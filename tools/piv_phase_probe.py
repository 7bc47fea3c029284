"""Cost of the pivoted-QR phase of k_jacobi_small<.., PIV>: a diagonal input needs no rotations (dev tool)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp
def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for k in (127, 96, 64, 48):
    D = torch.diag(torch.tensor(10.0 ** (-12 * np.arange(k) / (k - 1)), device="cuda"))
    rng = np.random.default_rng(k)
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k))); Q2, _ = np.linalg.qr(rng.standard_normal((k, k)))
    G = torch.tensor((Q1 * 10.0 ** (-12 * np.arange(k) / (k - 1))) @ Q2.T, device="cuda")
    t_diag = timeit(lambda: decomp.svd_left_pivoted(D))
    t_full = timeit(lambda: decomp.svd_left_pivoted(G))
    t_plain = timeit(lambda: decomp.svd_batched(D[None], right=False))
    print("k=%d: pivoted on a diagonal matrix (QR + one checking sweep) %.3f ms, graded dense %.3f ms; unpivoted kernel on the diagonal matrix (one sweep) %.3f ms" % (k, t_diag, t_full, t_plain))

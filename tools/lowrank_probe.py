"""left_sv routes on exactly rank-deficient wide matrices (ALS-like), dev tool."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp


def timeit(f, reps=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


rng = np.random.default_rng(0)
for k, m, r in [(48, 1024, 30), (64, 4096, 40), (64, 512, 50), (127, 2500, 60), (127, 2500, 127)]:
    X = rng.standard_normal((k, r)) * np.logspace(0, -9, r)
    Y = rng.standard_normal((r, m))
    M = torch.tensor(X @ Y, device="cuda")
    out = []
    for wide in (True, False):
        decomp._WIDE_ENABLED = wide
        t = timeit(lambda: decomp._left_sv(M, r))
        out.append("%s %.3f ms" % ("wide" if wide else "old", t))
    decomp._WIDE_ENABLED = True
    R = decomp.qr_r_wide([M])[0]
    t_q = timeit(lambda: decomp.qr_r_wide([M]))
    t_p = timeit(lambda: decomp.svd_left_pivoted(R.T.contiguous()))
    t_n = timeit(lambda: decomp.svd_batched(R.T.contiguous()[None], right=False))
    print("k=%d m=%d rank %d: %s | tsqr %.3f, pivoted jacobi %.3f, plain jacobi on R^T %.3f" % (k, m, r, ", ".join(out), t_q, t_p, t_n), flush=True)

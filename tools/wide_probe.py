"""Timing of the hand-written wide factorisations vs the library (dev tool)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp


def graded(k, m, grade, seed):
    rng = np.random.default_rng(seed)
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, k)))
    sv = 10.0 ** (-grade * np.arange(k) / (k - 1))
    return torch.tensor((Q1 * sv) @ Q2.T, device="cuda")


def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for k, m in [(127, 2039), (127, 8192), (127, 130000), (64, 2048), (48, 1024), (96, 30000), (127, 512)]:
    M = graded(k, m, 16.0, 1)
    Mt = M.T.contiguous().T
    t_lib = timeit(lambda: torch.linalg.qr(M.T, mode="r"))
    t_own = timeit(lambda: decomp.qr_r_wide([M]))
    t_own_t = timeit(lambda: decomp.qr_r_wide([Mt]))
    t_sv1 = timeit(lambda: decomp.left_sv_wide([M]))
    t_sv5 = timeit(lambda: decomp.left_sv_wide([M, Mt, M, M, Mt], vectors=[True, True, True, False, False]))
    t_vals = timeit(lambda: decomp.left_sv_wide([M], vectors=False))
    print("k=%d m=%d: qr lib %.3f ms, tsqr %.3f (transposed storage %.3f); left_sv 1: %.3f, batch of 5: %.3f, values only %.3f"
          % (k, m, t_lib, t_own, t_own_t, t_sv1, t_sv5, t_vals), flush=True)

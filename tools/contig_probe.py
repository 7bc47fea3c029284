"""Contiguous plain pass timing at n=511 (dev tool): lines of pitch 512 (padded) and 511 (dense)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1809_01971_b200 import _lib, full
n = 511; L = n * n
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
for P in (512, 511):
    x = torch.randn(L, P, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
    lay = (0, 1, 0, P)
    args = (_lib.ptr(x), _lib.ptr(y), None, n, 1, L, 1, 1, lay, lay, 1.0)
    ms = t(lambda: full.run_pass(args))
    full.run_pass(args); torch.cuda.synchronize()
    idx = torch.randint(0, L, (64,), device="cuda")
    want = oracle.dst(x[idx, :n].cpu().numpy(), axis=1)
    err = np.abs(y[idx, :n].cpu().numpy() - want).max() / np.abs(want).max()
    print("pitch %d: %.3f ms (%.0f GB/s), err %.2e" % (P, ms, 16 * n ** 3 / ms / 1e6, err))

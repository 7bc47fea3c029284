"""Existing kernel on unpadded (511) vs padded (512) row pitch (dev tool)."""
import torch
from paper_1809_01971_b200 import _lib
n = 511
st = _lib.stream_ptr()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
for P in (511, 512):
    x = torch.randn(n, n, P, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    m1 = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), n, n, P, 1.0, st))
    m0 = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), 1, n, n * P, 1.0, st))
    print("pitch %d: mode1 %.3f ms  mode0 %.3f ms  (per-DoF equivalent mode1 %.3f)" % (P, m1, m0, m1 * 511 / P))

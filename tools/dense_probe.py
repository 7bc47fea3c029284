"""Dense sine-matrix DST path (non-FFT n): fl_dst1 vs cuBLAS DGEMM (dev tool)."""
import time
import torch
from paper_1809_01971_b200 import _lib


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


st = _lib.stream_ptr()
for n, outer, inner in [(1000, 1000, 8), (1000, 1, 100000), (300, 300, 300), (100, 10000, 100), (1000, 1000, 1)]:
    x = torch.randn(outer, n, inner, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), outer, n, inner, 1.0, st))
    S = torch.randn(n, n, dtype=torch.float64, device="cuda")
    mb = t(lambda: torch.matmul(S, x))
    fl = 2.0 * n * n * outer * inner
    print("n=%d outer=%d inner=%d: fl_dst1 %.2f ms (%.1f TF/s)  cuBLAS %.2f ms (%.1f TF/s)" % (n, outer, inner, ms, fl / ms / 1e9, mb, fl / mb / 1e9))

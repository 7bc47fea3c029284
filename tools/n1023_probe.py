"""n=1023 transform / pass timings with the CTA kernel (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import full, _lib
n = 1023
spec = fl.laplacian_spectrum(n, 3)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
y = torch.empty_like(x)
st = _lib.stream_ptr()
ms = t(lambda: _lib.call("fl_transform_full", _lib.ptr(x), _lib.ptr(y), 3, _lib.dims_arr((n, n, n)), 1.0, st))
print("fl_transform_full n=1023: %.2f ms (%.0f GB/s per pass avg)" % (ms, 3 * 16 * n ** 3 / ms / 1e6))
for name, (o, i) in {"mode0": (1, n * n), "mode1": (n, n), "mode2": (n * n, 1)}.items():
    ms = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), o, n, i, 1.0, st))
    print(name, "%.2f ms (%.0f GB/s)" % (ms, 16 * n ** 3 / ms / 1e6))

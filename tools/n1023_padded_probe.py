"""n=1023 padded transform passes (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import full, _lib
n = 1023; P = 1024
spec = fl.laplacian_spectrum(n, 3)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
w = torch.zeros(n, n, P, dtype=torch.float64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
xp, wp = _lib.ptr(x), _lib.ptr(w)
B = 16 * n ** 3 / 1e9
lines, strided = full._padded_passes((n, n, n), P)
ms = t(lambda: full.run_pass((xp, wp, None, n, 3, lines, 1, 1, (0, 1, 0, n), (0, 1, 0, P), 1.0)))
print("contig dense->padded %.2f ms (%.0f GB/s)" % (ms, B / ms * 1e3))
for nn, outer, groups, width, lay in strided:
    ms = t(lambda: full.run_pass((wp, wp, None, nn, 0, outer, groups, width, lay, lay, 1.0)))
    print("strided outer %d groups %d: %.2f ms (%.0f GB/s)" % (outer, groups, ms, B / ms * 1e3))
ms = t(lambda: full.transform_full_padded(spec, x))
print("transform_full_padded %.2f ms; transform_full %.2f ms" % (ms, t(lambda: full.transform_full(spec, x))))

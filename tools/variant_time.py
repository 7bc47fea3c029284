"""Time the fused pass and the full apply for alternative library builds (dev tool)."""
import sys, ctypes, torch
from paper_1809_01971_b200 import _lib
path = sys.argv[1]
_lib.LIB_PATH = path
lib = _lib.load()
n = 511
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); core = torch.rand_like(x); y = torch.empty_like(x)
st = _lib.stream_ptr()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
tm = t(lambda: _lib.call("fl_dst1_core", _lib.ptr(x), _lib.ptr(y), _lib.ptr(core), n * n, n, 1, 1.0, st))
tp = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), n, n, n, 1.0, st))
tc = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), n * n, n, 1, 1.0, st))
print("%s: mid %.3f ms  plain-strided %.3f ms  plain-contig %.3f ms" % (path.split('/')[-1], tm, tp, tc))

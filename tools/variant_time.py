"""Per-pass times for an alternative library build (dev tool): python tools/variant_time.py LIB"""
import sys, torch
from paper_1809_01971_b200 import _lib
_lib.LIB_PATH = sys.argv[1]
_lib.load()
n = 511
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); core = torch.rand_like(x); y = torch.empty_like(x)
st = _lib.stream_ptr()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
r = {}
for name, (o, i) in {"mode0": (1, n * n), "mode1": (n, n), "mode2": (n * n, 1)}.items():
    r[name] = round(t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), o, n, i, 1.0, st)), 3)
r["mid"] = round(t(lambda: _lib.call("fl_dst1_core", _lib.ptr(x), _lib.ptr(y), _lib.ptr(core), n * n, n, 1, 1.0, st)), 3)
print(sys.argv[1].split("/")[-1], r)

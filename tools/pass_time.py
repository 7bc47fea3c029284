"""Per-pass timing, n=511 (dev tool). Env FL_DST_PIPE selects the kernel family."""
import os, torch
from paper_1809_01971_b200 import _lib
n = 511
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); core = torch.rand_like(x); y = torch.empty_like(x)
st = _lib.stream_ptr()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
B = 16 * n ** 3 / 1e9
r = {}
for name, (o, i) in {"mode0": (1, n * n), "mode1": (n, n), "mode2": (n * n, 1)}.items():
    ms = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), o, n, i, 1.0, st))
    r[name] = "%.3f ms (%.0f GB/s)" % (ms, B / ms * 1e3)
ms = t(lambda: _lib.call("fl_dst1_core", _lib.ptr(x), _lib.ptr(y), _lib.ptr(core), n * n, n, 1, 1.0, st))
r["mid"] = "%.3f ms (%.0f GB/s)" % (ms, 1.5 * B / ms * 1e3)
print("PIPE=%s" % os.environ.get("FL_DST_PIPE", "1"), r)

"""Run one DST pass a few times (ncu target)."""
import sys
import torch
from paper_1809_01971_b200 import _lib
n = int(sys.argv[1]); mode = sys.argv[2]
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
outer, inner = {"mode0": (1, n*n), "mode1": (n, n), "mode2": (n*n, 1)}[mode]
core = torch.rand_like(x) if len(sys.argv) > 3 else None
for _ in range(4):
    _lib.call("fl_dst1" if core is None else "fl_dst1", _lib.ptr(x), _lib.ptr(y), outer, n, inner, 1.0, _lib.stream_ptr())
torch.cuda.synchronize()
print("ok")

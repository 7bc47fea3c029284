"""Run the fused core pass a few times (ncu target)."""
import sys
import torch
from paper_1809_01971_b200 import _lib
n = int(sys.argv[1])
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); core = torch.rand_like(x)
for _ in range(4):
    _lib.call("fl_dst1_core", _lib.ptr(x), _lib.ptr(x), _lib.ptr(core), n * n, n, 1, 1.0, _lib.stream_ptr())
torch.cuda.synchronize()
print("ok")

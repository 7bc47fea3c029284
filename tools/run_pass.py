"""Run one pass of the padded n=511 apply a few times (ncu target; dev tool)."""
import sys
import torch
from paper_1809_01971_b200 import _lib, spectral, full
from paper_1809_01971_b200.fracop import CoreFunctionKind

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 511
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
name, a = op.passes(x, y)[idx]
for _ in range(4):
    full.run_pass(a)
torch.cuda.synchronize()
print("ran", name)

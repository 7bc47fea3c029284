"""One fused Khatri-Rao contraction at a configs[1] shape (a = 67, b = 72, R = 132000, N = 127) for ncu (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp
a, b, R, N = 67, 72, 132000, 127
g = torch.Generator(device="cuda").manual_seed(1)
Pa = torch.randn((a, R), dtype=torch.float64, device="cuda", generator=g)
Pb = torch.randn((b, R), dtype=torch.float64, device="cuda", generator=g)
Y = torch.randn((N, R), dtype=torch.float64, device="cuda", generator=g).T
for _ in range(3):
    out = decomp._kr_contract(Pa, Pb, Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    out = decomp._kr_contract(Pa, Pb, Y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("kr_contract a=%d b=%d R=%d N=%d: %.3f ms = %.1f TFLOP/s" % (a, b, R, N, ms, 2.0 * a * b * R * N / ms / 1e9))

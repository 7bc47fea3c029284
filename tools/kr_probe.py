"""Fused Khatri-Rao contraction vs the library route (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp
def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for a, b, R, N in [(50, 50, 100000, 127), (48, 45, 20000, 61), (40, 40, 8000, 60), (30, 30, 2000, 50), (72, 67, 130000, 127), (20, 20, 500, 40)]:
    Pa = torch.randn((a, R), dtype=torch.float64, device="cuda"); Pb = torch.randn((b, R), dtype=torch.float64, device="cuda")
    Y = torch.randn((N, R), dtype=torch.float64, device="cuda").T
    decomp._KR_FUSED = True; t1 = timeit(lambda: decomp._kr_contract(Pa, Pb, Y))
    decomp._KR_FUSED = False; t0 = timeit(lambda: decomp._kr_contract(Pa, Pb, Y))
    fl = 2.0 * a * b * R * N
    print("a=%d b=%d R=%d N=%d: fused %.3f ms (%.1f TFLOP/s), library route %.3f ms (%.1f)" % (a, b, R, N, t1, fl / t1 / 1e9, t0, fl / t0 / 1e9), flush=True)

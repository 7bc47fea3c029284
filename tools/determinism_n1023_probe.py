"""Bitwise repeatability of the N = 1024 register passes (dev tool): the
padded n = 1023 transform (one contiguous + two TMA-stored strided passes)
run 30 times; any differing element means a race in the tile/staging reuse."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import full
n = 1023
spec = fl.laplacian_spectrum(n, 3)
g = torch.Generator(device="cuda"); g.manual_seed(5)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda", generator=g)
ref = full.transform_full_padded(spec, x).clone()
bad = 0
for r in range(30):
    out = full.transform_full_padded(spec, x)
    d = int((out != ref).sum())
    bad += d != 0
    if d:
        print("run", r, "differing elements:", d, flush=True)
print("n1023 padded transform: %d of 30 runs differ" % bad, flush=True)

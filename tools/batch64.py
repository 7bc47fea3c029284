"""All 64 configs[4] problems at one n, sequential, one line per problem (dev tool)."""
import os, sys, time, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, spectral
n = int(sys.argv[1])
lo, hi = (int(v) for v in sys.argv[2].split(":")) if len(sys.argv) > 2 else (0, 64)
spec = spectral.laplacian_spectrum(n, 3)
batch._solve_one(0, n, spec, 1023)
t0 = time.perf_counter()
for i in range(lo, hi):
    r = batch._solve_one(i, n, spec, 1023)
    print(json.dumps(r), flush=True)
print("total %.1f s" % (time.perf_counter() - t0))

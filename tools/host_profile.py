"""cProfile of one configs[4] problem at n = 1023: where the HOST time goes (dev tool)."""
import os, sys, cProfile, pstats, io, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
batch.solve_batch(n, 1)
pr = cProfile.Profile()
pr.enable()
batch.solve_batch(n, 1)
torch.cuda.synchronize()
pr.disable()
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(28)
    print(s.getvalue()[:6000])

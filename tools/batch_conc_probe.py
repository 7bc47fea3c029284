"""configs[4] throughput vs concurrent problems per GPU (dev tool):
python tools/batch_conc_probe.py N COUNT C1,C2,..."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch
n, count = int(sys.argv[1]), int(sys.argv[2])
concs = [int(v) for v in sys.argv[3].split(",")]
batch.solve_batch(n, 1)  # warm-up
for c in concs:
    torch.cuda.reset_peak_memory_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs = batch.solve_batch(n, count, concurrency=c)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    its = [r["iterations"] for r in recs]
    print("n=%d count=%d conc=%d: %.2f s, %.3f solves/s, peak %.1f GB, its %s, all converged %s"
          % (n, count, c, t, count / t, torch.cuda.max_memory_allocated() / 1e9, its,
             all(r["converged"] for r in recs)), flush=True)

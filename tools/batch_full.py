"""The stated configs[4] batch at one n in chunks, one JSON record per problem as
chunks finish (dev tool): python tools/batch_full.py N [count] [concurrency] [chunk]"""
import os, sys, time, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch
n = int(sys.argv[1])
count = int(sys.argv[2]) if len(sys.argv) > 2 else 64
conc = int(sys.argv[3]) if len(sys.argv) > 3 else 4
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 8
batch.solve_batch(n, 1)  # warm-up (module loads, first allocations)
torch.cuda.synchronize()
t0 = time.perf_counter()
done = conv = 0
for lo in range(0, count, chunk):
    recs = batch.solve_batch(n, count, concurrency=conc, indices=range(lo, min(count, lo + chunk)))
    for r in recs:
        print(json.dumps(r), flush=True)
        done += 1
        conv += bool(r.get("converged"))
    print("# %d problems, %d converged, %.1f s so far, peak memory %.1f GB" % (
        done, conv, time.perf_counter() - t0, torch.cuda.max_memory_allocated() / 1e9), flush=True)
dt = time.perf_counter() - t0
print("# n=%d: %d problems (%d converged) in %.1f s = %.4f solves/s, concurrency %d" % (n, done, conv, dt, done / dt, conc))

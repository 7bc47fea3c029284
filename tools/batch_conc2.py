"""configs[4] concurrency without the linalg lock, SVD driver selectable (dev tool):
python tools/batch_conc2.py N COUNT DRIVER C1,C2 [lock]"""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, decomp
n, count, driver = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
concs = [int(v) for v in sys.argv[4].split(",")]
lock = len(sys.argv) > 5 and sys.argv[5] == "lock"
if driver != "default":
    def _svd(m, compute_uv=True):
        if compute_uv:
            return decomp._la(torch.linalg.svd, m, full_matrices=False, driver=driver)
        return decomp._la(torch.linalg.svd, m, full_matrices=False, driver=driver)[1]
    decomp._svd = _svd
batch.solve_batch(n, 1)
for c in concs:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        recs = batch.solve_batch(n, count, concurrency=c, serial_linalg=lock)
        t = time.perf_counter() - t0
        print("n=%d count=%d driver=%s conc=%d lock=%s: %.1f s, %.3f solves/s, its %s, errors %s" % (
            n, count, driver, c, lock, t, count / t, [r["iterations"] for r in recs],
            [r.get("error") for r in recs if r.get("error")]), flush=True)
    except Exception as e:
        print("conc=%d FAILED %s: %s" % (c, type(e).__name__, str(e)[:300]), flush=True)

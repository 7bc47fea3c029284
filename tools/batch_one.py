"""Solve single configs[4] problems (dev tool): python tools/batch_one.py N i [i ...]"""
import os, sys, time, traceback, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import batch, spectral
n = int(sys.argv[1])
spec = spectral.laplacian_spectrum(n, 3)
for i in [int(v) for v in sys.argv[2:]]:
    y, cfg = batch.problem(i, n)
    t0 = time.perf_counter()
    try:
        u, rep = batch.solve_control_large(y, cfg, spec)
        torch.cuda.synchronize()
        print("n=%d problem %d alpha %.4f beta %.3e: %d its conv %s rank %d res %s %.2f s" % (
            n, i, cfg.alpha, cfg.beta, rep.iterations, rep.converged, u.rank,
            ["%.2e" % r for r in rep.residuals], time.perf_counter() - t0), flush=True)
    except Exception as e:
        print("n=%d problem %d alpha %.4f beta %.3e: FAILED %s: %s" % (n, i, cfg.alpha, cfg.beta, type(e).__name__,
                                                                     str(e)[:200]), flush=True)
        traceback.print_exc(limit=-4)

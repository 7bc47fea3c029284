"""configs[4] throughput with P worker processes sharing one GPU (dev tool):
python tools/batch_procs.py N COUNT P1,P2,..."""
import json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    n, count, rank, world = (int(v) for v in sys.argv[2:6])
    import torch
    from paper_1809_01971_b200 import batch
    recs = batch.solve_batch(n, count, rank, world)
    print(json.dumps(recs), flush=True)
    sys.exit(0)
n, count = int(sys.argv[1]), int(sys.argv[2])
# warm the page cache / module load once
subprocess.run([sys.executable, __file__, "--child", str(n), "1", "0", "1"], capture_output=True)
for P in [int(v) for v in sys.argv[3].split(",")]:
    t0 = time.perf_counter()
    procs = [subprocess.Popen([sys.executable, __file__, "--child", str(n), str(count), str(r), str(P)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(P)]
    outs = [p.communicate() for p in procs]
    t = time.perf_counter() - t0
    recs = []
    for (o, e), p in zip(outs, procs):
        if p.returncode:
            print("worker failed:", e[-800:])
        else:
            recs += json.loads(o.strip().splitlines()[-1])
    its = sorted((r["problem"], r["iterations"], r["converged"]) for r in recs)
    print("n=%d count=%d procs=%d: %.1f s (incl. startup), %.3f solves/s, solved %d, its %s" % (
        n, count, P, t, len(recs) / t, len(recs), [i for _, i, _ in its]), flush=True)

"""Kernel-boundary cost of the 5-pass apply (dev tool): per-pass repeats vs the
pass sequence vs FullOperator.__call__, same process."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import full, spectral
from paper_1809_01971_b200.fracop import CoreFunctionKind
n = 511
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
passes = op.passes(x, y)
def t(fn, reps):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
def seq():
    for _, a in passes: full.run_pass(a)
for reps in (20, 100):
    per = [t(lambda a=a: full.run_pass(a), reps) for _, a in passes]
    print("reps %d: per-pass %s sum %.3f | sequence %.3f | apply %.3f" % (reps, ["%.3f" % v for v in per], sum(per),
          t(seq, reps), t(lambda: op(x, out=y), reps)), flush=True)
# one sequence with events between passes
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(passes) + 1)]
for _ in range(3): seq()
torch.cuda.synchronize()
evs[0].record()
for i, (_, a) in enumerate(passes):
    full.run_pass(a); evs[i + 1].record()
torch.cuda.synchronize()
print("in-sequence pass times", ["%.3f" % evs[i].elapsed_time(evs[i + 1]) for i in range(len(passes))])

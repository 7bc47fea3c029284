"""In-situ Khatri-Rao contraction shapes of configs[1] with both routes timed (dev tool)."""
import os, sys, collections, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp
hist = collections.defaultdict(lambda: [0, 0.0, 0.0])
orig = decomp._kr_contract
def ev(f):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = f(); b.record(); torch.cuda.synchronize()
    return out, a.elapsed_time(b)
def wrapped(Pa, Pb, Y):
    decomp._KR_FUSED = False; _, t0 = ev(lambda: orig(Pa, Pb, Y))
    decomp._KR_FUSED = True; out, t1 = ev(lambda: orig(Pa, Pb, Y))
    h = hist[(Pa.shape[0], Pb.shape[0], Pa.shape[1], Y.shape[1], Y.stride(0) == 1)]
    h[0] += 1; h[1] += t1; h[2] += t0
    return out
decomp._kr_contract = wrapped
n = 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
fl.solve_control(y, cfg, spec)
hist.clear()
fl.solve_control(y, cfg, spec)
tf = tl = 0.0
for k, (c, t1, t0) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:30]:
    print("a=%d b=%d R=%d N=%d rmajor=%s: %3d calls fused %.3f ms  library %.3f ms" % (*k, c, t1 / c, t0 / c))
for k, (c, t1, t0) in hist.items():
    tf += t1; tl += t0
print("total fused %.1f ms, library %.1f ms" % (tf, tl))

"""configs[3] solve at n=1023 on one GPU, dense vs padded spectral layout (dev tool)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import fullsolve, full
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
spec = fl.laplacian_spectrum(n, 3)
cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, residual_tol=1e-8)
y = full.cp_dense(fl.gaussian_bumps(n, 3, 16, seed=3))
A, P = fullsolve.control_cores(cfg, spec)
Ap, Pp = full.to_padded(A), full.to_padded(P)
def tm(fn):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return out, time.perf_counter() - t0
(u1, r1), t1 = tm(lambda: fullsolve.solve_control_full(y, cfg, spec, cores=(A, P)))
(u2, r2), t2 = tm(lambda: fullsolve.solve_control_full(y, cfg, spec, cores=(Ap, Pp)))
rel = float(torch.linalg.vector_norm(u1 - u2) / torch.linalg.vector_norm(u1))
print("n=%d dense %.3f s (%d its) | padded %.3f s (%d its) | rel diff %.2e" % (n, t1, r1.iterations, t2, r2.iterations, rel))
# parts
import paper_1809_01971_b200._lib as L
def ev(fn):
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); out = fn(); e.record(); torch.cuda.synchronize(); return out, s.elapsed_time(e)
for tag, (AA, PP) in (("dense", (A, P)), ("padded", (Ap, Pp))):
    padded = AA.shape[-1] != n
    bh, t_f = ev(lambda: full.transform_full_padded(spec, y) if padded else full.transform_full(spec, y))
    xh = torch.empty_like(bh); r = torch.empty_like(bh); p = torch.empty_like(bh)
    hist = torch.zeros(101, dtype=torch.float64, device="cuda"); st = torch.zeros(4, dtype=torch.int32, device="cuda")
    _, t_p = ev(lambda: L.call("fl_pcg_spectral", L.ptr(bh), L.ptr(xh), L.ptr(r), L.ptr(p), L.ptr(AA), L.ptr(PP), bh.numel(),
                               1e-8, 100, L.ptr(hist), L.ptr(st), L.stream_ptr()))
    _, t_b = ev(lambda: full.transform_full_from_padded(spec, xh) if padded else full.transform_full(spec, xh))
    print(tag, "fwd %.1f ms, pcg %.1f ms (%d its), inv %.1f ms" % (t_f, t_p, int(st[0]), t_b))

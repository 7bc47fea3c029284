"""torch.profiler view of configs[1] (dev tool): GPU busy time vs wall, top kernels."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from torch.profiler import profile, ProfilerActivity
n = int(sys.argv[1]) if len(sys.argv) > 1 else 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
fl.solve_control(y, cfg, spec)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    fl.solve_control(y, cfg, spec)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = prof.key_averages()
gpu_total = sum(e.self_device_time_total for e in ev) / 1e6
print("wall %.3f s, summed GPU kernel time %.3f s" % (wall, gpu_total))
print(ev.table(sort_by="self_device_time_total", row_limit=25, max_name_column_width=60))

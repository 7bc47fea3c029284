"""Pivoted small Jacobi timing for library variants: python tools/jacobi_lpp.py LIB... (dev tool)"""
import os, subprocess, sys
if len(sys.argv) > 2:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib])
    sys.exit(0)
os.environ["FL_LIB_OVERRIDE"] = os.path.abspath(sys.argv[1])
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_1809_01971_b200 import decomp
rng = np.random.default_rng(0)
out = []
for k, r in [(127, 127), (127, 60), (96, 96), (90, 50), (64, 64), (48, 30), (30, 30)]:
    X = rng.standard_normal((k, r)) * np.logspace(0, -12, r)
    Y = rng.standard_normal((r, 3000))
    M = torch.tensor(X @ Y, device="cuda")
    R = decomp.qr_r_wide([M])[0]
    T = R.T.contiguous()
    decomp.svd_left_pivoted(T); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        U, S = decomp.svd_left_pivoted(T)
    b.record(); torch.cuda.synchronize()
    want = np.linalg.svd(M.cpu().numpy(), compute_uv=False)
    err = float(np.abs(S.cpu().numpy() - want).max() / want[0])
    out.append("k=%d r=%d: %.3f ms (err %.0e)" % (k, r, a.elapsed_time(b) / 10, err))
print(os.path.basename(sys.argv[1]), " | ".join(out), flush=True)

"""k_jacobi_small timing for library variants (dev tool): python tools/jsmall_var.py LIB..."""
import os, subprocess, sys
if len(sys.argv) > 2:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib])
    sys.exit(0)
os.environ["FL_LIB_OVERRIDE"] = os.path.abspath(sys.argv[1])
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np
from paper_1809_01971_b200 import decomp
rng = np.random.default_rng(0)
out = []
for grade in (0.0, 18.0):
    k = 127
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k))); Q2, _ = np.linalg.qr(rng.standard_normal((k, k)))
    sv = 10.0 ** (-grade * np.arange(k) / (k - 1)) if grade else np.linspace(1, 0.5, k)
    A = (Q1 * sv) @ Q2.T
    At = torch.tensor(A[None], device="cuda")
    decomp.svd_batched(At, right=False); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        U, S, _ = decomp.svd_batched(At, right=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5 * 1e3
    err = float(np.abs(S[0].cpu().numpy() - np.linalg.svd(A, compute_uv=False)).max())
    out.append("grade %g: %.3f ms sv err %.1e" % (grade, dt, err))
print(os.path.basename(sys.argv[1]), " | ".join(out), flush=True)

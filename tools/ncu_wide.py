"""One batched wide left-SVD (five 127 x 2039 graded factors: the shape of c2t's
factor SVDs at configs[1]) for ncu captures of k_tsqr / k_jacobi_multi (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import decomp

rng = np.random.default_rng(3)
k, m = 127, 2039
mats = []
for i in range(5):
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, k)))
    sv = 10.0 ** (-16.0 * np.arange(k) / (k - 1))
    mats.append(torch.tensor((Q1 * sv) @ Q2.T, device="cuda"))
for _ in range(3):
    res = decomp.left_sv_wide(mats, vectors=[True, True, True, False, False])
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    res = decomp.left_sv_wide(mats, vectors=[True, True, True, False, False])
b.record(); torch.cuda.synchronize()
want = np.linalg.svd(mats[0].cpu().numpy(), compute_uv=False)
print("batch of 5 (127 x 2039): %.3f ms per call, sv err %.1e" % (a.elapsed_time(b) / 10,
      float(np.abs(res[0][1].cpu().numpy() - want).max() / want[0])))

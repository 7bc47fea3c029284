"""One-CTA Jacobi SVD timing for small square factors (dev tool)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200.decomp import svd_batched

rng = np.random.default_rng(0)
for k in (8, 16, 36, 64):
    for kind in ("random", "graded"):
        A = rng.standard_normal((k, k))
        if kind == "graded":
            A = A @ np.diag(np.logspace(0, -15, k)) @ np.linalg.qr(rng.standard_normal((k, k)))[0]
        M = torch.tensor(A, device="cuda")[None]
        for _ in range(3):
            svd_batched(M, right=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            svd_batched(M, right=False)
        e1.record()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            torch.linalg.svd(M[0], full_matrices=False)
        torch.cuda.synchronize()
        print("k=%d %s: jacobi %.3f ms, library %.3f ms" % (k, kind, e0.elapsed_time(e1) / 20,
                                                           (time.perf_counter() - t0) / 20 * 1e3), flush=True)
# accuracy of the last (graded, k = 64) case against numpy
U, S, _ = svd_batched(M, right=False)
s_ref = np.linalg.svd(A, compute_uv=False)
print("graded k=64: max rel sigma err %.2e, orthogonality %.2e" % (
    float(np.max(np.abs(S[0].cpu().numpy() - s_ref) / s_ref)),
    float(np.max(np.abs(U[0].cpu().numpy().T @ U[0].cpu().numpy() - np.eye(64))))), flush=True)

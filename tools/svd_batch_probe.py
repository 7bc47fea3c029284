"""Batched slice-SVD cost (t2c) on the device vs host (dev tool)."""
import time
import torch

for r in (32, 48, 64, 96):
    A = torch.randn(r, r, r, dtype=torch.float64, device="cuda")
    for label, X in (("gpu", A), ("cpu", A.cpu())):
        for _ in range(2):
            torch.linalg.svd(X, full_matrices=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            U, S, V = torch.linalg.svd(X, full_matrices=False)
        torch.cuda.synchronize()
        print("r=%d %s svd %.1f ms" % (r, label, (time.perf_counter() - t0) / 3 * 1e3))
    G = A.transpose(1, 2) @ A
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        torch.linalg.eigh(G)
    torch.cuda.synchronize()
    print("r=%d gpu eigh(gram) %.1f ms" % (r, (time.perf_counter() - t0) / 3 * 1e3))

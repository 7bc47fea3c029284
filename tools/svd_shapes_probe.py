"""SVD routes for the shapes of c2t/t2c at large n (dev tool)."""
import time
import torch


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def qr_route(M):
    _, R = torch.linalg.qr(M.T)
    return torch.linalg.svd(R.T)


for shape in [(60, 500000), (60, 50000), (60, 3600), (200, 50000), (100, 10000)]:
    M = torch.randn(*shape, dtype=torch.float64, device="cuda")
    a = t(lambda: torch.linalg.svd(M, full_matrices=False))
    b = t(lambda: qr_route(M))
    c = t(lambda: torch.linalg.svd(M, full_matrices=False, driver="gesvdj"))
    print(shape, "svd %.1f ms  qr-route %.1f ms  gesvdj %.1f ms" % (a, b, c))
for r in (48, 64, 96):
    A = torch.randn(r, r, r, dtype=torch.float64, device="cuda")
    for drv in ("gesvd", "gesvdj", "gesvda"):
        try:
            print("batch %d^3 %s %.1f ms" % (r, drv, t(lambda: torch.linalg.svd(A, full_matrices=False, driver=drv))))
        except Exception as e:
            print("batch", r, drv, "failed", str(e)[:80])

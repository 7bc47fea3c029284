import os, sys, torch, numpy as np
def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
rng = np.random.default_rng(0)
for k in (144, 176, 208, 256, 320, 432):
    Q1, _ = np.linalg.qr(rng.standard_normal((k, k))); Q2, _ = np.linalg.qr(rng.standard_normal((k, k)))
    A = torch.tensor(np.triu((Q1 * 10.0 ** (-16 * np.arange(k) / (k - 1))) @ Q2.T), device="cuda")
    out = ["k=%d" % k]
    for drv in (None, "gesvd", "gesvdj", "gesvda"):
        try:
            out.append("%s %.2f" % (drv, timeit(lambda: torch.linalg.svd(A, full_matrices=False, driver=drv))))
        except Exception as e:
            out.append("%s fail" % drv)
    out.append("eigh %.2f" % timeit(lambda: torch.linalg.eigh(A @ A.T)))
    out.append("qr %.2f" % timeit(lambda: torch.linalg.qr(A)))
    print(" | ".join(out), flush=True)

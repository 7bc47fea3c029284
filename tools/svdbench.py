import time, torch
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); s = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - s) / reps * 1e3
for shape in [(127, 127), (127, 1000), (127, 20000), (127, 130000), (40, 40)]:
    A = torch.randn(*shape, dtype=torch.float64, device="cuda")
    r = {}
    for drv in (None, "gesvd", "gesvdj", "gesvda"):
        try: r[str(drv)] = "%.2f" % t(lambda: torch.linalg.svd(A, full_matrices=False, driver=drv))
        except Exception as e: r[str(drv)] = "err"
    G = A @ A.T
    r["eigh(AAT)"] = "%.2f" % t(lambda: torch.linalg.eigh(A @ A.T))
    r["qr(AT)"] = "%.2f" % t(lambda: torch.linalg.qr(A.T))
    r["svdvals"] = "%.2f" % t(lambda: torch.linalg.svdvals(A))
    print(shape, r)

"""PCIe copy rates with pinned host memory (dev tool): H2D, D2H, both at once."""
import torch

nb = 1067462648 // 8
h1 = torch.empty(nb, dtype=torch.float64).pin_memory()
h2 = torch.empty(nb, dtype=torch.float64).pin_memory()
d1 = torch.empty(nb, dtype=torch.float64, device="cuda")
d2 = torch.empty(nb, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()


gb = nb * 8 / 1e9
a = t(lambda: d1.copy_(h1, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
c = t(both)
print("H2D %.2f ms (%.1f GB/s)  D2H %.2f ms (%.1f GB/s)  both %.2f ms (%.1f GB/s each)" % (a, gb / a * 1e3, b, gb / b * 1e3, c, gb / c * 1e3))

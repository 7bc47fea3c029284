"""Calibration (dev tool, not product): cuFFT batched complex FFT throughput
on the same element count as one DST pass at n=511 (two real lines packed
per complex line), for comparison with k_dst_fft."""
import torch


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


dof = 511 ** 3
for L in (512, 256, 1024):
    B = dof // (2 * L)
    x = torch.randn(B, L, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    ms = t(lambda: torch.fft.fft(x, dim=1, out=y))
    print("c2c L=%d batch=%d: %.3f ms  %.0f GB/s (read+write)" % (L, B, ms, 2 * x.numel() * 16 / ms / 1e6))
    xs = torch.randn(B, 511, 2, dtype=torch.float64, device="cuda")
    del x, y
# strided (mode-1 like): FFT along dim 1 of (511, 512, 511) complex? use real-to-complex on the middle axis
xr = torch.randn(511, 1024, 256, dtype=torch.float64, device="cuda")
ms = t(lambda: torch.fft.rfft(xr, dim=1))
print("r2c middle axis 1024 (511x1024x256): %.3f ms" % ms)

"""Compute-side ceiling of the DST kernel (dev tool): per-DoF time of one
pass on an L2-resident tensor vs an HBM-sized one, same shapes otherwise."""
import torch
from paper_1809_01971_b200 import _lib

n = 511
st = _lib.stream_ptr()


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for label, outer_l2, outer_big in (("contig", 20480, 511 * 511), ("strided", 20, 511)):
    for outer in (outer_l2, outer_big):
        if label == "contig":
            shape, args = (outer, n), (outer, n, 1)
        else:
            shape, args = (outer, n, 512), (outer, n, 512)
        x = torch.randn(*shape, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        ms = t(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), *args, 1.0, st))
        dof = x.numel()
        print("%-8s %9d DoF  %.4f ms  %.3f ns/kDoF  %6.0f GB/s-equiv (16 B/DoF)  [%.1f MB]"
              % (label, dof, ms, ms * 1e6 / dof * 1e3 / 1e3, 16 * dof / ms / 1e6, 8 * dof / 1e6))
        # also the fused pass
        if label == "contig":
            c = torch.rand_like(x)
            ms = t(lambda: _lib.call("fl_dst1_core", _lib.ptr(x), _lib.ptr(y), _lib.ptr(c), outer, n, 1, 1.0, st))
            print("%-8s %9d DoF  %.4f ms  fused  %6.0f GB/s-equiv (24 B/DoF)" % ("core", dof, ms, 24 * dof / ms / 1e6))
        del x, y

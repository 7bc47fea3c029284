"""Quick per-pass timing of the DST kernels (development tool)."""
import sys, time
import torch
from paper_1809_01971_b200 import _lib, spectral, full
from paper_1809_01971_b200.fracop import CoreFunctionKind

def t_events(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3

n = int(sys.argv[1]) if len(sys.argv) > 1 else 511
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
B = x.numel() * 8
st = _lib.stream_ptr()
for name, (outer, inner) in {"mode0": (1, n*n), "mode1": (n, n), "mode2": (n*n, 1)}.items():
    dt = t_events(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), outer, n, inner, 1.0, st))
    print(f"{name}: {dt*1e3:.3f} ms  {2*B/dt/1e9:.0f} GB/s")
spec = spectral.laplacian_spectrum(n, 3)
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec)
core = op.core
dt = t_events(lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), 0, n, 1, 1.0, st))
dt = t_events(lambda: op(x, out=y))
print(f"apply: {dt*1e3:.3f} ms  {x.numel()/dt/1e9:.2f} GDoF/s  eff {(10*B+B)/dt/1e9:.0f} GB/s (11 B-units)")
dt = t_events(lambda: y.copy_(x))
print(f"copy: {dt*1e3:.3f} ms {2*B/dt/1e9:.0f} GB/s")

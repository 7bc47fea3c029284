"""Per-pass timing of the padded full apply (dev tool): each launch of
FullOperator.passes() timed alone (20 reps after warm-up), n from argv."""
import sys
import torch
from paper_1809_01971_b200 import _lib, spectral, full
from paper_1809_01971_b200.fracop import CoreFunctionKind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 511
spec = spectral.laplacian_spectrum(n, 3)
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
st = _lib.stream_ptr()


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


B = 16 * n ** 3 / 1e9
tot = 0.0
for i, (name, a) in enumerate(op.passes(x, y)):
    ms = t(lambda: full.run_pass(a, st))
    tot += ms
    gb = (1.5 if "core" in name else 1.0) * B / ms * 1e3
    print("pass %d %-15s %.3f ms  %5.0f GB/s" % (i, name, ms, gb))
print("sum %.3f ms; op() %.3f ms" % (tot, t(lambda: op(x, out=y))))

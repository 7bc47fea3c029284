"""Per-pass timing and correctness of the padded n=511 apply (dev tool).

Env FL_REG=1 selects the register-resident N=512 kernels (dst_reg.cuh).
Checks the full apply against the CPU oracle (scipy DST-I) at n=511.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1809_01971_b200 import full, spectral  # noqa: E402
from paper_1809_01971_b200.fracop import CoreFunctionKind  # noqa: E402

n = int(os.environ.get("PROBE_N", "511"))
check = os.environ.get("PROBE_CHECK", "1") == "1"
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda", generator=g)
y = torch.empty_like(x)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


B = 16 * n ** 3 / 1e9
out = {"FL_REG": os.environ.get("FL_REG", "0")}
for k, (name, a) in enumerate(op.passes(x, y)):
    ms = t(lambda: full.run_pass(a))
    fac = 1.5 if "core" in name else 1.0
    out["%d:%s" % (k, name)] = "%.3f ms (%.0f GB/s)" % (ms, fac * B / ms * 1e3)
ms = t(lambda: op(x, out=y), reps=50)
out["apply"] = "%.3f ms (%.1f GDoF/s)" % (ms, n ** 3 / ms / 1e6)
print(out, flush=True)
if check:
    got = op(x, out=y).cpu().numpy()
    t0 = time.time()
    core = oracle.dense_core("g1", [oracle.laplacian_eigenvalues(n)] * 3, 0.5)
    want = oracle.apply_full(core, x.cpu().numpy())
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print("apply rel err vs oracle: %.3e (oracle %.1f s)" % (rel, time.time() - t0), flush=True)
    for name, a in op.passes(x, y):
        pass

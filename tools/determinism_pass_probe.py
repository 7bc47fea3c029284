"""Per-pass determinism of the lane apply (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import full, spectral
from paper_1809_01971_b200.fracop import CoreFunctionKind
n = 511
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
g = torch.Generator(device="cuda"); g.manual_seed(3)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda", generator=g)
y = torch.empty_like(x)
passes = op.passes(x, y)
# state before each pass
states = []
for name, a in passes:
    states.append((op.work.clone(), y.clone()))
    full.run_pass(a)
torch.cuda.synchronize()
for k, (name, a) in enumerate(passes):
    outs = []
    for r in range(6):
        op.work.copy_(states[k][0]); y.copy_(states[k][1])
        full.run_pass(a)
        torch.cuda.synchronize()
        outs.append((op.work.clone(), y.clone()))
    diffs = [int((o[0] != outs[0][0]).sum() + (o[1] != outs[0][1]).sum()) for o in outs[1:]]
    print(k, name, "differing elements vs first run:", diffs, flush=True)

"""Race detector (dev tool): the apply is deterministic, so repeated runs on the
same input must agree bit for bit; also each pass of the pass list."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01971_b200 import full, spectral
from paper_1809_01971_b200.fracop import CoreFunctionKind
n = 511
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
g = torch.Generator(device="cuda"); g.manual_seed(3)
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda", generator=g)
ref = op(x).clone()
bad = 0
for r in range(reps):
    y = op(x)
    if not torch.equal(y, ref):
        bad += 1
        d = (y != ref).nonzero()
        print("run %d: %d elements differ, first %s" % (r, d.shape[0], d[:3].tolist()), flush=True)
print("apply: %d of %d runs differ" % (bad, reps), flush=True)
# fl_apply_full_padded (non-lane operator) too, and in-place
nat = full.FullOperator(op.spectrum, op.core.contiguous(), padded=True, lanes=False)
ref2 = nat(x).clone()
bad2 = sum(0 if torch.equal(nat(x), ref2) else 1 for _ in range(reps // 2))
z = x.clone(); op(z, out=z)
print("padded: %d differ; in-place == out-of-place: %s" % (bad2, torch.equal(z, ref)), flush=True)

"""Locate TMA-store mismatches on small strided n=511 passes (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1809_01971_b200 import full, _lib, spectral
from paper_1809_01971_b200.fracop import CoreFunctionKind
n = 511; P = 512

def report(tag, got, want):
    bad = np.abs(got - want) > 1e-10 * np.abs(want).max()
    print(tag, "bad fraction %.4f" % bad.mean(), flush=True)
    if bad.any():
        idx = np.argwhere(bad)
        print("  first bad", idx[:6].tolist(), "axes any:", [np.unique(idx[:, k])[:12].tolist() for k in range(idx.shape[1])])

for blocks in (2, 5):
    x = torch.randn(blocks, n, P, dtype=torch.float64, device="cuda")
    want = oracle.dst(x.cpu().numpy(), axis=1)
    lay = (n * P, P, 0, 0)
    full.run_pass((_lib.ptr(x), _lib.ptr(x), None, n, 0, blocks, 1, P, lay, lay, 1.0))
    torch.cuda.synchronize()
    report("mode1 in-place blocks=%d" % blocks, x.cpu().numpy(), want)
# mode-0 strided with groups (like the fused pass layout, no core): [511][g][512]
for g in (1, 3):
    x = torch.randn(n, g, P, dtype=torch.float64, device="cuda")
    want = oracle.dst(x.cpu().numpy(), axis=0)
    lay = (0, g * P, P, 0)
    y = torch.zeros_like(x)
    full.run_pass((_lib.ptr(x), _lib.ptr(y), None, n, 0, 1, g, P, lay, lay, 1.0))
    torch.cuda.synchronize()
    report("mode0 groups=%d" % g, y.cpu().numpy(), want)
# fused lanes pass
for dims in ((511, 511), (511, 3, 511)):
    spec = spectral.EigenSpectrum(tuple(spectral.laplacian_mode(m) for m in dims))
    op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec)
    x = torch.randn(dims, dtype=torch.float64, device="cuda")
    core = op.core.cpu().numpy()
    want = oracle.dst(core * oracle.dst(x.cpu().numpy(), axis=0), axis=0)
    g = dims[1] if len(dims) == 3 else 1
    w = torch.zeros((511, g, 512), dtype=torch.float64, device="cuda")
    w[..., :511] = x.reshape(511, g, 511)
    full.run_pass(("lanes0", _lib.ptr(w), _lib.ptr(w), _lib.ptr(op.core_l), g, 1.0))
    torch.cuda.synchronize()
    report("fused %s" % (dims,), w[..., :511].reshape(dims).cpu().numpy(), want)

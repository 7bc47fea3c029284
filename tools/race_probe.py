"""Repeat the n=511 many-tiles strided pass to expose races (dev tool)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1809_01971_b200 import full, _lib
n, P = 511, 512
bad = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    torch.cuda.synchronize()
    blocks = 37 if trial % 2 == 0 else 40
    inplace = trial % 3 == 0
    g = torch.Generator(device="cuda"); g.manual_seed(trial)
    x = torch.randn((blocks, n, P), dtype=torch.float64, device="cuda", generator=g)
    want = oracle.dst(x.cpu().numpy(), axis=1)
    y = x if inplace else torch.full_like(x, 7.0)
    lay = (n * P, P, 0, 0)
    full.run_pass((_lib.ptr(x), _lib.ptr(y), None, n, 0, blocks, 1, P, lay, lay, 1.0))
    got = y.cpu().numpy()
    err = np.abs(got - want) > 1e-10 * np.abs(want).max()
    if err.any():
        bad += 1
        idx = np.argwhere(err)
        print("trial %d blocks %d inplace %d: %d bad, blocks %s rows %s cols %s" % (
            trial, blocks, inplace, len(idx), np.unique(idx[:, 0])[:6], np.unique(idx[:, 1])[:8], np.unique(idx[:, 2])[:20]), flush=True)
        b0, c0 = idx[0, 0], idx[0, 2]
        colv = got[b0, :, c0]
        print("   bad col values: first %s; ==7: %d; zeros: %d" % (colv[:4], int((colv == 7.0).sum()), int((colv == 0).sum())))
        # is it the DST of another column / of the input?
        xin = x.cpu().numpy()
        for cand in range(max(0, c0 - 20), min(P, c0 + 20)):
            if np.allclose(colv, want[b0, :, cand], rtol=0, atol=1e-9 * np.abs(want).max()):
                print("   equals want column", cand)
        print("   max |bad - want| %.3e, |want| max %.3e" % (np.abs(colv - want[b0, :, c0]).max(), np.abs(want[b0, :, c0]).max()))
        rowsbad = np.where(err[b0, :, c0])[0]
        print("   rows bad in that column:", rowsbad[:10], "...", rowsbad[-5:], len(rowsbad))
print("bad trials", bad, flush=True)

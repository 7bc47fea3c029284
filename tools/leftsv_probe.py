"""_left_sv / _pick_ranks shapes of configs[1] and the QR + Jacobi route on
the real matrices (dev tool).  Saves a few sample matrices to gpurun_out/."""
import os, sys, time, collections, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp

shapes = collections.Counter()
samples = []
orig = decomp._left_sv
orig_svd = decomp._svd


def tm(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return out, time.perf_counter() - t0


stats = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])


def left_sv(M, r):
    n, m = M.shape
    k = min(n, m)
    out, t_lib = tm(lambda: orig(M, r))
    if 64 < k <= 128:
        key = "%dx%d" % (n, min(m, 10 ** 9))
        shapes[(n, m)] += 1
        def route():
            R = torch.linalg.qr(M.T if n <= m else M, mode="r")[1]
            X = R.T.contiguous() if n <= m else R.contiguous()
            U, s, _ = decomp.svd_batched(X[None], right=False)
            return U[0], s[0]
        (U2, s2), t_new = tm(route)
        U1, s1, _ = torch.linalg.svd(M, full_matrices=False)
        err_s = float(((s2 - s1).abs() / s1[0]).max())
        st = stats["left_sv k=%d" % k]
        st[0] += 1; st[1] += t_lib; st[2] += t_new; st[3] = max(st[3], err_s)
        if len(samples) < 6 and m >= 1000:
            samples.append(M.cpu().numpy())
    return out


def svd(M, compute_uv=True):
    out, t = tm(lambda: orig_svd(M, compute_uv))
    st = stats["_svd %s uv=%d" % ("x".join(str(v) for v in M.shape) if M.numel() < 0 else "k=%d" % min(M.shape), compute_uv)]
    st[0] += 1; st[1] += t
    return out


decomp._left_sv = left_sv
decomp._svd = svd
n = int(sys.argv[1]) if len(sys.argv) > 1 else 127
spec = fl.laplacian_spectrum(n, 3)
y = fl.gaussian_bumps(n, 3, 8, seed=11)
cfg = fl.SolverConfig(alpha=0.5, beta=1e-2, eps=1e-8, precond_rank=6, residual_tol=1e-6, k_max=60)
u, rep = fl.solve_control(y, cfg, spec)
print("its", rep.iterations, "rank", u.rank)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print("%-28s calls %4d lib %.3f s  qr+jacobi %.3f s  max sv err %.1e" % (k, v[0], v[1], v[2], v[3]))
print("shapes (n, m):", sorted(shapes.items(), key=lambda kv: -kv[1])[:20])
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/leftsv_samples.npz", *samples)

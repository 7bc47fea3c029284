"""Where the time of a configs[4]-style canonical solve goes (dev tool):
wraps trunc / apply / cp_norm with timers and rank logs, runs batch problem 0
at the sizes given on the command line."""
import os
import sys
import time
import collections
import torch
from paper_1809_01971_b200 import batch, decomp, fracop, solver, tensor

stats = collections.defaultdict(lambda: [0, 0.0])
log = []


def wrap(mod, name, label, rank_of=None):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        stats[label][0] += 1
        stats[label][1] += dt
        if rank_of is not None:
            log.append((label, rank_of(a, out), round(dt, 4)))
            if os.environ.get("FL_VERBOSE"):
                print("   ", log[-1], "mem %.1f GB" % (torch.cuda.max_memory_allocated() / 1e9), flush=True)
        return out
    setattr(mod, name, g)


rin = lambda a, out: (a[0].rank, getattr(out, "rank", None))
import os
if os.environ.get("FL_COMPRESS_MIN_N"):
    decomp._COMPRESS_MIN_N = int(os.environ["FL_COMPRESS_MIN_N"])
_pcg_orig = solver.cp_norm
wrap(solver, "trunc", "trunc", rin)
wrap(solver, "apply", "apply", lambda a, out: (a[1].rank, out.rank))
wrap(solver, "apply_compressed", "apply_compressed", lambda a, out: (a[1].rank, out.rank))
wrap(decomp, "_range_basis_gen", "  ._range_basis_gen")
wrap(decomp, "c2t", "c2t")
wrap(decomp, "t2c", "t2c", lambda a, out: (tuple(a[0].core.shape), out.rank))
wrap(decomp, "_merge_collinear", "merge", lambda a, out: (a[0].rank, out.rank))
wrap(decomp, "cp_norm", "cp_norm(decomp)", lambda a, out: (a[0].rank,))
wrap(decomp, "_pick_ranks", "pick_ranks")
wrap(decomp, "rhosvd", "rhosvd")
for nm in ("_svd", "_left_sv", "_kr_contract", "_cp_project_core", "_range_basis", "_complete_columns", "cp_normalize",
           "_collinear_pairs", "_kept_rank", "_fix_signs", "_core_cp_als", "_lift_tucker", "_compress_cp"):
    wrap(decomp, nm, "  ." + nm)
for n in [int(v) for v in sys.argv[1:]]:
    stats.clear()
    log.clear()
    t0 = time.perf_counter()
    y, cfg = batch.problem(int(os.environ.get("FL_PROBLEM", "0")), n)
    kind = fracop.CoreFunctionKind("g2", cfg.alpha, coeff_minus=float(cfg.beta), coeff_plus=float(cfg.gamma) / float(cfg.beta))
    spec = __import__("paper_1809_01971_b200").spectral.laplacian_spectrum(n, 3)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    core = batch.control_core_expsum(kind, spec, float(cfg.eps))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    pre_core = batch.preconditioner_coarse(kind, spec, cfg.precond_rank, max_level=int(os.environ.get("FL_MAXLEVEL", "1023")),
                                           interp=os.environ.get("FL_INTERP", "spectral"))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print("n=%d alpha=%.3f beta=%.2e core rank %d (%.2fs) pre rank %d (%.2fs)" % (n, cfg.alpha, cfg.beta, core.rank, t2 - t1, pre_core.rank, t3 - t2), flush=True)
    stats.clear(); log.clear()
    fun = fracop.LowRankOperator(fracop.DiagOpFunction(spec, kind, core, 0.0))
    pre = fracop.LowRankOperator(fracop.DiagOpFunction(spec, kind, pre_core, 0.0, reciprocal=True))
    u, rep = solver.pcg(fun, pre, y, None, cfg)
    torch.cuda.synchronize()
    print("  residuals", ["%.2e" % v for v in rep.residuals])
    print("  pcg: %d its, %.2fs, final rank %d, per-iter %s" % (rep.iterations, time.perf_counter() - t3, u.rank,
          [round(v, 2) for v in rep.iteration_seconds]), flush=True)
    for k, (c, t) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
        print("  %-16s %4d calls %8.3f s" % (k, c, t))
    for e in log[:60]:
        print("   ", e)

"""Generate golden input/output vectors by running the REFERENCE package.

Run in the build container, where /root/reference is mounted:
    python tests/golden/make_golden.py
Writes tests/golden/*.npz (committed).  The GPU box never reads
/root/reference; tests compare the CUDA path and the oracle against these.
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import fraclap  # noqa: E402
import oracles as ref_oracles  # noqa: E402  (the reference's own dense test oracles)
from fraclap import fracop as ref_fracop  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cp_arrays(prefix, cp, d):
    out = {prefix + "_w": cp.weights}
    for l in range(d):
        out["%s_f%d" % (prefix, l)] = cp.factors[l]
    return out


def spectral_cases():
    data = {}
    rng = np.random.default_rng(1)
    for n in (1, 2, 3, 5, 7, 9, 12, 15, 16, 31, 63, 127, 255, 511):
        x = rng.standard_normal((n, 4))
        data["x_%d" % n] = x
        data["dst_%d" % n] = fraclap.dst_apply(fraclap.laplacian_mode(n), x)
        data["lam_%d" % n] = fraclap.laplacian_mode(n).eigenvalues
    np.savez_compressed(os.path.join(OUT, "spectral.npz"), **data)


def core_cases():
    data = {}
    for d, n in ((2, 9), (3, 7)):
        spec = fraclap.laplacian_spectrum(n, d)
        for tag in ("g1", "g2", "g3", "g4"):
            for agg in ("sum-then-power", "power-then-sum"):
                kind = fraclap.CoreFunctionKind(tag, 0.5, aggregation=agg, coeff_minus=1.3, coeff_plus=0.7)
                for rec in (False, True):
                    key = "core_d%d_n%d_%s_%s_%d" % (d, n, tag, agg, int(rec))
                    data[key] = ref_fracop._dense_core(kind, spec, reciprocal=rec)
    # sinc cores (fracop.sinc_inverse_power)
    spec = fraclap.laplacian_spectrum(32, 2)
    for M in (4, 9, 16):
        op = fraclap.sinc_inverse_power(spec, 0.5, M)
        data.update(cp_arrays("sinc_M%d" % M, op.core, 2))
        data["sinc_M%d_err" % M] = np.array(op.achieved_error)
    np.savez_compressed(os.path.join(OUT, "cores.npz"), **data)


def apply_cases():
    """Canonical apply through the reference (fracop.apply) and the reference's
    dense full-format oracle (tests/oracles.py dense_apply)."""
    data = {}
    for d, n, tag, alpha in ((2, 16, "g2", 0.5), (2, 15, "g1", 1.0), (3, 9, "g2", 0.5), (3, 15, "g4", 0.5)):
        spec = fraclap.laplacian_spectrum(n, d)
        kind = fraclap.CoreFunctionKind(tag, alpha)
        op = fraclap.LowRankOperator(fraclap.build_core(kind, spec, fraclap.TruncationSpec(tolerance=1e-12)))
        w, f, dense = ref_oracles.random_cp_dense((n,) * d, 3, seed=40 + n + d)
        x = fraclap.CpTensor(w, f)
        y = op(x)
        key = "ap_d%d_n%d_%s" % (d, n, tag)
        data.update(cp_arrays(key + "_core", op.diag.core, d))
        data.update(cp_arrays(key + "_x", x, d))
        data[key + "_y"] = fraclap.cp_to_dense(y)
        data[key + "_rank"] = np.array(y.rank)
        # full-format: reference dense oracle with the exact core
        core = ref_oracles.dense_core(tag, n, d, alpha)
        data[key + "_full_y"] = ref_oracles.dense_apply(core, dense, n, d)
        data[key + "_full_x"] = dense
    np.savez_compressed(os.path.join(OUT, "apply.npz"), **data)


def trunc_cases():
    data = {}
    for i, (dims, rank, tol) in enumerate((((12, 11), 6, 1e-6), ((7, 6, 8), 6, 1e-6), ((8, 8, 8), 8, 1e-10),
                                          ((10, 10, 10), 12, 1e-8))):
        w, f, dense = ref_oracles.random_cp_dense(dims, rank, seed=500 + i, scale=2.0)
        x = fraclap.CpTensor(w, f)
        out = fraclap.trunc(x, fraclap.TruncationSpec(tolerance=tol))
        key = "tr%d" % i
        data.update(cp_arrays(key + "_x", x, len(dims)))
        data[key + "_tol"] = np.array(tol)
        data[key + "_dense"] = dense
        data[key + "_out"] = fraclap.cp_to_dense(out)
        data[key + "_rank"] = np.array(out.rank)
    np.savez_compressed(os.path.join(OUT, "trunc.npz"), **data)


def solve_cases():
    data = {}
    # reference tests' small 2D control solve and 3D state solve
    n, d = 12, 2
    spec = fraclap.laplacian_spectrum(n, d)
    y_d = fraclap.DesignFunction("two-bumps").evaluate((n,) * d)
    cfg = fraclap.SolverConfig(alpha=0.5, beta=1.0, gamma=1e-2, eps=1e-10, precond_rank=8,
                               residual_tol=1e-10, k_max=60)
    u, rep = fraclap.solve_control(y_d, cfg, spec)
    data["c2_u"] = fraclap.cp_to_dense(u)
    data["c2_iters"] = np.array(rep.iterations)
    data["c2_res"] = np.array(rep.residuals)
    # 3D canonical control solve, Gaussian-bump target (BASELINE configs[1] shape, small n)
    for n3, alpha in ((15, 0.5), (31, 0.25)):
        spec3 = fraclap.laplacian_spectrum(n3, 3)
        w, fs = _bumps(n3, 3, 8, seed=11)
        y3 = fraclap.CpTensor(w, fs)
        cfg3 = fraclap.SolverConfig(alpha=alpha, beta=1e-2, eps=1e-8, precond_rank=6,
                                    residual_tol=1e-6, k_max=60)
        t0 = time.time()
        u3, rep3 = fraclap.solve_control(y3, cfg3, spec3)
        key = "c3_n%d" % n3
        data.update(cp_arrays(key + "_y", y3, 3))
        data[key + "_alpha"] = np.array(alpha)
        data[key + "_u"] = fraclap.cp_to_dense(u3)
        data[key + "_iters"] = np.array(rep3.iterations)
        data[key + "_res"] = np.array(rep3.residuals)
        print("3D control n=%d: %d iterations, %.1fs" % (n3, rep3.iterations, time.time() - t0))
    n, d = 9, 3
    spec = fraclap.laplacian_spectrum(n, d)
    y_d = fraclap.DesignFunction("gaussian-bump").evaluate((n,) * d)
    cfg = fraclap.SolverConfig(alpha=0.5, beta=2.0, gamma=1e-3, eps=1e-10, precond_rank=8,
                               residual_tol=1e-9, k_max=60)
    data["s3_y"] = fraclap.cp_to_dense(fraclap.solve_state(y_d, cfg, spec))
    np.savez_compressed(os.path.join(OUT, "solve.npz"), **data)


def _bumps(n, d, count, seed):
    """Seeded Gaussian bumps (same draw order as oracle.gaussian_bumps)."""
    rng = np.random.default_rng(seed)
    x = (np.arange(n) + 1.0) / (n + 1.0)
    w = rng.standard_normal(count)
    factors = [np.empty((n, count)) for _ in range(d)]
    for k in range(count):
        for l in range(d):
            c = rng.uniform(0.2, 0.8)
            s = rng.uniform(0.05, 0.2)
            factors[l][:, k] = np.exp(-((x - c) ** 2) / (2.0 * s * s))
    return w, factors


def config0_case():
    """BASELINE configs[0]: 2D control solve, n=255, alpha=0.5, beta=1e-3,
    4 seeded Gaussian bumps, PCG tol 1e-8, reference rank-6 preconditioner."""
    n, d = 255, 2
    spec = fraclap.laplacian_spectrum(n, d)
    w, fs = _bumps(n, d, 4, seed=2024)
    y = fraclap.CpTensor(w, fs)
    cfg = fraclap.SolverConfig(alpha=0.5, beta=1e-3, eps=1e-10, precond_rank=6,
                               residual_tol=1e-8, k_max=100)
    t0 = time.time()
    u, rep = fraclap.solve_control(y, cfg, spec)
    dt = time.time() - t0
    data = cp_arrays("y", y, d)
    data.update(cp_arrays("u", u, d))
    data["iters"] = np.array(rep.iterations)
    data["res"] = np.array(rep.residuals)
    data["seconds"] = np.array(dt)
    print("config0: %d iterations, rank %d, %.1fs" % (rep.iterations, u.rank, dt))
    np.savez_compressed(os.path.join(OUT, "config0.npz"), **data)


def config1_alpha_cases():
    """BASELINE configs[1] at reduced n: 3D canonical control solves for every
    alpha the config names (0.25, 0.5, 0.75), beta=1e-2, rank-8 bump target,
    eps=1e-8, residual tol 1e-6 (reference solver.py:203-216).  n=15 and 31
    finish in minutes on the reference; n=63 was attempted (C1_SIZES=63
    C1_ALPHAS=0.5, round 2): the reference process died with SIGSEGV after
    ~25 minutes in this container (its all-pairs cosine matrices outgrow the
    host memory), and n=127 needs a 128 GiB all-pairs merge matrix: both are
    out of the reference's reach here.  One file per (n, alpha)
    so that cases can be generated in parallel processes."""
    sizes = [int(v) for v in os.environ.get("C1_SIZES", "15,31").split(",")]
    alphas = [float(v) for v in os.environ.get("C1_ALPHAS", "0.25,0.5,0.75").split(",")]
    for n3 in sizes:
        for alpha in alphas:
            spec3 = fraclap.laplacian_spectrum(n3, 3)
            w, fs = _bumps(n3, 3, 8, seed=11)
            y3 = fraclap.CpTensor(w, fs)
            cfg3 = fraclap.SolverConfig(alpha=alpha, beta=1e-2, eps=1e-8, precond_rank=6,
                                        residual_tol=1e-6, k_max=60)
            t0 = time.time()
            u3, rep3 = fraclap.solve_control(y3, cfg3, spec3)
            dt = time.time() - t0
            data = cp_arrays("y", y3, 3)
            data["alpha"] = np.array(alpha)
            data["u"] = fraclap.cp_to_dense(u3)
            data["u_rank"] = np.array(u3.rank)
            data["iters"] = np.array(rep3.iterations)
            data["res"] = np.array(rep3.residuals)
            data["seconds"] = np.array(dt)
            name = "c1_n%d_a%02d.npz" % (n3, int(round(alpha * 100)))
            np.savez_compressed(os.path.join(OUT, name), **data)
            print("configs[1] n=%d alpha=%g: %d iterations, rank %d, %.1fs" % (n3, alpha, rep3.iterations,
                                                                              u3.rank, dt), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["spectral", "core", "apply", "trunc", "solve", "config0", "config1"]
    for name in which:
        t0 = time.time()
        {"spectral": spectral_cases, "core": core_cases, "apply": apply_cases, "trunc": trunc_cases,
         "solve": solve_cases, "config0": config0_case, "config1": config1_alpha_cases}[name]()
        print(name, "%.1fs" % (time.time() - t0))

"""numpy/scipy restatement of the reference fraclap hot path (TEST ORACLE ONLY).

Each function cites the reference file:line (under
/root/reference/pkg/src/fraclap/) whose behaviour it restates.  Written
independently in plain numpy; pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np
import scipy.fft
from scipy.special import gammaln

TAGS = ("g1", "g2", "g3", "g4")


# ---------------------------------------------------------------------------
# spectral (spectral.py)
# ---------------------------------------------------------------------------

def laplacian_eigenvalues(n):
    """lambda_k = (4/h^2) sin^2(pi k h / 2), k = 1..n, h = 1/(n+1) (spectral.py:100-113)."""
    n = int(n)
    h = 1.0 / (n + 1)
    k = np.arange(1, n + 1)
    return (4.0 / h ** 2) * np.sin(0.5 * np.pi * k * h) ** 2


def dst(x, axis=0):
    """Orthonormal DST-I along one axis (spectral.py:180-183: scipy.fft.dst type 1, ortho)."""
    # workers=-1: lines are transformed independently, so the result does not
    # depend on the thread count (bit-identical to workers=1)
    return scipy.fft.dst(np.asarray(x, dtype=float), type=1, norm="ortho", axis=axis, workers=-1)


def sine_matrix(n):
    """Dense orthonormal sine basis, F[j, k] = sqrt(2/(n+1)) sin(pi (j+1)(k+1)/(n+1))."""
    j = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(j, j) / (n + 1))


# ---------------------------------------------------------------------------
# cores (fracop.py)
# ---------------------------------------------------------------------------

def mode_values(eigs, alpha, aggregation="sum-then-power", transform=None):
    """Per-mode rho contributions and the outer exponent (fracop.py:93-106)."""
    eigs = [np.asarray(e, dtype=float) for e in eigs]
    if aggregation == "sum-then-power":
        return eigs, float(alpha)
    if aggregation == "power-then-sum":
        return [e ** float(alpha) for e in eigs], 1.0
    return [np.asarray(transform(e), dtype=float) for e in eigs], float(alpha)


def eval_on_rho(tag, rho, a, cm=1.0, cp=1.0, reciprocal=False):
    """The four core functions of rho (fracop.py:109-121)."""
    rho = np.asarray(rho, dtype=float)
    if tag == "g1":
        v = cm * rho ** (-a)
        return 1.0 / v if reciprocal else v
    if tag in ("g2", "g3"):
        s = cm * rho ** (-a) + cp * rho ** a
        return s if ((tag == "g2") != reciprocal) else 1.0 / s
    s = 1.0 + cp * rho ** (2.0 * a)
    return s if reciprocal else 1.0 / s


def rho_grid(mus):
    """rho on the full index grid, summed in the reference's order (fracop.py:144-147)."""
    if len(mus) == 2:
        return mus[0][:, None] + mus[1][None, :]
    return mus[0][:, None, None] + mus[1][None, :, None] + mus[2][None, None, :]


def dense_core(tag, mus, a, cm=1.0, cp=1.0, reciprocal=False):
    """Dense core tensor g(rho) (fracop.py:138-148)."""
    return eval_on_rho(tag, rho_grid(mus), a, cm, cp, reciprocal)


def sinc_terms(a, M, gamma_param=0.8):
    """Sinc nodes t_nu and log-weights for rho^-a (fracop.py:179-191)."""
    M = int(M)
    step = float(gamma_param) * np.pi / np.sqrt(M)
    u = step * np.arange(-M, M + 1, dtype=float)
    t = np.logaddexp(0.0, u)
    logt = np.where(u < -30.0, u, np.log(t))
    logphi = -np.logaddexp(0.0, -u)
    logw = np.log(step) + (a - 1.0) * logt + logphi - gammaln(a)
    return t, logw


def sinc_core(mus, a, M, gamma_param=0.8, scale=1.0):
    """Rank-(2M+1) exponential-sum core of rho^-a (fracop.py:194-199)."""
    rho_min = sum(float(np.min(mu)) for mu in mus)
    t, logw = sinc_terms(a, M, gamma_param)
    w = np.exp(logw - a * np.log(rho_min) + np.log(float(scale)))
    factors = [np.exp(-np.outer(mu / rho_min, t)) for mu in mus]
    return w, factors


def required_sinc_m(a, target):
    """Node count of the sinc route (fracop.py:293-297)."""
    target = max(float(target), 1e-15)
    root = np.log(10.0 / target) / (a * 0.8 * np.pi)
    return max(4, int(np.ceil(root * root)))


# ---------------------------------------------------------------------------
# full-format operator application (tests/oracles.py:56 dense_apply, with the
# fast per-mode DST of spectral.py:183 instead of a dense sine matrix)
# ---------------------------------------------------------------------------

def transform_full(x):
    z = np.asarray(x, dtype=float)
    for ax in range(z.ndim):
        z = dst(z, axis=ax)
    return z


def apply_full(core, x, alpha=1.0):
    """alpha * F diag(core) F x over every mode."""
    return alpha * transform_full(core * transform_full(x))


# ---------------------------------------------------------------------------
# canonical tensors (tensor.py)
# ---------------------------------------------------------------------------

def cp_to_dense(weights, factors):
    """tensor.py:217-225."""
    if len(factors) == 2:
        return (factors[0] * weights) @ factors[1].T
    return np.einsum("ik,jk,lk,k->ijl", factors[0], factors[1], factors[2], weights)


def cp_inner(wa, fa, wb, fb):
    """Gram-product inner product (tensor.py:156-167)."""
    if len(wa) == 0 or len(wb) == 0:
        return 0.0
    H = fa[0].T @ fb[0]
    for A, B in zip(fa[1:], fb[1:]):
        H = H * (A.T @ B)
    return float(wa @ H @ wb)


def cp_normalize(weights, factors):
    """Unit columns, weights absorb norms, zero columns -> zero weight + e_1 (tensor.py:180-197)."""
    w = np.array(weights, dtype=float, copy=True)
    out = []
    for U in factors:
        nrm = np.linalg.norm(U, axis=0)
        zero = nrm == 0.0
        V = U / np.where(zero, 1.0, nrm)
        if np.any(zero):
            V = V.copy()
            V[0, zero] = 1.0
        w = w * np.where(zero, 0.0, nrm)
        out.append(V)
    return w, out


def cp_apply(core_w, core_f, xw, xf, eigs_bases=None):
    """Canonical operator application, output rank R*S (fracop.py:474-495)."""
    R, S = len(core_w), len(xw)
    factors = []
    for U, X in zip(core_f, xf):
        Xs = dst(X, axis=0)
        Z = np.einsum("ik,ij->ikj", U, Xs).reshape(U.shape[0], R * S)
        factors.append(dst(Z, axis=0))
    return np.outer(core_w, xw).ravel(), factors


# ---------------------------------------------------------------------------
# design functions (rhs.py)
# ---------------------------------------------------------------------------

def grid_points(n):
    return (np.arange(n) + 1.0) / (n + 1.0)


def gaussian_bumps(n, d, count, seed, noise=0.0):
    """Seeded sum of separable Gaussian bumps (BASELINE.json configs): centres
    U(0.2, 0.8), widths U(0.05, 0.2), amplitudes N(0, 1) per bump; returns the
    canonical (weights, factors) and, when noise > 0, nothing else (the noise is
    a dense add done by the caller)."""
    rng = np.random.default_rng(seed)
    x = grid_points(n)
    w = rng.standard_normal(count)
    factors = [np.empty((n, count)) for _ in range(d)]
    for k in range(count):
        for l in range(d):
            c = rng.uniform(0.2, 0.8)
            s = rng.uniform(0.05, 0.2)
            factors[l][:, k] = np.exp(-((x - c) ** 2) / (2.0 * s * s))
    return w, factors


# ---------------------------------------------------------------------------
# PCG on dense arrays (solver.py:116-180, classical iteration; full format)
# ---------------------------------------------------------------------------

def pcg_dense(matvec, precond, b, tol, k_max):
    """Returns (x, residual history, iterations, converged) with the reference's
    stopping rule ||r|| / ||b|| <= tol checked after each update (solver.py:152-169)."""
    norm_b = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if norm_b == 0.0:
        return x, [0.0], 0, True
    r = b.copy()
    hist = [float(np.linalg.norm(r)) / norm_b]
    if hist[-1] <= tol:
        return x, hist, 0, True
    z = precond(r)
    p = z.copy()
    rz = float(np.vdot(r, z))
    it = 0
    for k in range(1, int(k_max) + 1):
        s = matvec(p)
        ps = float(np.vdot(p, s))
        step = rz / ps
        x = x + step * p
        r = r - step * s
        hist.append(float(np.linalg.norm(r)) / norm_b)
        it = k
        if hist[-1] <= tol:
            return x, hist, it, True
        z = precond(r)
        rz_new = float(np.vdot(r, z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, hist, it, False


def reciprocal_svd_core(tag, mus, a, cm, cp, r):
    """Rank-r reciprocal core by dense SVD (the 2D preconditioner route,
    fracop.py:392-402 with reciprocal=True and a fixed-rank spec) as a dense array."""
    G = dense_core(tag, mus, a, cm, cp, reciprocal=True)
    U, s, Vt = np.linalg.svd(G, full_matrices=False)
    k = min(int(r), int(np.count_nonzero(s > 0.0)))
    return (U[:, :k] * s[:k]) @ Vt[:k]


# ---------------------------------------------------------------------------
# dense helpers mirroring the reference's test oracles (tests/oracles.py)
# ---------------------------------------------------------------------------

def random_cp_dense(dims, rank, seed, scale=1.0):
    """Seeded random CP tensor as (weights, factors, dense) (tests/oracles.py:68-78)."""
    rng = np.random.default_rng(seed)
    weights = scale * rng.standard_normal(rank)
    factors = [rng.standard_normal((n, rank)) for n in dims]
    return weights, factors, cp_to_dense(weights, factors)


def dense_apply(core, x):
    """F f(Lambda) F^T x with the dense sine basis, mode by mode (tests/oracles.py:56-65)."""
    z = np.asarray(x, dtype=float)
    d = z.ndim
    for ax in range(d):
        F = sine_matrix(z.shape[ax])
        z = np.moveaxis(np.tensordot(F.T, z, axes=(1, ax)), 0, ax)
    z = core * z
    for ax in range(d):
        F = sine_matrix(z.shape[ax])
        z = np.moveaxis(np.tensordot(F, z, axes=(1, ax)), 0, ax)
    return z


def kkt_dense_solve(y_design, alpha, beta, gamma):
    """Spectral-space optimality solve (tests/oracles.py:105-124): returns (y, u)."""
    d = y_design.ndim
    lams = [laplacian_eigenvalues(n) for n in y_design.shape]
    rho = rho_grid(lams)
    z = transform_full(y_design)
    u = transform_full(z / (beta * rho ** (-alpha) + (gamma / beta) * rho ** alpha))
    y = transform_full(z / (1.0 + (gamma / beta ** 2) * rho ** (2.0 * alpha)))
    return y, u

"""CPU suite: pin the numpy/scipy oracle to golden vectors produced by the
reference package itself (tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name + ".npz"))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def cp(data, prefix, d):
    return data[prefix + "_w"], [data["%s_f%d" % (prefix, l)] for l in range(d)]


def test_eigenvalues_and_dst_match_reference():
    g = load("spectral")
    for n in (1, 2, 3, 5, 7, 9, 12, 15, 16, 31, 63, 127, 255, 511):
        assert np.array_equal(oracle.laplacian_eigenvalues(n), g["lam_%d" % n])
        assert rel(oracle.dst(g["x_%d" % n], axis=0), g["dst_%d" % n]) <= 1e-15
        # DST-I is orthonormal and involutive
        assert rel(oracle.dst(oracle.dst(g["x_%d" % n])), g["x_%d" % n]) <= 1e-13


def test_frozen_small_values():
    # reference tests/test_spectral.py:16-24 and SPEC examples
    assert np.allclose(oracle.laplacian_eigenvalues(2), [9.0, 27.0], atol=1e-12)
    assert np.allclose(oracle.laplacian_eigenvalues(3), [9.372583002030, 32.0, 54.627416997970], atol=1e-9)
    lam = oracle.laplacian_eigenvalues(2)
    assert oracle.eval_on_rho("g1", lam[0] + lam[0], 1.0) == pytest.approx(1.0 / 18.0, rel=1e-14)
    assert oracle.eval_on_rho("g4", lam[0] + lam[0], 1.0) == pytest.approx(1.0 / 325.0, rel=1e-14)
    assert oracle.eval_on_rho("g3", lam[1] + lam[1], 1.0) == pytest.approx(0.018512170037709975, rel=1e-14)


def test_dense_cores_match_reference():
    g = load("cores")
    for d, n in ((2, 9), (3, 7)):
        lam = oracle.laplacian_eigenvalues(n)
        for tag in ("g1", "g2", "g3", "g4"):
            for agg in ("sum-then-power", "power-then-sum"):
                mus, a = oracle.mode_values([lam] * d, 0.5, agg)
                for rec in (False, True):
                    want = g["core_d%d_n%d_%s_%s_%d" % (d, n, tag, agg, int(rec))]
                    got = oracle.dense_core(tag, mus, a, 1.3, 0.7, rec)
                    assert rel(got, want) <= 1e-15


def test_sinc_core_matches_reference():
    g = load("cores")
    lam = oracle.laplacian_eigenvalues(32)
    exact = oracle.dense_core("g1", [lam, lam], 0.5)
    for M in (4, 9, 16):
        w, f = oracle.sinc_core([lam, lam], 0.5, M)
        gw, gf = cp(g, "sinc_M%d" % M, 2)
        assert rel(w, gw) <= 1e-14
        for a, b in zip(f, gf):
            assert rel(a, b) <= 1e-14
        dense = oracle.cp_to_dense(w, f)
        err = np.max(np.abs(dense - exact) / exact)
        assert err == pytest.approx(float(g["sinc_M%d_err" % M]), rel=1e-8)


def test_canonical_and_full_apply_match_reference():
    g = load("apply")
    for d, n, tag in ((2, 16, "g2"), (2, 15, "g1"), (3, 9, "g2"), (3, 15, "g4")):
        key = "ap_d%d_n%d_%s" % (d, n, tag)
        cw, cf = cp(g, key + "_core", d)
        xw, xf = cp(g, key + "_x", d)
        yw, yf = oracle.cp_apply(cw, cf, xw, xf)
        assert len(yw) == int(g[key + "_rank"])
        assert rel(oracle.cp_to_dense(yw, yf), g[key + "_y"]) <= 1e-12
        # full format: exact core, per-mode fast DST vs the reference dense oracle
        alpha = 1.0 if tag == "g1" else 0.5
        core = oracle.dense_core(tag, [oracle.laplacian_eigenvalues(n)] * d, alpha)
        assert rel(oracle.apply_full(core, g[key + "_full_x"]), g[key + "_full_y"]) <= 1e-12


def test_cp_inner_and_normalize():
    rng = np.random.default_rng(3)
    for dims in ((7, 6), (4, 3, 5)):
        wa, fa = rng.standard_normal(3), [rng.standard_normal((n, 3)) for n in dims]
        wb, fb = rng.standard_normal(2), [rng.standard_normal((n, 2)) for n in dims]
        da, db = oracle.cp_to_dense(wa, fa), oracle.cp_to_dense(wb, fb)
        assert oracle.cp_inner(wa, fa, wb, fb) == pytest.approx(float(np.vdot(da, db)), rel=1e-12)
        w2, f2 = oracle.cp_normalize(wa, fa)
        assert rel(oracle.cp_to_dense(w2, f2), da) <= 1e-13
    # 3-4-5 and zero-column cases (reference tests/test_tensor.py:71-90)
    w, f = oracle.cp_normalize(np.array([2.0]), [np.array([[3.0], [4.0]]), np.array([[4.0], [3.0]])])
    assert w[0] == pytest.approx(50.0)
    w, f = oracle.cp_normalize(np.array([1.0, 3.0]), [np.array([[0.0, 1.0], [0.0, 2.0]]),
                                                      np.array([[1.0, 1.0], [1.0, 0.0]])])
    assert w[0] == 0.0 and np.isclose(np.linalg.norm(f[0][:, 0]), 1.0)


def test_pcg_dense_oracle_on_config0_operator():
    """The oracle's dense PCG with the reference's rank-6 preconditioner core
    reproduces the reference's config0 solution (full format vs canonical)."""
    g = load("config0")
    n = 255
    lam = oracle.laplacian_eigenvalues(n)
    beta, gamma, alpha = 1e-3, 1.0, 0.5
    A = oracle.dense_core("g2", [lam, lam], alpha, beta, gamma / beta)
    P = oracle.reciprocal_svd_core("g2", [lam, lam], alpha, beta, gamma / beta, 6)
    yw, yf = cp(g, "y", 2)
    b = oracle.cp_to_dense(yw, yf)
    x, hist, it, ok = oracle.pcg_dense(lambda v: oracle.apply_full(A, v), lambda v: oracle.apply_full(P, v),
                                       b, 1e-8, 100)
    uw, uf = cp(g, "u", 2)
    assert ok
    assert abs(it - int(g["iters"])) <= 1
    assert rel(x, oracle.cp_to_dense(uw, uf)) <= 1e-8


@pytest.mark.parametrize("n3", [15, 31])
def test_kkt_oracle_matches_reference_3d_control_solves(n3):
    """The oracle's exact spectral optimality solve reproduces the reference's
    truncated 3D control solves (solver.py:203-216, residual_tol 1e-6, eps 1e-8)
    to within the reference's own PCG tolerance, and the oracle's dense PCG
    (identity preconditioner) agrees with both."""
    g = load("solve")
    key = "c3_n%d" % n3
    y = oracle.cp_to_dense(g[key + "_y_w"], [g[key + "_y_f%d" % i] for i in range(3)])
    alpha, beta, gamma = float(g[key + "_alpha"]), 1e-2, 1.0
    _, u = oracle.kkt_dense_solve(y, alpha, beta, gamma)
    assert rel(u, g[key + "_u"]) <= 1e-6
    lam = oracle.laplacian_eigenvalues(n3)
    A = oracle.dense_core("g2", [lam] * 3, alpha, beta, gamma / beta)
    x, _, _, ok = oracle.pcg_dense(lambda v: oracle.apply_full(A, v), lambda v: v, y, 1e-6, 200)
    assert ok
    assert rel(x, u) <= 1e-5

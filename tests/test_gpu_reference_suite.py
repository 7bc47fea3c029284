"""The reference package's own test intents (pkg/tests/test_tensor.py,
test_decomp.py, test_fracop.py, test_solver.py), exercised against the
device implementation.  Expected values come from the CPU oracle (a
restatement pinned to the reference, see test_oracle_golden.py)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import decomp as fld

pytestmark = pytest.mark.gpu


def D(x):
    """dense host array of a CpTensor / TuckerTensor / device tensor"""
    if isinstance(x, fl.CpTensor):
        x = fl.cp_to_dense(x)
    elif isinstance(x, fl.TuckerTensor):
        x = fl.tucker_to_dense(x)
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def rcp(dims, rank, seed, scale=1.0):
    w, f, dense = oracle.random_cp_dense(dims, rank, seed, scale)
    return fl.CpTensor(w, f), dense


def decaying_matrix(n1, n2, seed, base=0.3):
    rng = np.random.default_rng(seed)
    q1 = np.linalg.qr(rng.standard_normal((n1, min(n1, n2))))[0]
    q2 = np.linalg.qr(rng.standard_normal((n2, min(n1, n2))))[0]
    s = base ** np.arange(min(n1, n2))
    return (q1 * s) @ q2.T, s


# ---------------------------------------------------------------- tensor ---

def test_cp_validation_and_shapes():
    with pytest.raises(ValueError):
        fl.CpTensor(np.ones(2), [np.ones((3, 2))])
    with pytest.raises(ValueError):
        fl.CpTensor(np.ones(2), [np.ones((3, 2)), np.ones((3, 3))])
    with pytest.raises(ValueError):
        fl.CpTensor(np.ones((2, 1)), [np.ones((3, 2)), np.ones((3, 2))])
    t = fl.CpTensor(np.ones(2), [np.ones((3, 2)), np.ones((4, 2))])
    assert t.dims == (3, 4) and t.rank == 2 and t.ndim == 2


def test_zero_rank_one_add_scale():
    z = fl.CpTensor.zero((3, 4, 5))
    assert z.rank == 0 and np.allclose(D(z), 0.0)
    t = fl.CpTensor.from_rank_one([np.ones(3), np.arange(4.0)], 2.0)
    assert np.allclose(D(t), 2.0 * np.outer(np.ones(3), np.arange(4.0)))
    for seed in range(3):
        a, da = rcp((6, 5), 3, seed)
        b, db = rcp((6, 5), 4, seed + 100)
        assert np.allclose(D(fl.cp_add(a, b)), da + db)
        assert np.allclose(D(fl.cp_scale(a, -2.5)), -2.5 * da)
    a, da = rcp((4, 5, 6), 3, 7)
    b, db = rcp((4, 5, 6), 2, 8)
    assert np.allclose(D(fl.cp_add(a, b)), da + db)
    with pytest.raises(ValueError):
        fl.cp_add(a, rcp((4, 5, 7), 1, 0)[0])


def test_inner_norm_and_normalize():
    for seed in range(3):
        for dims in ((7, 6), (4, 3, 5)):
            a, da = rcp(dims, 3, seed)
            b, db = rcp(dims, 2, seed + 50)
            assert np.isclose(fl.cp_inner(a, b), np.vdot(da, db), rtol=1e-10)
            assert np.isclose(fl.cp_norm(a), np.linalg.norm(da), rtol=1e-10)
    z = fl.CpTensor.zero((3, 3))
    assert fl.cp_inner(z, z) == 0.0 and fl.cp_norm(z) == 0.0
    t = fl.CpTensor(np.array([2.0]), [np.array([[3.0], [4.0]]), np.array([[4.0], [3.0]])])
    nt = fl.cp_normalize(t)
    assert np.isclose(float(nt.weights[0]), 50.0)
    assert np.allclose(D(nt), D(t))


def test_hadamard_tucker_cap_storage():
    a, da = rcp((5, 6), 3, 2)
    vecs = [np.linspace(1, 2, 5), np.linspace(-1, 1, 6)]
    prod = fl.cp_hadamard_rank1(a, vecs, 1.5)
    assert prod.rank == a.rank
    assert np.allclose(D(prod), da * 1.5 * np.outer(vecs[0], vecs[1]))
    core = np.random.default_rng(0).standard_normal((2, 3, 2))
    sides = [np.linalg.qr(np.random.default_rng(i).standard_normal((6, r)))[0] for i, r in enumerate((2, 3, 2))]
    tt = fl.TuckerTensor(core, sides)
    assert tt.dims == (6, 6, 6) and tt.ranks == (2, 3, 2)
    assert np.allclose(D(tt), np.einsum("abc,ia,jb,kc->ijk", core, *sides))
    with pytest.raises(ValueError):
        fl.TuckerTensor(np.zeros((7, 2)), [np.eye(6, 7), np.eye(6, 2)])
    big = fl.CpTensor(np.ones(1), [np.ones((5000, 1)), np.ones((5000, 1))])
    with pytest.raises(fl.ResourceLimitError):
        fl.cp_to_dense(big)
    t = fl.CpTensor(np.ones(3), [np.ones((10, 3)), np.ones((20, 3))])
    assert fl.storage_size(t) == 3 + 30 + 60


def test_dumps_roundtrip_and_reject(tmp_path):
    for dims, rank in (((5, 7), 3), ((4, 5, 6), 2)):
        t, _ = rcp(dims, rank, 9)
        p = tmp_path / "t.lrt"
        fl.save_tensor(str(p), t)
        back = fl.load_tensor(str(p))
        assert back.dims == t.dims and back.rank == t.rank
        assert np.array_equal(D(back), D(t))
    p = tmp_path / "bad.lrt"
    p.write_bytes(b"NOPE" + bytes(64))
    with pytest.raises(ValueError):
        fl.load_tensor(str(p))


# ---------------------------------------------------------------- decomp ---

def test_svd_truncate_tail_and_fixed_rank():
    m, s = decaying_matrix(20, 16, 1)
    for tol in (1e-2, 1e-5, 1e-9):
        t = fl.svd_truncate(m, fl.TruncationSpec(tolerance=tol))
        err = np.linalg.norm(D(t) - m)
        assert err <= tol * np.linalg.norm(m) + 1e-14
        assert np.isclose(err, np.sqrt(np.sum(s[t.rank:] ** 2)), rtol=1e-9, atol=1e-14)
    m, s = decaying_matrix(12, 12, 2)
    t = fl.svd_truncate(m, fl.TruncationSpec(max_rank=4, mode="fixed-rank"))
    assert t.rank == 4 and np.allclose(t.weights.cpu().numpy(), s[:4], rtol=1e-12)


def test_hosvd_and_als():
    _, dense = rcp((6, 5, 4), 3, 3)
    assert np.allclose(D(fl.hosvd(dense, (6, 5, 4))), dense, atol=1e-10)
    assert np.allclose(D(fl.hosvd(dense, (3, 3, 3))), dense, atol=1e-9)
    with pytest.raises(ValueError):
        fl.hosvd(dense, (7, 5, 4))
    _, dense = rcp((8, 8, 8), 5, 4)
    t = fl.hosvd(dense, (4, 4, 4))
    for U in t.sides:
        U = U.cpu().numpy()
        assert np.allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-12)
    dense = np.random.default_rng(5).standard_normal((9, 9, 9))
    h = fl.hosvd(dense, (4, 4, 4))
    a = fl.tucker_als(dense, (4, 4, 4), max_sweeps=20)
    assert np.linalg.norm(D(a) - dense) <= np.linalg.norm(D(h) - dense) * (1.0 + 1e-12)
    _, dense = rcp((7, 6, 5), 2, 6)
    assert np.linalg.norm(D(fl.tucker_als(dense, (2, 2, 2), max_sweeps=10)) - dense) <= 1e-9


def test_multigrid_tucker():
    assert fld.level_sizes(63, 2) == [63, 127] and fld.level_sizes(8, 4) == [8, 16, 32, 64]
    sizes = fld.level_sizes(15, 3)

    def sampler(i, j, k, level):
        n = sizes[level - 1]
        x, y, z = (i + 1.0) / (n + 1), (j + 1.0) / (n + 1), (k + 1.0) / (n + 1)
        return torch.exp(-x - 0.5 * y) * (1.0 + z) + 0.1 * torch.sin(x * y * z)

    tt = fl.multigrid_tucker(sampler, 15, 3, (5, 5, 5))
    n = sizes[-1]
    ar = torch.arange(n, device="cuda")
    dense = sampler(ar[:, None, None], ar[None, :, None], ar[None, None, :], 3).cpu().numpy()
    rel = np.linalg.norm(D(tt) - dense) / np.linalg.norm(dense)
    ref = np.linalg.norm(D(fl.hosvd(dense, (5, 5, 5))) - dense) / np.linalg.norm(dense)
    assert rel <= 1e-5 and rel <= 10.0 * ref + 1e-12
    with pytest.raises(ValueError):
        fl.multigrid_tucker(sampler, 15, 2, (16, 16, 16))


def test_rhosvd_c2t_t2c():
    t, dense = rcp((8, 8, 8), 10, 7)
    tk = fl.rhosvd(t, (5, 5, 5))
    err = np.linalg.norm(D(tk) - dense)
    best = np.linalg.norm(D(fl.hosvd(dense, (5, 5, 5))) - dense)
    assert best * (1 - 1e-12) <= err <= 25.0 * best + 1e-12
    with pytest.raises(ValueError):
        fl.rhosvd(t, (11, 5, 5))
    for dims in ((10, 9), (7, 8, 6)):
        t, dense = rcp(dims, 5, 11)
        tk = fl.c2t(t, fl.TruncationSpec(tolerance=1e-10))
        back = fl.t2c(tk, fl.TruncationSpec(tolerance=1e-10))
        assert np.linalg.norm(D(back) - dense) / np.linalg.norm(dense) <= 1e-8
    core = np.zeros((3, 3, 3))
    core[0, 0, 0], core[1, 1, 1], core[2, 2, 2] = 5.0, 3.0, 1.0
    sides = [np.linalg.qr(np.random.default_rng(i).standard_normal((8, 3)))[0] for i in range(3)]
    c = fl.t2c(fl.TuckerTensor(core, sides), fl.TruncationSpec(tolerance=0.0))
    assert c.rank == 3 and np.allclose(D(c), D(fl.TuckerTensor(core, sides)), atol=1e-12)


def test_trunc_properties():
    for seed in range(3):
        for dims in ((12, 11), (7, 6, 8)):
            t, dense = rcp(dims, 6, seed, scale=2.0)
            spec = fl.TruncationSpec(tolerance=1e-6)
            out = fl.trunc(t, spec)
            assert out.rank <= t.rank
            assert np.linalg.norm(D(out) - dense) <= 1e-6 * np.linalg.norm(dense) * 1.01 + 1e-13
            again = fl.trunc(out, spec)
            assert again.rank == out.rank
            assert np.linalg.norm(D(again) - D(out)) <= 1e-12 * max(1.0, np.linalg.norm(dense))
    t, dense = rcp((8, 8, 8), 4, 19)
    out = fl.trunc(fl.cp_add(t, t), fl.TruncationSpec(tolerance=1e-10))
    assert out.rank <= t.rank
    assert np.linalg.norm(D(out) - 2 * dense) <= 1e-10 * 2 * np.linalg.norm(dense) * 1.01 + 1e-12
    m, s = decaying_matrix(16, 16, 21)
    u, sv, vt = np.linalg.svd(m)
    t = fl.CpTensor(np.ones(16), [u * sv, vt.T])
    for r in (3, 6, 9):
        out = fl.trunc(t, fl.TruncationSpec(max_rank=r, mode="fixed-rank"))
        assert np.isclose(np.linalg.norm(D(out) - m), np.sqrt(np.sum(s[r:] ** 2)), rtol=1e-9, atol=1e-13)


# ---------------------------------------------------------------- fracop ---

def test_core_entries_and_identities():
    spec = fl.laplacian_spectrum(2, 2)
    assert fl.core_entry(fl.CoreFunctionKind("g1", 1.0), spec, (0, 0)) == pytest.approx(1 / 18, rel=1e-14)
    assert fl.core_entry(fl.CoreFunctionKind("g4", 1.0), spec, (0, 0)) == pytest.approx(1 / 325, rel=1e-14)
    assert fl.core_entry(fl.CoreFunctionKind("g3", 1.0), spec, (1, 1)) == pytest.approx(0.018512170037709975, rel=1e-14)
    with pytest.raises(ValueError):
        fl.core_entry(fl.CoreFunctionKind("g1", 0.5), fl.laplacian_spectrum(4, 2), (0, 4))
    for d in (2, 3):
        sp = fl.laplacian_spectrum(6, d)
        cp = fl.sum_core_exact(sp)
        lam = oracle.laplacian_eigenvalues(6)
        assert cp.rank == d and np.allclose(D(cp), oracle.rho_grid([lam] * d), rtol=1e-14, atol=0)
    for d in (2, 3):
        sp = fl.laplacian_spectrum(7, d)
        for kind in (fl.CoreFunctionKind("g1", 1.0, coeff_minus=2.0),
                     fl.CoreFunctionKind("g1", 0.4, aggregation="power-then-sum")):
            op = fl.reciprocal_core(kind, sp, fl.TruncationSpec(tolerance=1e-12))
            lam = oracle.laplacian_eigenvalues(7)
            a = kind.alpha if kind.aggregation == "power-then-sum" else 1.0
            want = oracle.rho_grid([lam ** a] * d) / kind.coeff_minus
            assert op.rank == d and op.reciprocal
            assert np.linalg.norm(D(op.core) - want) <= 1e-12 * np.linalg.norm(want)


def test_build_routes():
    spec = fl.laplacian_spectrum(24, 2)
    lam = oracle.laplacian_eigenvalues(24)
    for tag in ("g1", "g2", "g3", "g4"):
        for alpha in (1.0, 0.5, 0.1):
            op = fl.build_core(fl.CoreFunctionKind(tag, alpha), spec, fl.TruncationSpec(tolerance=1e-10),
                               method="dense-svd")
            want = oracle.dense_core(tag, [lam, lam], alpha)
            assert np.linalg.norm(D(op.core) - want) / np.linalg.norm(want) <= 1e-9
            assert op.achieved_error <= 1e-10
    sp = fl.laplacian_spectrum(8, 2)
    with pytest.raises(ValueError):
        fl.build_core(fl.CoreFunctionKind("g2", 0.5), sp, fl.TruncationSpec(tolerance=1e-6), method="sinc")
    with pytest.raises(ValueError):
        fl.build_core(fl.CoreFunctionKind("g2", 0.5), sp, fl.TruncationSpec(tolerance=1e-6), method="qr")
    with pytest.raises(ValueError):
        fl.build_core(fl.CoreFunctionKind("g2", 0.5), fl.laplacian_spectrum(8, 3),
                      fl.TruncationSpec(tolerance=1e-6), method="dense-svd")
    spec3 = fl.laplacian_spectrum(15, 3)
    op = fl.build_core(fl.CoreFunctionKind("g2", 0.5), spec3, fl.TruncationSpec(tolerance=1e-6), method="mg-tucker")
    want = oracle.dense_core("g2", [oracle.laplacian_eigenvalues(15)] * 3, 0.5)
    rel = np.linalg.norm(D(op.core) - want) / np.linalg.norm(want)
    assert rel <= 1e-6 and op.achieved_error == pytest.approx(rel, rel=1e-8)
    op3 = fl.build_core(fl.CoreFunctionKind("g3", 0.5), spec3, fl.TruncationSpec(max_rank=5, mode="fixed-rank"))
    assert op3.rank <= 5
    # aggregations
    kind = fl.CoreFunctionKind("g2", 0.3, aggregation="power-then-sum")
    op = fl.build_core(kind, fl.laplacian_spectrum(16, 2), fl.TruncationSpec(tolerance=1e-10))
    lam = oracle.laplacian_eigenvalues(16)
    want = oracle.dense_core("g2", [lam ** 0.3] * 2, 1.0)
    assert np.linalg.norm(D(op.core) - want) <= 1e-9 * np.linalg.norm(want)
    kind = fl.CoreFunctionKind("g1", 0.5, aggregation="generalized", transform=lambda lam: np.log1p(lam))
    mu = np.log1p(oracle.laplacian_eigenvalues(12))
    op = fl.build_core(kind, fl.laplacian_spectrum(12, 2), fl.TruncationSpec(tolerance=1e-10))
    want = (mu[:, None] + mu[None, :]) ** -0.5
    assert np.linalg.norm(D(op.core) - want) <= 1e-9 * np.linalg.norm(want)


def test_apply_identity_symmetry_validation(tmp_path):
    for d in (2, 3):
        spec = fl.laplacian_spectrum(9, d)
        ident = fl.LowRankOperator(fl.DiagOpFunction(spec, fl.CoreFunctionKind("g1", 1.0),
                                                     fl.CpTensor(np.ones(1), [np.ones((9, 1))] * d), 0.0))
        x, dense = rcp((9,) * d, 3, d)
        y = ident(x)
        assert y.rank == x.rank and np.allclose(D(y), dense, rtol=0, atol=1e-12 * np.abs(dense).max())
    n = 8
    spec = fl.laplacian_spectrum(n, 2)
    op = fl.LowRankOperator(fl.build_core(fl.CoreFunctionKind("g2", 0.5), spec, fl.TruncationSpec(tolerance=1e-12)))
    for seed in range(3):
        x, _ = rcp((n, n), 2, seed)
        y, _ = rcp((n, n), 2, 200 + seed)
        assert fl.cp_inner(op(x), y) == pytest.approx(fl.cp_inner(x, op(y)), rel=1e-10, abs=1e-12)
        assert fl.cp_inner(op(x), x) > 0.0
    with pytest.raises(ValueError):
        fl.apply(op.diag, rcp((n, n), 2, 0)[0])
    with pytest.raises(ValueError):
        op(rcp((5, 5), 2, 0)[0])
    # operator dumps
    kind = fl.CoreFunctionKind("g2", 0.5, coeff_minus=2.0, coeff_plus=0.75)
    rop = fl.reciprocal_core(kind, fl.laplacian_spectrum(10, 2), fl.TruncationSpec(tolerance=1e-9))
    path = tmp_path / "op.lro"
    fl.save_operator(path, rop)
    back = fl.load_operator(path)
    assert back.diag.kind == kind and back.diag.reciprocal
    assert np.array_equal(D(back.diag.core), D(rop.core))
    gk = fl.CoreFunctionKind("g1", 0.5, aggregation="generalized", transform=lambda lam: lam + 1.0)
    with pytest.raises(ValueError):
        fl.save_operator(tmp_path / "g.lro", fl.build_core(gk, spec, fl.TruncationSpec(tolerance=1e-8)))


def test_generalized_mode_dense_basis_apply():
    rng = np.random.default_rng(5)
    n = 7

    def spd():
        K = np.diag(2.5 + rng.uniform(0.0, 1.0, size=n))
        off = -rng.uniform(0.1, 0.5, size=n - 1)
        return K + np.diag(off, 1) + np.diag(off, -1)

    K1, K2 = spd(), spd()
    modes = (fl.generalized_mode(K1), fl.generalized_mode(K2))
    spec = fl.EigenSpectrum(modes)
    kind = fl.CoreFunctionKind("g3", 0.5)
    op = fl.LowRankOperator(fl.build_core(kind, spec, fl.TruncationSpec(tolerance=1e-12), method="dense-svd"))
    x, dense = rcp((n, n), 2, 9)
    # dense oracle: Q diag(g) Q^T per mode
    lam1, Q1 = np.linalg.eigh(K1)
    lam2, Q2 = np.linalg.eigh(K2)
    G = oracle.eval_on_rho("g3", lam1[:, None] + lam2[None, :], 0.5)
    want = Q1 @ (G * (Q1.T @ dense @ Q2)) @ Q2.T
    assert np.linalg.norm(D(op(x)) - want) <= 1e-10 * np.linalg.norm(want)


# ---------------------------------------------------------------- solver ---

def laplace_system(n, d):
    spec = fl.laplacian_spectrum(n, d)
    fun = fl.LowRankOperator(fl.reciprocal_core(fl.CoreFunctionKind("g1", 1.0), spec,
                                                fl.TruncationSpec(tolerance=1e-15)))
    rho = oracle.rho_grid([oracle.laplacian_eigenvalues(n)] * d)
    return spec, fun, (lambda v: oracle.dense_apply(rho, v))


def test_pcg_matches_dense_cg():
    n, d = 6, 2
    spec, fun, matvec = laplace_system(n, d)
    ident = fl.LowRankOperator(fl.DiagOpFunction(spec, fl.CoreFunctionKind("g1", 1.0),
                                                 fl.CpTensor(np.ones(1), [np.ones((n, 1))] * d), 0.0))
    b, bd = rcp((n, n), 1, 7)
    cfg = fl.SolverConfig(alpha=1.0, eps=0.0, residual_tol=1e-12, k_max=6)
    x, rep = fl.pcg(fun, ident, b, None, cfg)
    _, hist, _, _ = oracle.pcg_dense(matvec, lambda r: r.copy(), bd, 1e-12, 6)
    assert len(rep.residuals) == len(hist)
    for mine, ref in zip(rep.residuals, hist):
        if ref > 1e-7:
            assert mine == pytest.approx(ref, rel=1e-7)
    pre = fl.build_preconditioner(fl.CoreFunctionKind("g1", 1.0), spec, 3)
    P = D(pre.diag.core)
    b, bd = rcp((n, n), 1, 11)
    x, rep = fl.pcg(fun, pre, b, None, fl.SolverConfig(alpha=1.0, eps=0.0, residual_tol=1e-12, k_max=4))
    _, hist, _, _ = oracle.pcg_dense(matvec, lambda r: oracle.dense_apply(P, r), bd, 1e-12, 4)
    for mine, ref in zip(rep.residuals, hist):
        if ref > 1e-7:
            assert mine == pytest.approx(ref, rel=1e-7)


def test_pcg_edge_cases():
    n = 6
    spec, fun, _ = laplace_system(n, 2)
    cfg = fl.SolverConfig(alpha=1.0, eps=0.0, residual_tol=1e-8, k_max=10)
    x, rep = fl.pcg(fun, fun, fl.CpTensor.zero((n, n)), None, cfg)
    assert rep.converged and rep.iterations == 0 and x.rank == 0
    with pytest.raises(ValueError):
        fl.pcg(fun, fun, rcp((n, n), 1, 0)[0], None, None)
    with pytest.raises(ValueError):
        fl.pcg(fun, fun, rcp((5, 5), 1, 0)[0], None, cfg)
    neg = fl.LowRankOperator(fl.DiagOpFunction(spec, fl.CoreFunctionKind("g1", 1.0),
                                               fl.CpTensor(np.array([-1.0]), [np.ones((n, 1))] * 2), 0.0))
    ident = fl.LowRankOperator(fl.DiagOpFunction(spec, fl.CoreFunctionKind("g1", 1.0),
                                                 fl.CpTensor(np.ones(1), [np.ones((n, 1))] * 2), 0.0))
    with pytest.raises(fl.PcgBreakdownError) as info:
        fl.pcg(neg, ident, rcp((n, n), 1, 0)[0], None, fl.SolverConfig(alpha=1.0, eps=0.0, k_max=5))
    assert info.value.iteration == 1 and "iteration 1" in str(info.value)


def test_pcg_truncated_rank_cap_and_solves():
    n, d = 16, 2
    spec = fl.laplacian_spectrum(n, d)
    kind = fl.CoreFunctionKind("g2", 0.5)
    fun = fl.LowRankOperator(fl.build_core(kind, spec, fl.TruncationSpec(tolerance=1e-10)))
    pre = fl.build_preconditioner(kind, spec, 5)
    b, _ = rcp((n, n), 2, 5)
    x, rep = fl.pcg(fun, pre, b, None, fl.SolverConfig(alpha=0.5, eps=1e-8, residual_tol=1e-6, k_max=40, max_rank=5))
    assert rep.converged and x.rank <= 5 and rep.final_rank == x.rank and rep.residuals[-1] <= 1e-6
    # control / state / KKT against the spectral dense solve
    n, d, alpha, beta, gamma = 10, 2, 0.5, 1.0, 1e-2
    spec = fl.laplacian_spectrum(n, d)
    y_d = fl.DesignFunction("gaussian-bump").evaluate((n,) * d)
    y_want, u_want = oracle.kkt_dense_solve(D(y_d), alpha, beta, gamma)
    cfg = fl.SolverConfig(alpha=alpha, beta=beta, gamma=gamma, eps=1e-11, residual_tol=1e-10, k_max=60)
    u, rep = fl.solve_control(y_d, cfg, spec, method="direct")
    y = fl.solve_state(y_d, cfg, spec)
    assert np.linalg.norm(D(u) - u_want) <= 1e-6 * np.linalg.norm(u_want)
    assert np.linalg.norm(D(y) - y_want) <= 1e-6 * np.linalg.norm(y_want)
    r1, r2, r3 = fl.kkt_residual(y, u, None, y_d, cfg, spec)
    assert r1 <= 1e-6 and r2 <= 1e-12 and r3 <= 1e-6
    _, _, r3_bad = fl.kkt_residual(y, fl.cp_scale(u, 2.0), None, y_d, cfg, spec)
    assert r3_bad > 1e-3
    with pytest.raises(ValueError):
        fl.solve_control(y_d, cfg, spec, method="cholesky")
    with pytest.raises(ValueError):
        fl.solve_state(y_d, cfg, spec, method="lu")


def test_design_functions():
    n = 9
    g = fl.DesignFunction("gaussian-bump").evaluate((n, n))
    assert g.rank == 1 and D(g)[4, 4] == pytest.approx(1.0, rel=1e-13)
    assert fl.DesignFunction("two-bumps").evaluate((n, n, n)).rank <= 2
    x = (np.arange(n) + 1.0) / (n + 1.0)
    ind = ((x >= 0.25) & (x <= 0.75)).astype(float)
    assert np.allclose(D(fl.DesignFunction("box-indicator").evaluate((n, n))), np.outer(ind, ind), atol=1e-14)
    c = fl.DesignFunction("custom-separable", profiles=[np.sin, np.cos]).evaluate((n, n))
    assert np.allclose(D(c), np.outer(np.sin(x), np.cos(x)), rtol=1e-13)
    a = fl.random_smooth((10, 10), rank=3, seed=4)
    b = fl.random_smooth((10, 10), rank=3, seed=4)
    assert a.rank == 3 and np.array_equal(D(a), D(b))

"""CPU suite: host-side argument validation mirrors the reference's ValueErrors
(tests/test_fracop.py:29-44, test_decomp.py:40-50, test_solver.py:40-62)."""

import numpy as np
import pytest

from paper_1809_01971_b200.decomp import TruncationSpec, _kept_rank, level_sizes
from paper_1809_01971_b200.fracop import CoreFunctionKind, _coarsen_sizes, _decimate, _required_sinc_m
from paper_1809_01971_b200.solver import REPORT_COLUMNS, PcgReport, SolverConfig, report_row
from paper_1809_01971_b200.spectral import EigenSpectrum, Mode1D, dense_laplacian_1d, laplacian_mode, laplacian_spectrum


def test_kind_validation():
    with pytest.raises(ValueError):
        CoreFunctionKind("g5", 0.5)
    with pytest.raises(ValueError):
        CoreFunctionKind("g1", 0.5, aggregation="mean")
    for bad in (0.0, -0.5, 1.5, np.nan):
        with pytest.raises(ValueError):
            CoreFunctionKind("g1", bad)
    with pytest.raises(ValueError):
        CoreFunctionKind("g2", 0.5, coeff_minus=0.0)
    with pytest.raises(ValueError):
        CoreFunctionKind("g1", 0.5, aggregation="generalized")
    CoreFunctionKind("g1", 0.5, aggregation="generalized", transform=lambda lam: lam + 1.0)


def test_truncation_spec_and_kept_rank():
    TruncationSpec(tolerance=0.0)
    TruncationSpec(max_rank=3, mode="fixed-rank")
    for kw in ({"mode": "fixed-rank"}, {"tolerance": -1e-3}, {"max_rank": 0}, {"mode": "whatever"}):
        with pytest.raises(ValueError):
            TruncationSpec(**kw)
    s = np.array([1.0, 1e-12])
    assert _kept_rank(s, TruncationSpec(tolerance=1e-6)) == 1
    assert _kept_rank(np.zeros(3), TruncationSpec(tolerance=1e-6)) == 0
    assert _kept_rank(np.array([3.0, 2.0, 1.0]), TruncationSpec(max_rank=2, mode="fixed-rank")) == 2
    assert _kept_rank(np.array([3.0, 2.0, 1.0]), TruncationSpec(tolerance=1e-14, max_rank=1)) == 1


def test_solver_config_validation_and_report():
    SolverConfig(alpha=0.5)
    for kw in ({"alpha": 0.0}, {"alpha": 1.5}, {"alpha": 0.5, "beta": 0.0}, {"alpha": 0.5, "gamma": -1.0},
               {"alpha": 0.5, "eps": -1e-9}, {"alpha": 0.5, "residual_tol": 0.0},
               {"alpha": 0.5, "residual_tol": 1.0}, {"alpha": 0.5, "k_max": 0},
               {"alpha": 0.5, "precond_rank": 0}, {"alpha": 0.5, "max_rank": 0}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)
    rep = PcgReport(iterations=4, residuals=[1.0, 1e-7], final_rank=6, converged=True,
                    iteration_seconds=[0.1], seconds_per_iteration=0.125)
    row = report_row("g2", 2, 64, 0.5, 6, 1e-8, rep)
    assert len(row) == len(REPORT_COLUMNS) and row[7] == "1.000000e-07" and row[8] == "1.250000e-01"


def test_spectrum_validation_and_ladders():
    m = laplacian_mode(2)
    assert np.allclose(m.eigenvalues, [9.0, 27.0])
    assert laplacian_spectrum(8, 3).mode_sizes == (8, 8, 8)
    with pytest.raises(ValueError):
        laplacian_spectrum(4, 4)
    with pytest.raises(ValueError):
        laplacian_spectrum(0, 2)
    with pytest.raises(ValueError):
        EigenSpectrum((laplacian_mode(4),))
    with pytest.raises(ValueError):
        Mode1D(n=3, h=0.25, eigenvalues=np.array([1.0, 2.0]))
    assert np.allclose(dense_laplacian_1d(2), [[18.0, -9.0], [-9.0, 18.0]])
    assert level_sizes(63, 2) == [63, 127] and level_sizes(15, 3) == [15, 31, 63]
    assert _coarsen_sizes(1023) == [63, 127, 255, 511, 1023]
    assert _coarsen_sizes(127) == [63, 127]
    assert list(_decimate(np.arange(7.0), 3)) == [1.0, 3.0, 5.0]
    assert _required_sinc_m(0.5, 1e-8) >= 4


def test_lane_core_order_roundtrip():
    """The lane orders of the n = 511 cores (host-side permutations) are
    bijections onto the documented entries, with zero padding."""
    import torch
    from paper_1809_01971_b200.full import lane_core, lane_core_inverse, line_lane_core
    c = torch.randn(3, 11, 511, dtype=torch.float64)
    cl = line_lane_core(c)
    assert cl.shape == (12, 32, 2, 16, 2)  # 33 lines -> 48 (multiple of 16) -> 12 units
    flat = cl.reshape(12, 32, 32, 2)
    lines = c.reshape(33, 511)
    for u, i, f, q in [(0, 1, 0, 0), (2, 31, 1, 15), (7, 7, 1, 3)]:
        for e in range(2):
            line, row = 4 * u + 2 * f + e, 32 * q + i
            assert flat[u, i, 16 * f + q, e] == lines[line, row - 1]
    assert torch.all(flat[:, 0, 0, :] == 0)  # row 0
    assert torch.all(flat[9:] == 0)  # padded lines
    # mode-0 order
    g = torch.randn(511, 3, 511, dtype=torch.float64)
    gl = lane_core(g)
    assert gl.shape == (3 * 128, 32, 2, 16, 2)
    assert torch.equal(lane_core_inverse(gl, (511, 3, 511)), g)
    fl = gl.reshape(3 * 128, 32, 32, 2)
    for i1, cc, w, i, f, q in [(0, 0, 0, 1, 0, 0), (2, 31, 3, 31, 1, 15), (1, 7, 2, 5, 0, 9)]:
        u = (i1 * 32 + cc) * 4 + w
        for e in range(2):
            col, r = 16 * cc + 4 * w + 2 * f + e, 32 * q + i
            want = g[r - 1, i1, col] if col < 511 else 0.0
            assert fl[u, i, 16 * f + q, e] == want
    assert torch.all(fl[:, 0, 0, :] == 0)
    g2 = torch.randn(511, 511, dtype=torch.float64)
    assert torch.equal(lane_core_inverse(lane_core(g2), (511, 511)), g2)

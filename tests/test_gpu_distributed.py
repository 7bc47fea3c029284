"""Slab path with the CUDA bindings on one rank (world 1) vs the single-GPU path."""

import numpy as np
import pytest
import torch

import oracle
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import distributed as D, fullsolve
from paper_1809_01971_b200.fracop import CoreFunctionKind

pytestmark = pytest.mark.gpu


def test_slab_single_rank_matches_fused_path():
    n = 31
    spec = fl.laplacian_spectrum(n, 3)
    lay = D.SlabLayout((n, n, n), 1, 0)
    ops = D.CudaOps()
    x = torch.randn((n, n, n), dtype=torch.float64, device="cuda")
    kind = CoreFunctionKind("g1", 0.5)
    A = D.spectral_core(kind, spec, lay)
    y = D.apply_slab(x, A, lay, ops)
    want = oracle.apply_full(oracle.dense_core("g1", [oracle.laplacian_eigenvalues(n)] * 3, 0.5), x.cpu().numpy())
    assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)
    cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, precond_rank=5, residual_tol=1e-9, k_max=80)
    Af, Pf = fullsolve.control_cores(cfg, spec)
    u1, rep = fullsolve.solve_control_full(x, cfg, spec, cores=(Af, Pf))
    u2, its, hist, conv = D.pcg_slab(x, Af.contiguous(), Pf.contiguous(), lay, ops, 1e-9, 80)
    assert conv and its == rep.iterations
    assert float(torch.linalg.vector_norm(u1 - u2) / torch.linalg.vector_norm(u1)) <= 1e-10

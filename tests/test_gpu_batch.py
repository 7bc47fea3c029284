"""Large-grid core routes (configs[4] machinery) at small n, checked against exact cores."""

import numpy as np
import pytest
import torch

import oracle
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alpha", [0.25, 0.5, 0.9, 1.0])
def test_expsum_control_core_meets_tolerance(alpha):
    n = 31
    spec = fl.laplacian_spectrum(n, 3)
    kind = fl.CoreFunctionKind("g2", alpha, coeff_minus=1e-2, coeff_plus=1.0 / 1e-2)
    core = batch.control_core_expsum(kind, spec, 1e-8)
    want = oracle.dense_core("g2", [oracle.laplacian_eigenvalues(n)] * 3, alpha, 1e-2, 1e2)
    got = fl.cp_to_dense(core).cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-7 * np.linalg.norm(want)


def test_coarse_preconditioner_and_batch_solve():
    n = 63
    recs = batch.solve_batch(n, 2, max_level=31)
    for r in recs:
        assert r["converged"] and r["iterations"] <= 12
    # the interpolated preconditioner approximates 1/g2 to preconditioner accuracy
    spec = fl.laplacian_spectrum(n, 3)
    kind = fl.CoreFunctionKind("g2", 0.5, coeff_minus=1e-2, coeff_plus=1e2)
    P = fl.cp_to_dense(batch.preconditioner_coarse(kind, spec, 6, max_level=31)).cpu().numpy()
    inv = 1.0 / oracle.dense_core("g2", [oracle.laplacian_eigenvalues(n)] * 3, 0.5, 1e-2, 1e2)
    assert np.linalg.norm(P - inv) <= 5e-2 * np.linalg.norm(inv)

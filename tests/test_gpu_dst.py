"""DST-I and full-format operator parity: CUDA path vs the numpy/scipy oracle."""

import numpy as np
import pytest
import torch

import oracle
from paper_1809_01971_b200 import spectral, full
from paper_1809_01971_b200.fracop import CoreFunctionKind

pytestmark = pytest.mark.gpu

# FFT lengths (n+1 = 2^k, 4..8192) and dense-path lengths
FFT_N = [3, 7, 15, 31, 63, 127, 255, 511, 1023, 2047, 4095, 8191]
DENSE_N = [1, 2, 5, 9, 12, 16, 24, 33, 100]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n", FFT_N + DENSE_N)
@pytest.mark.parametrize("inner", [1, 3, 16, 37])
def test_dst1_matches_scipy(n, inner):
    if n >= 4095 and inner > 3:
        pytest.skip("large case covered at inner<=3")
    rng = np.random.default_rng(n * 100 + inner)
    outer = 3
    x = rng.standard_normal((outer, n, inner))
    want = oracle.dst(x, axis=1)
    xt = torch.tensor(x, device="cuda")
    y = torch.empty_like(xt)
    from paper_1809_01971_b200 import _lib
    _lib.call("fl_dst1", _lib.ptr(xt), _lib.ptr(y), outer, n, inner, 1.0, _lib.stream_ptr())
    got = y.cpu().numpy()
    assert rel(got, want) <= 1e-13
    # in place and scaled
    _lib.call("fl_dst1", _lib.ptr(xt), _lib.ptr(xt), outer, n, inner, 2.5, _lib.stream_ptr())
    assert rel(xt.cpu().numpy(), 2.5 * want) <= 1e-13


@pytest.mark.parametrize("n", [4, 9, 16, 63, 64, 511])
def test_dst_apply_api(n):
    m = spectral.laplacian_mode(n)
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 5))
    got = spectral.dst_apply(m, X).cpu().numpy()
    assert rel(got, oracle.dst(X, axis=0)) <= 1e-13
    v = rng.standard_normal(n)
    back = spectral.dst_apply(m, spectral.dst_apply(m, v), "inverse").cpu().numpy()
    assert rel(back, v) <= 1e-13
    with pytest.raises(ValueError):
        spectral.dst_apply(m, np.zeros(n + 1))
    with pytest.raises(ValueError):
        spectral.dst_apply(m, np.zeros(n), "sideways")


@pytest.mark.parametrize("d,n", [(2, 9), (2, 16), (2, 255), (3, 7), (3, 15), (3, 16), (3, 63), (3, 127)])
@pytest.mark.parametrize("tag", ["g1", "g2", "g3", "g4"])
def test_apply_full_matches_oracle(d, n, tag):
    alpha = 0.5
    spec = spectral.laplacian_spectrum(n, d)
    kind = CoreFunctionKind(tag, alpha, coeff_minus=1.3, coeff_plus=0.7)
    lam = oracle.laplacian_eigenvalues(n)
    core_want = oracle.dense_core(tag, [lam] * d, alpha, 1.3, 0.7)
    op = full.FullOperator.from_kind(kind, spec)
    assert rel(op.core.cpu().numpy(), core_want) <= 1e-14
    rng = np.random.default_rng(7 + n + d)
    x = rng.standard_normal((n,) * d)
    want = oracle.apply_full(core_want, x)
    got = op(torch.tensor(x, device="cuda")).cpu().numpy()
    assert rel(got, want) <= 1e-12


def test_apply_host_stream_matches_device_apply():
    n = 63
    spec = spectral.laplacian_spectrum(n, 3)
    op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec)
    xs = [torch.randn((n, n, n), dtype=torch.float64).pin_memory() for _ in range(5)]
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    full.apply_host_stream(op, xs, ys)
    torch.cuda.synchronize()
    for x, y in zip(xs, ys):
        want = op(x.cuda()).cpu()
        assert torch.allclose(y, want, rtol=0, atol=1e-12 * float(want.abs().max()))

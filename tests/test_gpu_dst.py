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
    got = spectral.dst_apply(m, X)
    assert isinstance(got, np.ndarray)  # numpy in -> numpy out, like the reference
    assert rel(got, oracle.dst(X, axis=0)) <= 1e-13
    v = rng.standard_normal(n)
    back = spectral.dst_apply(m, spectral.dst_apply(m, v), "inverse")
    assert rel(back, v) <= 1e-13
    Xt = torch.tensor(X, device="cuda")
    gt = spectral.dst_apply(m, Xt)
    assert isinstance(gt, torch.Tensor) and gt.is_cuda  # device tensors stay on the device
    assert rel(gt.cpu().numpy(), oracle.dst(X, axis=0)) <= 1e-13
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


@pytest.mark.parametrize("dims", [(7, 15), (63, 255), (7, 7, 7), (15, 31, 63), (31, 7, 127), (63, 63, 63),
                                  (3, 127, 255)])
@pytest.mark.parametrize("tag", ["g1", "g4"])
def test_apply_full_padded_matches_oracle(dims, tag):
    """FullOperator on the padded layout (fl_apply_full_padded) vs the oracle
    and vs the unpadded fl_apply_full on the same core."""
    alpha = 0.5
    spec = spectral.EigenSpectrum(tuple(spectral.laplacian_mode(n) for n in dims))
    kind = CoreFunctionKind(tag, alpha, coeff_minus=1.3, coeff_plus=0.7)
    lams = [oracle.laplacian_eigenvalues(n) for n in dims]
    core_want = oracle.dense_core(tag, lams, alpha, 1.3, 0.7)
    op = full.FullOperator.from_kind(kind, spec, padded=True)
    assert op.padded and op.pitch == full.padded_pitch(dims[-1]) and op.pitch % 16 == 0
    assert rel(op.core.cpu().numpy(), core_want) <= 1e-14
    rng = np.random.default_rng(sum(dims))
    x = rng.standard_normal(dims)
    want = oracle.apply_full(core_want, x)
    xt = torch.tensor(x, device="cuda")
    got = op(xt)
    assert rel(got.cpu().numpy(), want) <= 1e-12
    plain = full.FullOperator(spec, op.core.contiguous(), padded=False)
    assert not plain.padded
    assert rel(got.cpu().numpy(), plain(xt).cpu().numpy()) <= 1e-13
    # in place, and repeated application keeps the padding inert
    y = xt.clone()
    op(y, out=y)
    op(y, out=y)
    assert rel(y.cpu().numpy(), oracle.apply_full(core_want, want)) <= 1e-12
    # the per-pass list launches the same computation
    z = torch.empty_like(xt)
    for _, a in op.passes(xt, z):
        full.run_pass(a)
    assert rel(z.cpu().numpy(), want) <= 1e-12


def test_apply_full_padded_big():
    """n = 511 (the bench size): padded vs unpadded and Parseval-type checks."""
    n = 511
    spec = spectral.laplacian_spectrum(n, 3)
    op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec)
    assert op.padded and op.pitch == 512
    plain = full.FullOperator(spec, op.core.contiguous(), padded=False)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
    a = op(x)
    b = plain(x)
    assert float(torch.linalg.vector_norm(a - b)) <= 1e-13 * float(torch.linalg.vector_norm(b))
    # self-adjointness: <Ax, y> = <x, Ay>
    yv = torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
    lhs = float(torch.dot(a.reshape(-1), yv.reshape(-1)))
    rhs = float(torch.dot(x.reshape(-1), op(yv).reshape(-1)))
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)


@pytest.mark.parametrize("kind", [CoreFunctionKind("g1", 0.5),
                                  CoreFunctionKind("g2", 0.5, coeff_minus=1.0, coeff_plus=1.0)],
                         ids=["g1_A^-a", "g2_control"])
def test_apply_511_cube_matches_oracle(kind):
    """BASELINE configs[2] at its exact size: the n = 511 apply of A^-alpha and
    of the control-system operator (the production lane-ordered path) against
    the CPU oracle's scipy DST-I route (reference spectral.py:163-186) on the
    same seeded N(0,1) tensor; north_star tolerance 1e-10 relative (fp64)."""
    import os
    import scipy.fft
    n = 511
    spec = spectral.laplacian_spectrum(n, 3)
    op = full.FullOperator.from_kind(kind, spec)
    assert op.lanes, "the configs[2] operator must take the register-resident lane path"
    x = np.random.default_rng(20511).standard_normal((n, n, n))
    got = op(torch.tensor(x, device="cuda")).cpu().numpy()
    lam = oracle.laplacian_eigenvalues(n)
    core = oracle.dense_core(kind.tag, [lam] * 3, 0.5, kind.coeff_minus, kind.coeff_plus)
    w = os.cpu_count() or 1
    z = x
    for ax in range(3):
        z = scipy.fft.dst(z, type=1, norm="ortho", axis=ax, workers=w)
    z *= core
    for ax in range(3):
        z = scipy.fft.dst(z, type=1, norm="ortho", axis=ax, workers=w)
    d = got - z
    rel_l2 = float(np.linalg.norm(d) / np.linalg.norm(z))
    max_rel = float(np.abs(d).max() / np.abs(z).max())
    print("configs[2] %s parity: rel_l2 %.3e max_rel %.3e" % (kind.tag, rel_l2, max_rel))
    assert rel_l2 <= 1e-10 and max_rel <= 1e-10


@pytest.mark.parametrize("n", [7, 63, 255])
def test_dst1_pass_layouts(n):
    """fl_dst1_pass with distinct input/output layouts vs scipy."""
    from paper_1809_01971_b200 import _lib
    rng = np.random.default_rng(n)
    blocks, groups, width = 2, 3, 5
    # input: [blocks][n][groups][width] dense; output: [blocks][groups][n][width+3] padded
    x = rng.standard_normal((blocks, n, groups, width))
    want = oracle.dst(x, axis=1)
    xt = torch.tensor(x, device="cuda")
    yt = torch.full((blocks, groups, n, width + 3), 7.0, dtype=torch.float64, device="cuda")
    lin = (n * groups * width, groups * width, width, 0)
    lout = (groups * n * (width + 3), width + 3, n * (width + 3), 0)
    full.run_pass((_lib.ptr(xt), _lib.ptr(yt), None, n, 0, blocks, groups, width, lin, lout, 2.0))
    got = yt.cpu().numpy()
    assert rel(got[..., :width], 2.0 * want.transpose(0, 2, 1, 3)) <= 1e-13
    assert np.all(got[..., width:] == 7.0)  # padding columns untouched
    # contiguous lines with pitches, fused core
    L = 9
    xl = rng.standard_normal((L, n + 5))
    core = rng.standard_normal((L, n + 5))
    xlt = torch.tensor(xl, device="cuda")
    ct = torch.tensor(core, device="cuda")
    ylt = torch.zeros((L, n + 1), dtype=torch.float64, device="cuda")
    full.run_pass((_lib.ptr(xlt), _lib.ptr(ylt), _lib.ptr(ct), n, 1, L, 1, 1, (0, 1, 0, n + 5), (0, 1, 0, n + 1), 1.0))
    # the core shares the input layout (pitch n+5): core row l starts at l*(n+5)
    cl = core[:, :n]
    want_l = oracle.dst(cl * oracle.dst(xl[:, :n], axis=1), axis=1)
    assert rel(ylt.cpu().numpy()[:, :n], want_l) <= 1e-13
    assert np.all(ylt.cpu().numpy()[:, n:] == 0.0)


def test_padded_errors():
    from paper_1809_01971_b200 import _lib
    spec = spectral.laplacian_spectrum(12, 3)  # not an FFT length
    with pytest.raises(ValueError):
        full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec, padded=True)
    assert not full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spec).padded
    x = torch.zeros((15, 15, 15), dtype=torch.float64, device="cuda")
    w = torch.zeros((15, 15, 16), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        _lib.call("fl_apply_full_padded", _lib.ptr(x), _lib.ptr(x), _lib.ptr(w), _lib.ptr(w), 3,
                  _lib.dims_arr((15, 15, 15)), 14, 1.0, _lib.stream_ptr())
    with pytest.raises(ValueError):
        full.run_pass((_lib.ptr(x), _lib.ptr(x), None, 12, 1, 1, 1, 1, (0, 1, 0, 12), (0, 1, 0, 12), 1.0))


@pytest.mark.parametrize("L", [1, 4, 15, 16, 37, 1000])
def test_dst1_core_lanes_matches_oracle(L):
    """Register-resident fused pass with the lane-ordered core (n = 511):
    ragged line counts (tiles of 16 lines, units of 4), in place, pitch 512."""
    from paper_1809_01971_b200 import _lib
    n = 511
    rng = np.random.default_rng(L)
    x = rng.standard_normal((L, n))
    core = rng.standard_normal((L, n))
    want = oracle.dst(core * oracle.dst(x, axis=1), axis=1)
    xp = torch.full((L, 512), 3.0, dtype=torch.float64, device="cuda")  # padding column must stay inert
    xp[:, :n] = torch.tensor(x, device="cuda")
    cl = full.line_lane_core(torch.tensor(core, device="cuda"))
    full.run_pass(("lanes", _lib.ptr(xp), _lib.ptr(xp), _lib.ptr(cl), L, 512, 2.0))
    got = xp.cpu().numpy()
    assert rel(got[:, :n], 2.0 * want) <= 1e-13
    assert np.all(got[:, n:] == 3.0)


@pytest.mark.parametrize("dims", [(511, 511), (511, 7, 511), (511, 63, 511)])
def test_apply_full_lanes_matches_oracle(dims):
    """fl_apply_full_lanes (register-resident passes, lane-ordered core) vs
    the oracle and vs the padded path with the natural core layout."""
    spec = spectral.EigenSpectrum(tuple(spectral.laplacian_mode(n) for n in dims))
    kind = CoreFunctionKind("g2", 0.75, coeff_minus=1.3, coeff_plus=0.7)
    op = full.FullOperator(spec, full.dense_core(kind, spec), lanes=True)
    assert op.lanes and op.padded and op.core_l is not None
    core_want = oracle.dense_core("g2", [oracle.laplacian_eigenvalues(n) for n in dims], 0.75, 1.3, 0.7)
    assert rel(op.core.cpu().numpy(), core_want) <= 1e-14
    rng = np.random.default_rng(sum(dims))
    x = rng.standard_normal(dims)
    xt = torch.tensor(x, device="cuda")
    want = oracle.apply_full(core_want, x)
    assert rel(op(xt).cpu().numpy(), want) <= 1e-12
    natural = full.FullOperator(spec, op.core.contiguous(), padded=True, lanes=False)
    assert rel(op(xt).cpu().numpy(), natural(xt).cpu().numpy()) <= 1e-13
    z = torch.empty_like(xt)
    for _, a in op.passes(xt, z):
        full.run_pass(a)
    assert rel(z.cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("blocks,inplace", [(40, True), (37, False)])
def test_dst1_pass_n511_many_tiles_per_cta(blocks, inplace):
    """n = 511 strided passes with more tiles than resident CTAs (TMA loads,
    TMA tensor stores through the CTA-wide staging, in place and not)."""
    from paper_1809_01971_b200 import _lib
    n, P = 511, 512
    g = torch.Generator(device="cuda")
    g.manual_seed(blocks)
    x = torch.randn((blocks, n, P), dtype=torch.float64, device="cuda", generator=g)
    want = oracle.dst(x.cpu().numpy(), axis=1)
    y = x if inplace else torch.full_like(x, 7.0)
    lay = (n * P, P, 0, 0)
    full.run_pass((_lib.ptr(x), _lib.ptr(y), None, n, 0, blocks, 1, P, lay, lay, 1.0))
    assert rel(y.cpu().numpy(), want) <= 1e-13


@pytest.mark.parametrize("width,groups,pad", [(5, 3, 0), (37, 2, 3), (16, 1, 0), (40, 2, 2), (511, 1, 1)])
def test_dst1_pass_n511_strided_layouts(width, groups, pad):
    """n = 511 strided passes through the register kernel with partial
    16-column chunks, odd widths (scalar sides), several groups and distinct
    input/output layouts; padding columns of the output stay untouched."""
    from paper_1809_01971_b200 import _lib
    n, blocks = 511, 2
    rng = np.random.default_rng(width * 7 + groups)
    x = rng.standard_normal((blocks, n, groups, width))
    want = oracle.dst(x, axis=1)
    xt = torch.tensor(x, device="cuda")
    wo = width + pad
    yt = torch.full((blocks, groups, n, wo), 7.0, dtype=torch.float64, device="cuda")
    lin = (n * groups * width, groups * width, width, 0)
    lout = (groups * n * wo, wo, n * wo, 0)
    full.run_pass((_lib.ptr(xt), _lib.ptr(yt), None, n, 0, blocks, groups, width, lin, lout, 0.5))
    got = yt.cpu().numpy()
    assert rel(got[..., :width], 0.5 * want.transpose(0, 2, 1, 3)) <= 1e-13
    assert np.all(got[..., width:] == 7.0)


@pytest.mark.parametrize("lines,pin,pout", [(1, 511, 512), (17, 511, 511), (33, 512, 515), (100, 515, 512), (16, 512, 512)])
def test_dst1_pass_n511_contiguous(lines, pin, pout):
    """n = 511 contiguous passes through the register kernel: dense (511),
    padded (512) and odd (515) pitches on either side, ragged line counts
    (bulk copies for whole 4-line units, cp.async with zero fill otherwise)."""
    from paper_1809_01971_b200 import _lib
    n = 511
    rng = np.random.default_rng(lines + pin)
    x = rng.standard_normal((lines, pin))
    want = oracle.dst(x[:, :n], axis=1)
    xt = torch.tensor(x, device="cuda")
    yt = torch.full((lines, pout), 7.0, dtype=torch.float64, device="cuda")
    full.run_pass((_lib.ptr(xt), _lib.ptr(yt), None, n, 1, lines, 1, 1, (0, 1, 0, pin), (0, 1, 0, pout), 1.0))
    got = yt.cpu().numpy()
    assert rel(got[:, :n], want) <= 1e-13
    assert np.all(got[:, n:] == 7.0)


def test_apply_lanes_bitwise_deterministic():
    """n = 511 lane apply: repeated runs, and in place vs out of place, agree
    bit for bit (the kernels are deterministic; a race or a stale padding
    column would show up as last-bit differences)."""
    n = 511
    op = full.FullOperator.from_kind(CoreFunctionKind("g1", 0.5), spectral.laplacian_spectrum(n, 3))
    g = torch.Generator(device="cuda")
    g.manual_seed(17)
    x = torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
    ref = op(x).clone()
    for _ in range(3):
        assert torch.equal(op(x), ref)
    z = x.clone()
    op(z, out=z)
    assert torch.equal(z, ref)


@pytest.mark.parametrize("blocks,width", [(3, 1024), (40, 48), (7, 30)])
def test_dst1_pass_n1023_strided(blocks, width):
    """n = 1023 strided passes with 16-byte aligned sides (register-resident
    N = 1024 kernel: TMA loads and stores, many tiles per CTA) vs scipy."""
    from paper_1809_01971_b200 import _lib
    n = 1023
    g = torch.Generator(device="cuda")
    g.manual_seed(blocks + width)
    x = torch.randn((blocks, n, width), dtype=torch.float64, device="cuda", generator=g)
    want = oracle.dst(x.cpu().numpy(), axis=1)
    y = torch.full_like(x, 7.0)
    lay = (n * width, width, 0, 0)
    full.run_pass((_lib.ptr(x), _lib.ptr(y), None, n, 0, blocks, 1, width, lay, lay, 1.0))
    assert rel(y.cpu().numpy(), want) <= 1e-13


def test_apply_full_padded_n1023():
    """Padded operator at n_0 = n_last = 1023 (the configs[3] size along two
    modes): mid passes on the N = 1024 register kernel, vs the oracle."""
    dims = (1023, 3, 1023)
    spec = spectral.EigenSpectrum(tuple(spectral.laplacian_mode(n) for n in dims))
    op = full.FullOperator.from_kind(CoreFunctionKind("g2", 0.75, coeff_minus=1.0, coeff_plus=1.0), spec)
    assert op.padded and op.pitch == 1024
    core = oracle.dense_core("g2", [oracle.laplacian_eigenvalues(n) for n in dims], 0.75, 1.0, 1.0)
    x = np.random.default_rng(1023).standard_normal(dims)
    got = op(torch.tensor(x, device="cuda")).cpu().numpy()
    assert rel(got, oracle.apply_full(core, x)) <= 1e-12


@pytest.mark.parametrize("lines,pin,pout", [(1, 1023, 1024), (17, 1023, 1023), (33, 1024, 1027), (100, 1027, 1024),
                                            (16, 1024, 1024)])
def test_dst1_pass_n1023_contiguous(lines, pin, pout):
    """n = 1023 contiguous passes through the N = 1024 register kernel: dense
    (1023), padded (1024) and odd (1027) pitches, ragged line counts (bulk
    copies for whole line pairs, cp.async with shifts and zero fill
    otherwise); the padding of the output stays untouched."""
    from paper_1809_01971_b200 import _lib
    n = 1023
    rng = np.random.default_rng(lines + pin + pout)
    x = rng.standard_normal((lines, pin))
    want = oracle.dst(x[:, :n], axis=1)
    xt = torch.tensor(x, device="cuda")
    yt = torch.full((lines, pout), 7.0, dtype=torch.float64, device="cuda")
    full.run_pass((_lib.ptr(xt), _lib.ptr(yt), None, n, 1, lines, 1, 1, (0, 1, 0, pin), (0, 1, 0, pout), 0.5))
    got = yt.cpu().numpy()
    assert rel(got[:, :n], 0.5 * want) <= 1e-13
    assert np.all(got[:, n:] == 7.0)


def test_transform_full_padded_n1023_deterministic():
    """The padded n = 1023 transform (contiguous pass, then two TMA-stored
    strided passes whose store drain overlaps the next tile) repeats bit for
    bit, and matches the dense-layout transform."""
    n = 1023
    dims = (n, 7, n)
    spec = spectral.EigenSpectrum(tuple(spectral.laplacian_mode(m) for m in dims))
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    x = torch.randn(dims, dtype=torch.float64, device="cuda", generator=g)
    ref = full.transform_full_padded(spec, x).clone()
    for _ in range(5):
        assert torch.equal(full.transform_full_padded(spec, x), ref)
    assert torch.all(ref[..., n:] == 0)
    dense = full.transform_full(spec, x)
    assert rel(ref[..., :n].cpu().numpy(), dense.cpu().numpy()) <= 1e-13
    back = full.transform_full_from_padded(spec, ref.clone())
    assert rel(back.cpu().numpy(), x.cpu().numpy()) <= 1e-13

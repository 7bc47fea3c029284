"""One launch each of the non-DST kernels, for ncu --set full (dev tool):
DMMA dense sine GEMM, spectral PCG, canonical apply (k_dst_fft KR loader),
Gram-Hadamard inner product, batched Jacobi SVD.  Also prints CUDA-event
times of the same launches (plain run)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import _lib, fullsolve, full, fracop, decomp, tensor


def ev(label, fn, flops=None, nbytes=None, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    extra = ""
    if flops:
        extra += " %.1f TFLOP/s" % (flops / ms / 1e9)
    if nbytes:
        extra += " %.0f GB/s" % (nbytes / ms / 1e6)
    print("%-34s %9.3f ms%s" % (label, ms, extra), flush=True)


which = sys.argv[1:] or ["dmma", "pcg", "canon", "svd"]
if "dmma" in which:
    n, inner = 1000, 65536
    x = torch.randn((1, n, inner), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ev("dmma dst1 n=1000 inner=65536", lambda: _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), 1, n, inner, 1.0,
                                                          _lib.stream_ptr()), flops=2.0 * n * n * inner)
    lines = torch.randn((65536, n), dtype=torch.float64, device="cuda")
    lo = torch.empty_like(lines)
    ev("dmma dst1 lines 65536 x n=1000", lambda: _lib.call("fl_dst1", _lib.ptr(lines), _lib.ptr(lo), 65536, n, 1,
                                                            1.0, _lib.stream_ptr()), flops=2.0 * n * n * 65536)
if "pcg" in which:
    n = 511
    spec = fl.laplacian_spectrum(n, 3)
    cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, precond_rank=6, residual_tol=1e-8, k_max=100)
    w, f = fl.gaussian_bumps(n, 3, 16, seed=7).weights, None
    y = full.cp_dense(fl.gaussian_bumps(n, 3, 16, seed=7))
    A, P = fullsolve.control_cores(cfg, spec, layout="padded")
    bh = full.transform_full_padded(spec, y)
    xh, r, p = torch.empty_like(bh), torch.empty_like(bh), torch.empty_like(bh)
    hist = torch.zeros(101, dtype=torch.float64, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    run = lambda: _lib.call("fl_pcg_spectral", _lib.ptr(bh), _lib.ptr(xh), _lib.ptr(r), _lib.ptr(p), _lib.ptr(A),
                            _lib.ptr(P), bh.numel(), 1e-8, 100, _lib.ptr(hist), _lib.ptr(st), _lib.stream_ptr())
    run(); torch.cuda.synchronize()
    its = int(st[0])
    # bytes: init 5 reads/writes... count per iteration 96 B/DoF (+ init 48)
    ev("pcg_spectral n=511 (%d its)" % its, run, nbytes=(64.0 * its + 48.0) * bh.numel())
if "canon" in which:
    n = 127
    spec = fl.laplacian_spectrum(n, 3)
    kind = fl.CoreFunctionKind("g2", 0.5, coeff_minus=1e-2, coeff_plus=1e2)
    op = fl.LowRankOperator(fl.build_core(kind, spec, fl.TruncationSpec(tolerance=1e-8)))
    rng = np.random.default_rng(3)
    x = fl.CpTensor(rng.standard_normal(200), [rng.standard_normal((n, 200)) for _ in range(3)])
    ev("canonical apply R=%d S=200 n=127" % op.diag.core.rank, lambda: fracop.apply(op, x))
    yv = fracop.apply(op, x)
    ev("cp_inner rank %d" % yv.rank, lambda: tensor.cp_inner(yv, x))
if "svd" in which:
    A = torch.randn((64, 64, 64), dtype=torch.float64, device="cuda")
    ev("svd_batched 64 x (64x64)", lambda: decomp.svd_batched(A))

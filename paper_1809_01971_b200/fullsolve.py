"""Full-format control and state solves (dense n^d tensors on the device).

The reference solves the control equation (solver.py:203-231)
    (beta A^-alpha + (gamma/beta) A^alpha) u = y_design
by PCG with the rank-r Kronecker preconditioner (solver.py:183-189) in
canonical arithmetic.  On dense tensors both the system operator and the
preconditioner are F diag(.) F with the same orthonormal DST-I basis F, so
the PCG iteration runs on spectral coefficients (fl_pcg_spectral: one
cooperative persistent kernel for the whole solve).  mode="nodal" runs the
same iteration with an explicit F diag F application per operator call (the
literal Algorithm 1 on dense tensors) for validation.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .fracop import CoreFunctionKind, dense_core_dev
from .full import (apply_full, cp_dense, dense_core, padded_pitch, padded_transform_ok, to_padded, transform_full,
                   transform_full_from_padded, transform_full_padded)
from .solver import PcgBreakdownError, PcgReport, SolverConfig, build_preconditioner

__all__ = ["control_cores", "pcg_full", "solve_control_full", "solve_state_full"]


def _control_kind(cfg):
    return CoreFunctionKind("g2", cfg.alpha, coeff_minus=float(cfg.beta), coeff_plus=float(cfg.gamma) / float(cfg.beta))


def control_cores(cfg, spectrum, precond="kronecker", seed=0, layout="dense"):
    """Dense system core A = g2(beta, gamma/beta) and preconditioner core P.

    precond: "kronecker" (the reference's rank-r reciprocal core, expanded to
    dense), "exact" (1/g2, i.e. g3), or "identity".  layout="padded" returns
    them in the padded layout (zero padding) that pcg_full runs on with the
    register-resident transforms (when padded_transform_ok(spectrum)).
    """
    kind = _control_kind(cfg)
    A = dense_core(kind, spectrum)
    if precond == "kronecker":
        pre = kronecker_preconditioner(cfg, spectrum, seed)
        P = cp_dense(pre.diag.core)
    elif precond == "exact":
        P = dense_core(kind, spectrum, reciprocal=True)
    elif precond == "identity":
        P = torch.ones_like(A)
    else:
        raise ValueError("precond must be 'kronecker', 'exact' or 'identity'")
    if layout == "padded" and padded_transform_ok(spectrum):
        return to_padded(A), to_padded(P)
    if layout not in ("dense", "padded"):
        raise ValueError("layout must be 'dense' or 'padded'")
    return A, P


def kronecker_preconditioner(cfg, spectrum, seed=0):
    """The reference's rank-r reciprocal core (solver.py:183-189), built on the
    device with the dense-level cap lifted to the full grid."""
    from .decomp import dense_budget
    kind = _control_kind(cfg)
    total = int(np.prod(spectrum.mode_sizes, dtype=np.int64))
    with dense_budget(max(total, 2 ** 24)):
        return build_preconditioner(kind, spectrum, cfg.precond_rank, seed=seed)


def pcg_full(spectrum, A, P, b, tol, k_max, mode="spectral"):
    """PCG for F diag(A) F x = b with preconditioner F diag(P) F on dense tensors.

    Returns (x, PcgReport).  Raises PcgBreakdownError on <R,Z> <= 0 or
    <P,S> <= 0 exactly as the reference (solver.py:154-159).
    """
    if mode == "nodal":
        nl = spectrum.mode_sizes[-1]
        if A.shape[-1] != nl:  # padded-layout cores: the literal iteration wants dense ones
            A, P = A[..., :nl].contiguous(), P[..., :nl].contiguous()
        return _pcg_nodal(spectrum, A, P, b, tol, k_max)
    if mode != "spectral":
        raise ValueError("mode must be 'spectral' or 'nodal'")
    dev = b.device
    dims = tuple(spectrum.mode_sizes)
    padded = padded_transform_ok(spectrum) and tuple(A.shape) == dims[:-1] + (padded_pitch(dims[-1]),)
    if padded:
        # cores in the padded layout (zero padding): the iteration runs on
        # padded spectral coefficients (the padding stays zero: P_pad = 0 keeps
        # the search directions there at zero), both transforms on the
        # register-resident kernels
        if tuple(P.shape) != tuple(A.shape):
            raise ValueError("A and P must share the (padded) layout")
        bh = transform_full_padded(spectrum, b)
    else:
        bh = transform_full(spectrum, b)
    N = bh.numel()
    xh = torch.empty_like(bh)
    r = torch.empty_like(bh)
    p = torch.empty_like(bh)
    hist = torch.zeros(int(k_max) + 1, dtype=torch.float64, device=dev)
    status = torch.zeros(4, dtype=torch.int32, device=dev)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    _lib.call("fl_pcg_spectral", _lib.ptr(bh), _lib.ptr(xh), _lib.ptr(r), _lib.ptr(p), _lib.ptr(A), _lib.ptr(P),
              N, float(tol), int(k_max), _lib.ptr(hist), _lib.ptr(status), _lib.stream_ptr())
    end.record()
    x = (transform_full_from_padded(spectrum, xh) if padded
         else transform_full(spectrum, xh, direction="inverse"))
    st = status.cpu().numpy()
    its, conv, bk_it, bk_kind = (int(v) for v in st)
    if bk_kind:
        raise PcgBreakdownError(bk_it, float(hist[bk_it]), what="<R, Z>" if bk_kind == 1 else "<P, S>")
    torch.cuda.synchronize()
    secs = start.elapsed_time(end) / 1e3
    residuals = hist[: its + 1].cpu().numpy().tolist() if its else [float(hist[0])]
    per = secs / its if its else 0.0
    return x, PcgReport(iterations=its, residuals=residuals, final_rank=0, converged=bool(conv),
                        iteration_seconds=[per] * its, seconds_per_iteration=per)


def _pcg_nodal(spectrum, A, P, b, tol, k_max):
    """The literal iteration with F diag F applications (validation path)."""
    def fun(v):
        return apply_full(spectrum, A, v.contiguous())

    def pre(v):
        return apply_full(spectrum, P, v.contiguous())

    def dot(u, v):
        return float(torch.dot(u.reshape(-1), v.reshape(-1)))

    norm_b = dot(b, b) ** 0.5
    x = torch.zeros_like(b)
    if norm_b == 0.0:
        return x, PcgReport(iterations=0, residuals=[0.0], converged=True)
    r = b.clone()
    residuals = [1.0]
    z = pre(r)
    p = z.clone()
    rz = dot(r, z)
    its, conv = 0, False
    for k in range(1, int(k_max) + 1):
        if rz <= 0.0:
            raise PcgBreakdownError(k, rz, what="<R, Z>")
        s = fun(p)
        ps = dot(p, s)
        if ps <= 0.0:
            raise PcgBreakdownError(k, ps)
        step = rz / ps
        x.add_(p, alpha=step)
        r.add_(s, alpha=-step)
        rel = dot(r, r) ** 0.5 / norm_b
        residuals.append(rel)
        its = k
        if rel <= tol:
            conv = True
            break
        z = pre(r)
        rzn = dot(r, z)
        p = z + (rzn / rz) * p
        rz = rzn
    return x, PcgReport(iterations=its, residuals=residuals, converged=conv)


def solve_control_full(y_design, cfg, spectrum, precond="kronecker", mode="spectral", seed=0, cores=None):
    """Optimal control on dense tensors: PCG on the g2 system (solver.py:203-216)."""
    if not isinstance(cfg, SolverConfig):
        raise ValueError("expected a SolverConfig")
    if tuple(y_design.shape) != tuple(spectrum.mode_sizes):
        raise ValueError("design function dims do not match the spectrum")
    if cores is None:
        cores = control_cores(cfg, spectrum, precond, seed, layout="padded" if mode == "spectral" else "dense")
    A, P = cores
    return pcg_full(spectrum, A, P, y_design, cfg.residual_tol, cfg.k_max, mode)


def solve_state_full(y_design, cfg, spectrum):
    """y = (I + (gamma/beta^2) A^(2 alpha))^-1 y_design: one g4 application (solver.py:245-249)."""
    kind = CoreFunctionKind("g4", cfg.alpha, coeff_plus=float(cfg.gamma) / float(cfg.beta) ** 2)
    return apply_full(spectrum, dense_core(kind, spectrum), y_design)

"""Full-format (dense n^d) operator functions of the separable Laplacian.

The reference applies F(A) only to canonical tensors; its dense oracle
(tests/oracles.py:56 dense_apply) is F diag(G) F^T x on a full array.  This
module is that full-format path on the device: G is a dense core tensor
resident in HBM (evaluated once per operator by fl_core_eval, or expanded
from a canonical core by fl_cp_to_dense), and every application is one
fl_apply_full call: per-mode DST-I passes with the last mode's forward
transform, core scaling and inverse transform fused into one kernel.
FullOperator additionally pads the last mode's rows to a 128-byte multiple
(fl_apply_full_padded) so the intermediate passes run on aligned rows.
"""

from __future__ import annotations

import os

import numpy as np

import torch

from . import _lib
from .fracop import CoreFunctionKind, mode_values_device
from .spectral import EigenSpectrum, transform_axis

__all__ = ["FullOperator", "padded_pitch", "run_pass", "dense_core", "apply_full", "transform_full", "apply_host_stream", "inner", "norm",
           "transform_full_padded", "transform_full_from_padded", "to_padded", "padded_transform_ok"]


def _shape_check(spectrum, x):
    if tuple(x.shape) != tuple(spectrum.mode_sizes):
        raise ValueError("operand dims %r do not match operator dims %r"
                         % (tuple(x.shape), spectrum.mode_sizes))


def dense_core(kind, spectrum, reciprocal=False, device=None):
    """g(rho) on the full eigenvalue grid (fracop.py:138-148), evaluated on the device."""
    if not isinstance(kind, CoreFunctionKind):
        raise ValueError("expected a CoreFunctionKind")
    _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    mus, a = mode_values_device(kind, spectrum, dev)
    out = torch.empty(spectrum.mode_sizes, dtype=torch.float64, device=dev)
    _lib.call("fl_core_eval", _lib.ptr(out), spectrum.d, _lib.dims_arr(spectrum.mode_sizes),
              _lib.ptr_arr(mus), _lib.TAGS.index(kind.tag), float(a), float(kind.coeff_minus),
              float(kind.coeff_plus), 1 if reciprocal else 0, _lib.stream_ptr())
    return out


def cp_dense(cp, device=None):
    """Dense expansion of a canonical tensor on the device (tensor.py:217-225)."""
    dims = cp.dims
    out = torch.empty(dims, dtype=torch.float64, device=cp.weights.device)
    _lib.call("fl_cp_to_dense", _lib.ptr(out), len(dims), _lib.dims_arr(dims), cp.rank,
              _lib.ptr(cp.weights), _lib.ptr_arr(list(cp.factors)), _lib.stream_ptr())
    return out


def _check_operand(x):
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64:
        raise ValueError("full-format operands are float64 CUDA tensors")
    if not x.is_contiguous():
        raise ValueError("full-format operands must be contiguous (C order)")


def apply_full(spectrum, core, x, alpha=1.0, out=None):
    """out = alpha * F diag(core) F x."""
    _check_operand(x)
    _shape_check(spectrum, x)
    y = out if out is not None else torch.empty_like(x)
    if spectrum.all_sine:
        _lib.call("fl_apply_full", _lib.ptr(x), _lib.ptr(y), _lib.ptr(core), spectrum.d,
                  _lib.dims_arr(spectrum.mode_sizes), float(alpha), _lib.stream_ptr())
        return y
    z = x
    for ax, m in enumerate(spectrum.modes):
        z = transform_axis(m, z.contiguous(), "forward", ax)
    z = z * core
    for ax, m in enumerate(spectrum.modes):
        z = transform_axis(m, z.contiguous(), "inverse", ax)
    if alpha != 1.0:
        z = z * alpha
    y.copy_(z)
    return y


def transform_full(spectrum, x, direction="forward", alpha=1.0, out=None):
    """Full spectral transform over all modes (forward F or inverse F^T)."""
    _check_operand(x)
    _shape_check(spectrum, x)
    y = out if out is not None else torch.empty_like(x)
    if spectrum.all_sine:
        _lib.call("fl_transform_full", _lib.ptr(x), _lib.ptr(y), spectrum.d,
                  _lib.dims_arr(spectrum.mode_sizes), float(alpha), _lib.stream_ptr())
        return y
    z = x
    for ax, m in enumerate(spectrum.modes):
        z = transform_axis(m, z.contiguous(), direction, ax)
    y.copy_(z * alpha if alpha != 1.0 else z)
    return y


def padded_transform_ok(spectrum):
    """Whether the padded spectral layout (last mode of pitch padded_pitch(n))
    applies: sine modes of FFT length, d = 2 or 3, last mode not a multiple
    of 16."""
    dims = tuple(spectrum.mode_sizes)
    return (spectrum.all_sine and len(dims) in (2, 3) and all(_fft_length(n) for n in dims)
            and dims[-1] % 16 != 0)


def _padded_passes(dims, P):
    """(first contiguous pass layouts, strided passes) of the padded transform."""
    nl = dims[-1]
    lines = 1
    for n in dims[:-1]:
        lines *= n
    strided = []
    if len(dims) == 3:
        n0, n1 = dims[0], dims[1]
        mid = (n1 * P, P, 0, 0)
        strided.append((n1, n0, 1, P, mid))
        strided.append((n0, 1, n1, P, (0, n1 * P, P, 0)))
    else:
        strided.append((dims[0], 1, 1, P, (0, P, 0, 0)))
    return lines, strided


def transform_full_padded(spectrum, x):
    """F x for a dense x, returned in the padded layout (last mode of pitch
    padded_pitch(n), padding zero): the last mode as contiguous lines (dense
    rows -> padded rows), then the other modes on aligned strided layouts, so
    every pass can run on the register-resident kernels."""
    _check_operand(x)
    _shape_check(spectrum, x)
    dims = tuple(spectrum.mode_sizes)
    nl, P = dims[-1], padded_pitch(dims[-1])
    out = torch.empty(dims[:-1] + (P,), dtype=torch.float64, device=x.device)
    lines, strided = _padded_passes(dims, P)
    xp, op_ = _lib.ptr(x), _lib.ptr(out)
    # flag 3 = contiguous | FL_PASS_PAD_WRITE: the padding is zeroed
    run_pass((xp, op_, None, nl, 3, lines, 1, 1, (0, 1, 0, nl), (0, 1, 0, P), 1.0))
    for n, outer, groups, width, lay in reversed(strided):
        run_pass((op_, op_, None, n, 0, outer, groups, width, lay, lay, 1.0))
    out[..., nl:].zero_()  # the strided passes leave rounding noise in the padding
    return out


def transform_full_from_padded(spectrum, xp, alpha=1.0, out=None):
    """Inverse of transform_full_padded (F is involutive): xp (padded layout,
    consumed: transformed in place) -> dense alpha * F xp."""
    dims = tuple(spectrum.mode_sizes)
    nl, P = dims[-1], padded_pitch(dims[-1])
    if tuple(xp.shape) != dims[:-1] + (P,) or not xp.is_contiguous():
        raise ValueError("expected a contiguous padded-layout tensor of shape %r" % (dims[:-1] + (P,),))
    y = out if out is not None else torch.empty(dims, dtype=torch.float64, device=xp.device)
    lines, strided = _padded_passes(dims, P)
    p_ = _lib.ptr(xp)
    for n, outer, groups, width, lay in strided:
        run_pass((p_, p_, None, n, 0, outer, groups, width, lay, lay, 1.0))
    run_pass((p_, _lib.ptr(y), None, nl, 1, lines, 1, 1, (0, 1, 0, P), (0, 1, 0, nl), float(alpha)))
    return y


def to_padded(t, fill=0.0):
    """Copy of a dense tensor in the padded layout (padding = fill)."""
    dims = tuple(t.shape)
    P = padded_pitch(dims[-1])
    out = torch.full(dims[:-1] + (P,), float(fill), dtype=torch.float64, device=t.device)
    out[..., :dims[-1]].copy_(t)
    return out


def _fft_length(n):
    return 4 <= n + 1 <= 8192 and (n + 1) & n == 0


def padded_pitch(n):
    """Row pitch of the padded internal layout for a last mode of size n:
    the next multiple of 16 doubles (128 B), e.g. 512 for n = 511."""
    return (n + 15) // 16 * 16


def line_lane_core(core):
    """Lane order of a core over contiguous lines (fl_dst1_core_lanes):
    lines = all but the last mode (n_last = 511), padded to a multiple of
    16; rows 1-based in [0, 512) with row 0 = 0."""
    n = core.shape[-1]
    if n != 511:
        raise ValueError("lane order is defined for n_last = 511")
    L = core.numel() // n
    Lp = (L + 15) // 16 * 16
    c = torch.zeros((Lp, 512), dtype=torch.float64, device=core.device)
    c[:L, 1:].copy_(core.reshape(L, n))
    # line = 4u + 2f + e, row = 32q + i  ->  [u][i][f][q][e]
    return c.reshape(Lp // 4, 2, 2, 16, 32).permute(0, 4, 1, 3, 2).contiguous()


def lane_core(core):
    """The core of an operator with n_0 = n_last = 511 in the mode-0 lane
    order read by the fused pass of fl_apply_full_lanes (see
    include/fraclap_b200.h): G padded to [511][n1][512], unit
    u = (i1 * 32 + c) * 4 + w over columns 16c + 4w + (2f + e), entry
    [u][i][f][q][e] = G[32q + i - 1][i1][16c + 4w + 2f + e] (row 0 = 0)."""
    if core.shape[0] != 511 or core.shape[-1] != 511:
        raise ValueError("mode-0 lane order is defined for n_0 = n_last = 511")
    g = core.numel() // (511 * 511)
    c = torch.zeros((512, g, 512), dtype=torch.float64, device=core.device)
    c[1:, :, :511].copy_(core.reshape(511, g, 511))
    # r = 32q + i, column = 16c + 4w + 2f + e  ->  [g][c][w][i][f][q][e]
    c = c.reshape(16, 32, g, 32, 4, 2, 2).permute(2, 3, 4, 1, 5, 0, 6)
    return c.reshape(g * 128, 32, 2, 16, 2).contiguous()


def lane_core_inverse(core_l, dims):
    """Dense core (dims) from its mode-0 lane order (inverse of lane_core)."""
    g = 1
    for d in dims[1:-1]:
        g *= d
    c = core_l.reshape(g, 32, 4, 32, 2, 16, 2).permute(5, 3, 0, 1, 2, 4, 6).reshape(512, g, 512)
    return c[1:, :, :511].reshape(dims).contiguous()


class FullOperator:
    """alpha * F diag(G) F on dense tensors; G resident in HBM.

    When every mode is an FFT length (n+1 a power of two) and the last mode
    is not already a multiple of 16, the operator keeps G in a padded
    layout (last-mode rows of pitch `padded_pitch(n)`, so every row starts
    on a 128-byte boundary) together with a padded work tensor, and applies
    through fl_apply_full_padded: the first pass reads x into the padded
    layout, the last writes y back dense.  `core` is then a view of the
    valid part.  The work tensor makes one operator single-stream: concurrent
    applications of the same operator on different streams would race."""

    def __init__(self, spectrum, core, alpha=1.0, padded=None, lanes=None):
        if not isinstance(spectrum, EigenSpectrum):
            raise ValueError("expected an EigenSpectrum")
        if tuple(core.shape) != tuple(spectrum.mode_sizes):
            raise ValueError("core dims do not match the spectrum")
        self.spectrum = spectrum
        self.alpha = float(alpha)
        dims = tuple(spectrum.mode_sizes)
        can_pad = spectrum.all_sine and len(dims) in (2, 3) and all(_fft_length(n) for n in dims)
        if padded is None:
            padded = can_pad and dims[-1] % 16 != 0
        if padded and not can_pad:
            raise ValueError("the padded layout needs sine modes of FFT length")
        self.pitch = padded_pitch(dims[-1]) if padded else None
        lane_dims = dims[0] == 511 and dims[-1] == 511
        if lanes is None:
            lanes = bool(padded) and lane_dims and os.environ.get("FL_REG", "1") != "0"
        if lanes and not (padded and lane_dims):
            raise ValueError("the lane-ordered core is defined for a padded operator with n_0 = n_last = 511")
        self.lanes = bool(lanes)
        self.core_p = self.core_l = None
        if padded:
            pshape = dims[:-1] + (self.pitch,)
            if self.lanes:
                self.core_l = lane_core(core)
            else:
                self.core_p = torch.zeros(pshape, dtype=torch.float64, device=core.device)
                self.core_p[..., :dims[-1]].copy_(core)
            self.work = torch.zeros(pshape, dtype=torch.float64, device=core.device)
            self._core = None
        else:
            self.work = None
            self._core = core.contiguous()
        for m in spectrum.modes:
            _lib.call("fl_prepare", m.n)

    @classmethod
    def from_kind(cls, kind, spectrum, reciprocal=False, device=None, padded=None):
        return cls(spectrum, dense_core(kind, spectrum, reciprocal, device), padded=padded)

    @classmethod
    def from_cp(cls, spectrum, cp, padded=None):
        return cls(spectrum, cp_dense(cp), padded=padded)

    @property
    def dims(self):
        return self.spectrum.mode_sizes

    @property
    def padded(self):
        return self.pitch is not None

    @property
    def core(self):
        """The dense core G (a view of the padded storage when padded)."""
        if self._core is not None:
            return self._core
        if self.core_l is not None:
            return lane_core_inverse(self.core_l, tuple(self.dims))
        return self.core_p[..., :self.dims[-1]]

    def __call__(self, x, out=None):
        if not self.padded:
            return apply_full(self.spectrum, self._core, x, self.alpha, out)
        _check_operand(x)
        _shape_check(self.spectrum, x)
        if x.device != self.work.device:
            raise ValueError("operand on %s, operator on %s" % (x.device, self.work.device))
        y = out if out is not None else torch.empty_like(x)
        if self.lanes:
            _lib.call("fl_apply_full_lanes", _lib.ptr(x), _lib.ptr(y), _lib.ptr(self.core_l), _lib.ptr(self.work),
                      len(self.dims), _lib.dims_arr(self.dims), self.alpha, _lib.stream_ptr())
            return y
        _lib.call("fl_apply_full_padded", _lib.ptr(x), _lib.ptr(y), _lib.ptr(self.core_p), _lib.ptr(self.work),
                  len(self.dims), _lib.dims_arr(self.dims), self.pitch, self.alpha, _lib.stream_ptr())
        return y

    def passes(self, x, y):
        """The DST passes of one application as (name, fl_dst1_pass args)
        tuples, in launch order (for per-pass timing; same launches as
        __call__ on a padded operator)."""
        if not self.padded:
            raise ValueError("per-pass list is defined for the padded layout")
        dims, P = tuple(self.dims), self.pitch
        nl = dims[-1]
        xp, yp, wp = _lib.ptr(x), _lib.ptr(y), _lib.ptr(self.work)
        cp = _lib.ptr(self.core_l if self.lanes else self.core_p)
        if self.lanes:
            # fl_apply_full_lanes: last mode contiguous (dense rows -> padded),
            # mode 1, mode 0 fused with the core, mode 1, last mode back
            n1 = dims[1] if len(dims) == 3 else 1
            lines = dims[0] * n1
            dl, pl = (0, 1, 0, nl), (0, 1, 0, P)
            mid = (n1 * P, P, 0, 0)
            # flags 1 | 2 = contiguous | FL_PASS_PAD_WRITE (the padding position is zeroed)
            out = [("dst_mode2", (xp, wp, None, nl, 3, lines, 1, 1, dl, pl, 1.0))]
            if len(dims) == 3:
                out.append(("dst_mode1", (wp, wp, None, n1, 0, dims[0], 1, P, mid, mid, 1.0)))
            out.append(("dst_core_mode0", ("lanes0", wp, wp, cp, n1, 1.0)))
            if len(dims) == 3:
                out.append(("dst_mode1", (wp, wp, None, n1, 0, dims[0], 1, P, mid, mid, 1.0)))
            out.append(("dst_mode2", (wp, yp, None, nl, 1, lines, 1, 1, pl, dl, self.alpha)))
            return out
        if len(dims) == 2:
            n0 = dims[0]
            dense, pad, line = (0, nl, 0, 0), (0, P, 0, 0), (0, 1, 0, P)
            fused = (wp, wp, cp, nl, 1, n0, 1, 1, line, line, 1.0)
            # flag 2 = FL_PASS_PAD_WRITE: the first pass may write the work tensor's padding
            return [("dst_mode0", (xp, wp, None, n0, 2, 1, 1, nl, dense, pad, 1.0)),
                    ("dst_core_mode1", fused),
                    ("dst_mode0", (wp, yp, None, n0, 0, 1, 1, nl, pad, dense, self.alpha))]
        n0, n1 = dims[0], dims[1]
        dense0, pad0 = (0, n1 * nl, nl, 0), (0, n1 * P, P, 0)
        mid, line = (n1 * P, P, 0, 0), (0, 1, 0, P)
        fused = (wp, wp, cp, nl, 1, n0 * n1, 1, 1, line, line, 1.0)
        # flag 2 = FL_PASS_PAD_WRITE: the first pass may write the work tensor's padding
        return [("dst_mode0", (xp, wp, None, n0, 2, 1, n1, nl, dense0, pad0, 1.0)),
                ("dst_mode1", (wp, wp, None, n1, 0, n0, 1, P, mid, mid, 1.0)),
                ("dst_core_mode2", fused),
                ("dst_mode1", (wp, wp, None, n1, 0, n0, 1, P, mid, mid, 1.0)),
                ("dst_mode0", (wp, yp, None, n0, 0, 1, n1, nl, pad0, dense0, self.alpha))]


def run_pass(args, stream=None):
    """Launch one fl_dst1_pass from a FullOperator.passes() entry."""
    s = _lib.stream_ptr() if stream is None else stream
    if args[0] == "lanes":
        _, x, y, c, lines, pitch, scale = args
        _lib.call("fl_dst1_core_lanes", x, y, c, lines, pitch, float(scale), s)
        return
    if args[0] == "lanes0":
        _, x, y, c, groups, scale = args
        _lib.call("fl_dst1_core_lanes_mode0", x, y, c, groups, float(scale), s)
        return
    x, y, c, n, contig, outer, groups, width, lin, lout, scale = args
    _lib.call("fl_dst1_pass", x, y, c, n, contig, outer, groups, width, _lib.dims_arr(lin), _lib.dims_arr(lout),
              float(scale), s)


def apply_host_stream(op, host_inputs, host_outputs, device=None):
    """Apply `op` to a sequence of host (pinned) tensors, writing host outputs.

    Three CUDA streams pipeline the steps: while step i computes, step i+1's
    input crosses PCIe host->device and step i-1's result crosses
    device->host (PCIe is full duplex), with two device buffers per side.
    Returns the list of host outputs (the `host_outputs` tensors, filled)."""
    if len(host_inputs) != len(host_outputs):
        raise ValueError("need one output buffer per input")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    shape = tuple(op.dims)
    h2d, comp, d2h = (torch.cuda.Stream(dev) for _ in range(3))
    xin = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(2)]
    yout = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    drained = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    cur = torch.cuda.current_stream(dev)
    for s in (h2d, comp, d2h):
        s.wait_stream(cur)
    for i, (xh, yh) in enumerate(zip(host_inputs, host_outputs)):
        b = i & 1
        with torch.cuda.stream(h2d):
            if i >= 2:
                h2d.wait_event(consumed[b])
            xin[b].copy_(xh, non_blocking=True)
            loaded[b].record(h2d)
        with torch.cuda.stream(comp):
            comp.wait_event(loaded[b])
            if i >= 2:
                comp.wait_event(drained[b])
            op(xin[b], out=yout[b])
            consumed[b].record(comp)
            done[b].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[b])
            yh.copy_(yout[b], non_blocking=True)
            drained[b].record(d2h)
    for s in (h2d, comp, d2h):
        cur.wait_stream(s)
    return host_outputs


def inner(a, b):
    return float(torch.dot(a.reshape(-1), b.reshape(-1)))


def norm(a):
    return float(torch.linalg.vector_norm(a.reshape(-1)))

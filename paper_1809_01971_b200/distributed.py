"""Slab-partitioned 3D full-format operators and PCG across GPUs.

Layouts (n0 x n1 x n2 tensor, P ranks, one process per GPU):
  nodal    rank r holds planes i0 in X_r            -> (|X_r|, n1, n2) dense
  spectral rank r holds the transform for i1 in S_r -> (n0, |S_r|, P)
with P = padded_pitch(n2) (1024 for n = 1023, padding zero) when every mode
is an FFT length, so every strided pass runs on aligned rows (the register-
resident TMA kernels), else P = n2.  Forward transform: DST-I along modes 2
and 1 inside the slab (dense rows -> padded rows), an all-to-all transpose
(one torch.distributed.all_to_all_single over NCCL / NVLink), DST-I along
mode 0 on the transposed slab.  The inverse runs the same steps backwards.
Cores (system operator, preconditioner) are evaluated directly in the
spectral layout, so the PCG iteration is one fused streaming pass
(fl_pcg_phase) plus ONE all-reduce of 4 scalars per iteration; the two
all-to-alls happen once per solve (b -> b_hat, x_hat -> x).  The rank-r
Kronecker preconditioner core is built on rank 0 and broadcast
(broadcast_cp), not rebuilt on every rank.

The compute primitives come from an ops object; `CudaOps` binds them to
libfraclap_b200 (the product).  Tests substitute a host implementation to
exercise the decomposition, transposes and reduction logic with gloo on CPU,
and drive `CudaOps` with gloo (host-staged collectives) from two ranks on one
GPU.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["split", "SlabLayout", "CudaOps", "transform_fwd", "transform_bwd", "apply_slab", "pcg_slab",
           "broadcast_cp", "spectral_core", "spectral_cp_core"]


def split(n, parts):
    """Balanced contiguous ranges [(start, stop)] covering range(n)."""
    base, rem = divmod(int(n), int(parts))
    out, s = [], 0
    for q in range(parts):
        e = s + base + (1 if q < rem else 0)
        out.append((s, e))
        s = e
    return out


class SlabLayout:
    def __init__(self, dims, world, rank):
        if len(dims) != 3:
            raise ValueError("slab partitioning is for 3D tensors")
        self.dims = tuple(int(n) for n in dims)
        self.world, self.rank = int(world), int(rank)
        self.X = split(self.dims[0], world)  # nodal slabs over i0
        self.S = split(self.dims[1], world)  # spectral slabs over i1

    @property
    def nodal_shape(self):
        s, e = self.X[self.rank]
        return (e - s, self.dims[1], self.dims[2])

    @property
    def spectral_shape(self):
        s, e = self.S[self.rank]
        return (self.dims[0], e - s, self.dims[2])


class CudaOps:
    """Local compute through libfraclap_b200 (device tensors).

    When every mode is an FFT length the spectral slabs use the padded
    layout of the single-GPU path (last mode of pitch padded_pitch(n2), e.g.
    1024 for n = 1023, padding zero): the first pass writes the padded
    layout, so every strided pass (mode 1 in the nodal slab, mode 0 in the
    spectral slab) runs on 16-byte aligned rows, i.e. on the register-
    resident TMA kernels instead of the CTA kernel of odd-width layouts."""

    def pitch(self, lay):
        from .full import _fft_length, padded_pitch
        n2 = lay.dims[2]
        return padded_pitch(n2) if all(_fft_length(n) for n in lay.dims) else n2

    def dst_inner_fwd(self, x, P):
        """DST-I along modes 2 and 1 of a dense (m, n1, n2) slab into a new
        (m, n1, P) tensor whose padding columns are zero (x is untouched)."""
        m, n1, n2 = x.shape
        y = torch.empty((m, n1, P), dtype=torch.float64, device=x.device)
        if m == 0:
            return y
        x = x.contiguous()
        st = _lib.stream_ptr()
        if P == n2:
            _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), m * n1, n2, 1, 1.0, st)
            _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(y), m, n1, n2, 1.0, st)
            return y
        # flag 3 = contiguous | FL_PASS_PAD_WRITE: dense rows -> padded rows
        _pass(x, y, n2, 3, m * n1, 1, 1, (0, 1, 0, n2), (0, 1, 0, P), 1.0, st)
        _pass(y, y, n1, 0, m, 1, P, (n1 * P, P, 0, 0), (n1 * P, P, 0, 0), 1.0, st)
        y[..., n2:].zero_()  # the strided pass leaves rounding noise in the padding
        return y

    def dst_inner_bwd(self, y, n2, scale=1.0):
        """Inverse of dst_inner_fwd: (m, n1, P) -> dense (m, n1, n2), scaled.
        y is a temporary of the caller and is transformed in place."""
        m, n1, P = y.shape
        x = torch.empty((m, n1, n2), dtype=torch.float64, device=y.device)
        if m == 0:
            return x
        st = _lib.stream_ptr()
        if P == n2:
            _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(y), m, n1, n2, 1.0, st)
            _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(x), m * n1, n2, 1, float(scale), st)
            return x
        _pass(y, y, n1, 0, m, 1, P, (n1 * P, P, 0, 0), (n1 * P, P, 0, 0), 1.0, st)
        _pass(y, x, n2, 1, m * n1, 1, 1, (0, 1, 0, P), (0, 1, 0, n2), float(scale), st)
        return x

    def dst_mode0(self, y, scale=1.0):
        """DST-I along mode 0 of a (n0, m, P) slab into a new tensor."""
        n0, m, P = y.shape
        if m * P == 0:
            return y.clone()
        y = y.contiguous()
        out = torch.empty_like(y)
        _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(out), 1, n0, m * P, float(scale), _lib.stream_ptr())
        return out

    def pcg_phase(self, phase, b, x, r, p, A, P, alpha, beta, out, work):
        _lib.call("fl_pcg_phase", phase, _lib.ptr(b), _lib.ptr(x), _lib.ptr(r), _lib.ptr(p), _lib.ptr(A),
                  _lib.ptr(P), b.numel(), float(alpha), float(beta), _lib.ptr(out), _lib.ptr(work),
                  _lib.stream_ptr())

    def new_work(self, like):
        return torch.zeros(_lib.FL_PCG_WORK, dtype=torch.float64, device=like.device)


def _pass(x, y, n, flags, outer, groups, width, lin, lout, scale, st):
    _lib.call("fl_dst1_pass", _lib.ptr(x), _lib.ptr(y), None, n, flags, outer, groups, width, _lib.dims_arr(lin),
              _lib.dims_arr(lout), float(scale), st)


def _staged(t):
    """Collectives of a host-only backend (gloo) on device tensors go through
    host copies (used by the one-GPU multi-rank test; NCCL takes device
    tensors directly)."""
    return t.is_cuda and dist.get_backend() == "gloo"


def _a2a(out, inp, out_splits, in_splits, group=None):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out.copy_(inp)
        return
    if _staged(inp):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), output_split_sizes=out_splits, input_split_sizes=in_splits,
                               group=group)
        out.copy_(o)
        return
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


def transpose_fwd(x, lay, group=None):
    """(|X_r|, n1, P) nodal slab -> (n0, |S_r|, P) spectral-layout slab."""
    n0, n1, _ = lay.dims
    m, _, P = x.shape
    send = torch.cat([x[:, s:e, :].reshape(-1) for (s, e) in lay.S]) if m else x.new_zeros(0)
    ls = lay.S[lay.rank][1] - lay.S[lay.rank][0]
    recv = x.new_empty(n0 * ls * P)
    _a2a(recv, send, [(e - s) * ls * P for (s, e) in lay.X], [m * (e - s) * P for (s, e) in lay.S], group)
    return recv.reshape(n0, ls, P)


def transpose_bwd(y, lay, group=None):
    """(n0, |S_r|, P) -> (|X_r|, n1, P)."""
    n0, n1, _ = lay.dims
    _, ls, P = y.shape
    # the nodal ranges X partition axis 0 in order: the send buffer is y itself
    send = y.contiguous().reshape(-1)
    m = lay.X[lay.rank][1] - lay.X[lay.rank][0]
    recv = y.new_empty(m * n1 * P)
    _a2a(recv, send, [m * (e - s) * P for (s, e) in lay.S], [(e - s) * ls * P for (s, e) in lay.X], group)
    parts = []
    off = 0
    for (s, e) in lay.S:
        cnt = m * (e - s) * P
        parts.append(recv[off:off + cnt].reshape(m, e - s, P))
        off += cnt
    return torch.cat(parts, dim=1).contiguous()


def transform_fwd(x, lay, ops, group=None):
    """Full orthonormal DST-I of a dense nodal slab -> spectral slab (n0,
    |S_r|, P), P = ops.pitch(lay) (padding zero)."""
    y = ops.dst_inner_fwd(x, ops.pitch(lay))  # new tensor, x untouched
    return ops.dst_mode0(transpose_fwd(y, lay, group))


def transform_bwd(y, lay, ops, scale=1.0, group=None):
    """Inverse of transform_fwd (DST-I is involutive): dense nodal slab."""
    y = ops.dst_mode0(y, scale)  # new tensor, y untouched
    return ops.dst_inner_bwd(transpose_bwd(y, lay, group), lay.dims[2])


def apply_slab(x, core_spec, lay, ops, alpha=1.0, group=None):
    """alpha F diag(core) F x for a slab-partitioned x; core_spec in the
    spectral layout (spectral_core(..., pitch=ops.pitch(lay)))."""
    y = transform_fwd(x, lay, ops, group)
    y.mul_(core_spec)
    return transform_bwd(y, lay, ops, alpha, group)


def _allreduce(t, group=None):
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if _staged(t):
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=group)
    return t


def pcg_slab(b, A_spec, P_spec, lay, ops, tol, k_max, group=None):
    """Slab-partitioned PCG (reference solver.py:116-180 in spectral space).

    One fused streaming pass per iteration (fl_pcg_phase 1, the pass of
    fl_pcg_spectral) and ONE all-reduce of its 4 partial sums, i.e. one host
    round trip per iteration (the convergence test).  Returns (x nodal slab,
    iterations, residual history, converged); the breakdown conditions
    raise PcgBreakdownError like the reference."""
    from .solver import PcgBreakdownError

    bh = transform_fwd(b, lay, ops, group)
    if bh.shape[-1] != lay.dims[2]:
        bh[..., lay.dims[2]:].zero_()  # mode 0 leaves rounding noise in the padding
    xh = torch.empty_like(bh)
    r = torch.empty_like(bh)
    p = torch.empty_like(bh)
    out = torch.zeros(4, dtype=torch.float64, device=bh.device)
    work = ops.new_work(bh)
    ops.pcg_phase(0, bh, xh, r, p, A_spec, P_spec, 0.0, 0.0, out, work)
    s = _allreduce(out.clone(), group).cpu().numpy()
    norm_b, rz, ps, beta = float(np.sqrt(s[0])), float(s[1]), float(s[2]), 0.0
    if norm_b == 0.0:
        return torch.zeros_like(b), 0, [0.0], True
    hist = [1.0]
    its, conv = 0, False
    for k in range(1, int(k_max) + 1):
        if rz <= 0.0:
            raise PcgBreakdownError(k, rz, what="<R, Z>")
        if ps <= 0.0:
            raise PcgBreakdownError(k, ps)
        ops.pcg_phase(1, bh, xh, r, p, A_spec, P_spec, rz / ps, beta, out, work)
        s = _allreduce(out.clone(), group).cpu().numpy()
        rel = float(np.sqrt(max(s[0], 0.0))) / norm_b
        hist.append(rel)
        its = k
        if rel <= tol:
            conv = True
            break
        bn = float(s[1]) / rz
        ps = float(s[2]) + 2.0 * bn * float(s[3]) + bn * bn * ps
        beta, rz = bn, float(s[1])
    x = transform_bwd(xh, lay, ops, 1.0, group)
    return x, its, hist, conv


def broadcast_cp(cp, src=0, group=None):
    """Broadcast a (small) canonical tensor from rank `src`: the Kronecker
    preconditioner core is built once instead of on every rank.  Other ranks
    pass cp=None and receive it."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return cp
    from .tensor import CpTensor
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    if dist.get_rank(group) == src:
        meta = torch.tensor([cp.rank, len(cp.factors)] + [f.shape[0] for f in cp.factors], dtype=torch.int64,
                            device=dev)
    else:
        meta = torch.zeros(5, dtype=torch.int64, device=dev)
    _bcast(meta, src, group)
    R, d = int(meta[0]), int(meta[1])
    dims = [int(v) for v in meta[2:2 + d]]
    if dist.get_rank(group) == src:
        w, fs = cp.weights.contiguous(), [f.contiguous() for f in cp.factors]
    else:
        w = torch.empty(R, dtype=torch.float64, device=dev)
        fs = [torch.empty((n, R), dtype=torch.float64, device=dev) for n in dims]
    for t in [w] + fs:
        _bcast(t, src, group)
    return CpTensor(w, fs)


def _bcast(t, src, group):
    if _staged(t):
        h = t.cpu()
        dist.broadcast(h, src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src, group=group)


def _pad_last(t, pitch):
    if pitch is None or pitch == t.shape[-1]:
        return t
    out = torch.zeros(t.shape[:-1] + (pitch,), dtype=t.dtype, device=t.device)
    out[..., :t.shape[-1]].copy_(t)
    return out


def spectral_core(kind, spectrum, lay, reciprocal=False, pitch=None):
    """Dense core of `kind` evaluated directly in the spectral slab layout
    (last mode padded to `pitch` with zeros when given)."""
    from .fracop import mode_values_device
    dev = torch.device("cuda", torch.cuda.current_device())
    mus, a = mode_values_device(kind, spectrum, dev)
    s, e = lay.S[lay.rank]
    mus = [mus[0], mus[1][s:e].contiguous(), mus[2]]
    shape = lay.spectral_shape
    out = torch.empty(shape, dtype=torch.float64, device=dev)
    if out.numel():
        _lib.call("fl_core_eval", _lib.ptr(out), 3, _lib.dims_arr(shape), _lib.ptr_arr(mus),
                  _lib.TAGS.index(kind.tag), float(a), float(kind.coeff_minus), float(kind.coeff_plus),
                  1 if reciprocal else 0, _lib.stream_ptr())
    return _pad_last(out, pitch)


def spectral_cp_core(cp, lay, pitch=None):
    """Dense expansion of a canonical core restricted to the spectral slab
    (last mode padded to `pitch` with zeros when given)."""
    s, e = lay.S[lay.rank]
    fs = [cp.factors[0], cp.factors[1][s:e].contiguous(), cp.factors[2]]
    shape = lay.spectral_shape
    out = torch.empty(shape, dtype=torch.float64, device=cp.weights.device)
    if out.numel():
        _lib.call("fl_cp_to_dense", _lib.ptr(out), 3, _lib.dims_arr(shape), cp.rank, _lib.ptr(cp.weights),
                  _lib.ptr_arr(fs), _lib.stream_ptr())
    return _pad_last(out, pitch)

"""Slab-partitioned 3D full-format operators and PCG across GPUs.

Layouts (n0 x n1 x n2 tensor, P ranks, one process per GPU):
  nodal    rank r holds planes i0 in X_r            -> (|X_r|, n1, n2)
  spectral rank r holds the transform for i1 in S_r -> (n0, |S_r|, n2)
Forward transform: DST-I along modes 2 and 1 inside the slab, an all-to-all
transpose (one torch.distributed.all_to_all_single over NCCL / NVLink), DST-I
along mode 0 on the transposed slab.  The inverse runs the same steps
backwards.  Cores (system operator, preconditioner) are evaluated directly in
the spectral layout, so the PCG iteration (three streaming phases per
iteration) needs only 3 scalar all-reduces per iteration; the two all-to-alls
happen once per solve (b -> b_hat, x_hat -> x).

The compute primitives come from a `LocalOps` object (each returns a new
tensor and leaves its input untouched); `CudaOps` binds them to
libfraclap_b200 (the product; the first DST pass of each primitive writes out
of place, so no defensive copies are made).  Tests substitute a host implementation to
exercise the decomposition, transposes and reduction logic with gloo on CPU.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["split", "SlabLayout", "CudaOps", "transform_fwd", "transform_bwd", "apply_slab", "pcg_slab"]


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
    """Local compute through libfraclap_b200 (device tensors)."""

    def dst_inner_modes(self, x, n1, n2):
        """DST-I along modes 2 and 1 of a (m, n1, n2) slab into a new tensor
        (x is not modified; the first pass writes out of place, so no copy)."""
        m = x.shape[0]
        st = _lib.stream_ptr()
        if m == 0:
            return x.clone()
        x = x.contiguous()
        y = torch.empty_like(x)
        _lib.call("fl_dst1", _lib.ptr(x), _lib.ptr(y), m * n1, n2, 1, 1.0, st)
        _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(y), m, n1, n2, 1.0, st)
        return y

    def dst_mode0(self, y, scale=1.0):
        """DST-I along mode 0 of a (n0, m, n2) slab into a new tensor."""
        n0, m, n2 = y.shape
        if m * n2 == 0:
            return y.clone()
        y = y.contiguous()
        out = torch.empty_like(y)
        _lib.call("fl_dst1", _lib.ptr(y), _lib.ptr(out), 1, n0, m * n2, float(scale), _lib.stream_ptr())
        return out

    def pcg_phase(self, phase, b, x, r, p, A, P, s, out, work):
        _lib.call("fl_pcg_phase", phase, _lib.ptr(b), _lib.ptr(x), _lib.ptr(r), _lib.ptr(p), _lib.ptr(A),
                  _lib.ptr(P), b.numel(), float(s), _lib.ptr(out), _lib.ptr(work), _lib.stream_ptr())

    def new_work(self, like):
        return torch.zeros(_lib.FL_PCG_WORK, dtype=torch.float64, device=like.device)


def _a2a(out, inp, out_splits, in_splits, group=None):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out.copy_(inp)
        return
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


def transpose_fwd(x, lay, group=None):
    """(|X_r|, n1, n2) nodal slab -> (n0, |S_r|, n2) spectral-layout slab."""
    n0, n1, n2 = lay.dims
    m = x.shape[0]
    send = torch.cat([x[:, s:e, :].reshape(-1) for (s, e) in lay.S]) if m else x.new_zeros(0)
    ls = lay.S[lay.rank][1] - lay.S[lay.rank][0]
    recv = x.new_empty(n0 * ls * n2)
    _a2a(recv, send, [(e - s) * ls * n2 for (s, e) in lay.X], [m * (e - s) * n2 for (s, e) in lay.S], group)
    return recv.reshape(n0, ls, n2)


def transpose_bwd(y, lay, group=None):
    """(n0, |S_r|, n2) -> (|X_r|, n1, n2)."""
    n0, n1, n2 = lay.dims
    ls = y.shape[1]
    # the nodal ranges X partition axis 0 in order: the send buffer is y itself
    send = y.contiguous().reshape(-1)
    m = lay.X[lay.rank][1] - lay.X[lay.rank][0]
    recv = y.new_empty(m * n1 * n2)
    _a2a(recv, send, [m * (e - s) * n2 for (s, e) in lay.S], [(e - s) * ls * n2 for (s, e) in lay.X], group)
    parts = []
    off = 0
    for (s, e) in lay.S:
        cnt = m * (e - s) * n2
        parts.append(recv[off:off + cnt].reshape(m, e - s, n2))
        off += cnt
    return torch.cat(parts, dim=1).contiguous()


def transform_fwd(x, lay, ops, group=None):
    """Full orthonormal DST-I of a nodal slab -> spectral slab."""
    x = ops.dst_inner_modes(x, lay.dims[1], lay.dims[2])  # new tensor, x untouched
    return ops.dst_mode0(transpose_fwd(x, lay, group).contiguous())


def transform_bwd(y, lay, ops, scale=1.0, group=None):
    """Inverse of transform_fwd (DST-I is involutive)."""
    y = ops.dst_mode0(y, scale)  # new tensor, y untouched
    return ops.dst_inner_modes(transpose_bwd(y, lay, group), lay.dims[1], lay.dims[2])


def apply_slab(x, core_spec, lay, ops, alpha=1.0, group=None):
    """alpha F diag(core) F x for a slab-partitioned x; core_spec in the spectral layout."""
    y = transform_fwd(x, lay, ops, group)
    y.mul_(core_spec)
    return transform_bwd(y, lay, ops, alpha, group)


def _allreduce(t, group=None):
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, group=group)
    return t


def pcg_slab(b, A_spec, P_spec, lay, ops, tol, k_max, group=None):
    """Slab-partitioned PCG (reference solver.py:116-180 in spectral space).

    Returns (x nodal slab, iterations, residual history, converged).  The
    breakdown conditions raise PcgBreakdownError like the reference."""
    from .solver import PcgBreakdownError

    bh = transform_fwd(b, lay, ops, group)
    xh = torch.empty_like(bh)
    r = torch.empty_like(bh)
    p = torch.empty_like(bh)
    out = torch.zeros(3, dtype=torch.float64, device=bh.device)
    work = ops.new_work(bh)
    ops.pcg_phase(0, bh, xh, r, p, A_spec, P_spec, 0.0, out, work)
    s = _allreduce(out.clone(), group).cpu().numpy()
    norm_b, rz, ps = float(np.sqrt(s[0])), float(s[1]), float(s[2])
    if norm_b == 0.0:
        return torch.zeros_like(b), 0, [0.0], True
    hist = [1.0]
    its, conv = 0, False
    for k in range(1, int(k_max) + 1):
        if rz <= 0.0:
            raise PcgBreakdownError(k, rz, what="<R, Z>")
        if ps <= 0.0:
            raise PcgBreakdownError(k, ps)
        ops.pcg_phase(1, bh, xh, r, p, A_spec, P_spec, rz / ps, out, work)
        s = _allreduce(out[:2].clone(), group).cpu().numpy()
        rel = float(np.sqrt(max(s[0], 0.0))) / norm_b
        hist.append(rel)
        its = k
        if rel <= tol:
            conv = True
            break
        rzn = float(s[1])
        ops.pcg_phase(2, bh, xh, r, p, A_spec, P_spec, rzn / rz, out, work)
        ps = float(_allreduce(out[:1].clone(), group).cpu().numpy()[0])
        rz = rzn
    x = transform_bwd(xh, lay, ops, 1.0, group)
    return x, its, hist, conv


def spectral_core(kind, spectrum, lay, reciprocal=False):
    """Dense core of `kind` evaluated directly in the spectral slab layout."""
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
    return out


def spectral_cp_core(cp, lay):
    """Dense expansion of a canonical core restricted to the spectral slab."""
    s, e = lay.S[lay.rank]
    fs = [cp.factors[0], cp.factors[1][s:e].contiguous(), cp.factors[2]]
    shape = lay.spectral_shape
    out = torch.empty(shape, dtype=torch.float64, device=cp.weights.device)
    if out.numel():
        _lib.call("fl_cp_to_dense", _lib.ptr(out), 3, _lib.dims_arr(shape), cp.rank, _lib.ptr(cp.weights),
                  _lib.ptr_arr(fs), _lib.stream_ptr())
    return out

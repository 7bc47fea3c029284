"""Multi-process (gloo, CPU) test of the slab-partitioned host logic:
decomposition, all-to-all transposes, spectral-layout cores and the PCG
reduction protocol.  Local compute is a host stand-in built on the oracle
(the product binds the same interface to libfraclap_b200)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1809_01971_b200 import distributed as D


class HostOps:
    """Host stand-in for CudaOps (oracle DSTs, numpy phases); pad > 0 adds
    that many zero padding columns to the spectral layout, like CudaOps on
    FFT lengths."""

    def __init__(self, pad=0):
        self.pad = pad

    def pitch(self, lay):
        return lay.dims[2] + self.pad

    def dst_inner_fwd(self, x, P):
        m, n1, n2 = x.shape
        out = torch.zeros((m, n1, P), dtype=torch.float64)
        if m:
            out[..., :n2] = torch.from_numpy(oracle.dst(oracle.dst(x.numpy(), axis=2), axis=1))
        return out

    def dst_inner_bwd(self, y, n2, scale=1.0):
        if y.shape[0] == 0:
            return torch.zeros(y.shape[:2] + (n2,), dtype=torch.float64)
        z = oracle.dst(oracle.dst(y.numpy()[..., :n2], axis=1), axis=2)
        return torch.from_numpy(np.ascontiguousarray(scale * z))

    def dst_mode0(self, y, scale=1.0):
        if y.numel() == 0:
            return y.clone()
        return torch.from_numpy(np.ascontiguousarray(scale * oracle.dst(y.numpy(), axis=0)))

    def pcg_phase(self, phase, b, x, r, p, A, P, alpha, beta, out, work):
        if phase == 0:
            x.zero_(); r.copy_(b); p.zero_()
            z = P * b
            out[0], out[1], out[2], out[3] = (b * b).sum(), (b * z).sum(), (z * A * z).sum(), 0.0
        else:
            p.mul_(beta).add_(P * r)
            x.add_(alpha * p); r.sub_(alpha * A * p)
            z = P * r
            out[0], out[1], out[2], out[3] = (r * r).sum(), (r * z).sum(), (z * A * z).sum(), (z * A * p).sum()

    def new_work(self, like):
        return torch.zeros(8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, q, pad=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = D.SlabLayout(dims, world, rank)
        ops = HostOps(pad)
        rng = np.random.default_rng(5)
        x_full = rng.standard_normal(dims)
        lam = [oracle.laplacian_eigenvalues(n) for n in dims]
        A_full = oracle.dense_core("g2", lam, 0.5, 1e-2, 1.0 / 1e-2)
        P_full = 1.0 / A_full * (1.0 + 0.05 * np.cos(np.arange(A_full.size)).reshape(A_full.shape))
        xs, xe = lay.X[rank]
        ss, se = lay.S[rank]
        x = torch.from_numpy(x_full[xs:xe].copy())
        # forward transform lands in the spectral layout
        yh = D.transform_fwd(x, lay, ops)
        full_hat = oracle.transform_full(x_full)
        n2 = dims[2]
        err_fwd = float(np.abs(yh.numpy()[..., :n2] - full_hat[:, ss:se, :]).max())
        back = D.transform_bwd(yh, lay, ops)
        err_rt = float(np.abs(back.numpy() - x_full[xs:xe]).max())
        # operator application (cores padded with zeros like the spectral layout)
        A = D._pad_last(torch.from_numpy(np.ascontiguousarray(A_full[:, ss:se, :])), ops.pitch(lay))
        P = D._pad_last(torch.from_numpy(np.ascontiguousarray(P_full[:, ss:se, :])), ops.pitch(lay))
        y = D.apply_slab(x, A, lay, ops, alpha=0.5)
        ya = 0.5 * oracle.apply_full(A_full, x_full)
        err_apply = float(np.abs(y.numpy() - ya[xs:xe]).max() / np.abs(ya).max())
        # PCG
        sol, its, hist, conv = D.pcg_slab(x, A, P, lay, ops, 1e-10, 50)
        xo, histo, ito, convo = oracle.pcg_dense(lambda v: oracle.apply_full(A_full, v),
                                                 lambda v: oracle.apply_full(P_full, v), x_full, 1e-10, 50)
        err_pcg = float(np.abs(sol.numpy() - xo[xs:xe]).max() / np.abs(xo).max())
        q.put((rank, err_fwd, err_rt, err_apply, err_pcg, its, ito, conv, convo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,pad", [(2, (7, 6, 5), 0), (2, (8, 9, 7), 0), (3, (7, 5, 4), 0),
                                            (2, (7, 6, 7), 1), (3, (7, 5, 4), 4)])
def test_slab_partitioned_matches_oracle(world, dims, pad):
    """Decomposition, transposes (dense and padded spectral layouts), fused
    PCG pass protocol (one all-reduce of 4 sums per iteration) vs the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q, pad)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e_fwd, e_rt, e_ap, e_pcg, its, ito, conv, convo in res:
        assert e_fwd <= 1e-12 and e_rt <= 1e-12 and e_ap <= 1e-12
        assert conv and convo and its == ito
        assert e_pcg <= 1e-10


def test_split_is_balanced_and_covering():
    for n in (1, 5, 7, 1023):
        for p in (1, 2, 3, 8):
            b = D.split(n, p)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(p - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1


def _batch_worker(rank, world, port, count, q):
    from paper_1809_01971_b200 import batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = [(i,) + batch.problem_params(i) for i in batch.problem_indices(count, rank, world)]
        got = [None] * world
        dist.all_gather_object(got, mine)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 64), (3, 7)])
def test_batch_problems_spread_over_ranks(world, count):
    """configs[4]: independent problems spread over ranks (batch.solve_batch)
    with no data-path collective; the gathered assignment is a disjoint cover
    of the batch and each problem's parameters do not depend on the rank count."""
    from paper_1809_01971_b200 import batch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = {i: batch.problem_params(i) for i in range(count)}
    for _, got in res:
        flat = [rec for part in got for rec in part]
        assert sorted(r[0] for r in flat) == list(range(count))
        for i, alpha, beta, tseed in flat:
            assert (alpha, beta, tseed) == want[i]
            assert 0.1 <= alpha <= 0.9 and 1e-5 <= beta <= 1e-1
    with pytest.raises(ValueError):
        batch.problem_indices(4, 2, 2)

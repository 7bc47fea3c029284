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
    def dst_inner_modes(self, x, n1, n2):
        if x.shape[0] == 0:
            return x
        z = oracle.dst(oracle.dst(x.numpy(), axis=2), axis=1)
        return torch.from_numpy(np.ascontiguousarray(z))

    def dst_mode0(self, y, scale=1.0):
        if y.numel() == 0:
            return y
        return torch.from_numpy(np.ascontiguousarray(scale * oracle.dst(y.numpy(), axis=0)))

    def pcg_phase(self, phase, b, x, r, p, A, P, s, out, work):
        if phase == 0:
            x.zero_(); r.copy_(b); p.copy_(P * b)
            out[0], out[1], out[2] = (b * b).sum(), (b * P * b).sum(), (p * A * p).sum()
        elif phase == 1:
            x.add_(s * p); r.sub_(s * A * p)
            out[0], out[1] = (r * r).sum(), (r * P * r).sum()
        else:
            p.mul_(s).add_(P * r)
            out[0] = (p * A * p).sum()

    def new_work(self, like):
        return torch.zeros(8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = D.SlabLayout(dims, world, rank)
        ops = HostOps()
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
        err_fwd = float(np.abs(yh.numpy() - full_hat[:, ss:se, :]).max())
        back = D.transform_bwd(yh, lay, ops)
        err_rt = float(np.abs(back.numpy() - x_full[xs:xe]).max())
        # operator application
        A = torch.from_numpy(np.ascontiguousarray(A_full[:, ss:se, :]))
        P = torch.from_numpy(np.ascontiguousarray(P_full[:, ss:se, :]))
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


@pytest.mark.parametrize("world,dims", [(2, (7, 6, 5)), (2, (8, 9, 7)), (3, (7, 5, 4))])
def test_slab_partitioned_matches_oracle(world, dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
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

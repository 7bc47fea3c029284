"""Slab path with the CUDA bindings on one rank (world 1) vs the single-GPU path."""

import numpy as np
import pytest
import torch

import oracle
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import distributed as D, fullsolve
from paper_1809_01971_b200.fracop import CoreFunctionKind

pytestmark = pytest.mark.gpu


def test_slab_single_rank_matches_fused_path():
    n = 31
    spec = fl.laplacian_spectrum(n, 3)
    lay = D.SlabLayout((n, n, n), 1, 0)
    ops = D.CudaOps()
    x = torch.randn((n, n, n), dtype=torch.float64, device="cuda")
    kind = CoreFunctionKind("g1", 0.5)
    A = D.spectral_core(kind, spec, lay, pitch=ops.pitch(lay))
    assert A.shape[-1] == 32  # padded spectral layout on FFT lengths
    y = D.apply_slab(x, A, lay, ops)
    want = oracle.apply_full(oracle.dense_core("g1", [oracle.laplacian_eigenvalues(n)] * 3, 0.5), x.cpu().numpy())
    assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)
    cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, precond_rank=5, residual_tol=1e-9, k_max=80)
    Af, Pf = fullsolve.control_cores(cfg, spec)
    u1, rep = fullsolve.solve_control_full(x, cfg, spec, cores=(Af, Pf))
    P32 = ops.pitch(lay)
    u2, its, hist, conv = D.pcg_slab(x, D._pad_last(Af, P32), D._pad_last(Pf, P32), lay, ops, 1e-9, 80)
    assert conv and its == rep.iterations
    assert float(torch.linalg.vector_norm(u1 - u2) / torch.linalg.vector_norm(u1)) <= 1e-10


def _two_rank_worker(rank, world, port, n, q):
    """One rank of the slab path on the SHARED GPU 0: CudaOps (the product
    kernels, fl_pcg_phase) with gloo collectives staged through the host."""
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = fl.laplacian_spectrum(n, 3)
        lay = D.SlabLayout((n, n, n), world, rank)
        ops = D.CudaOps()
        Pp = ops.pitch(lay)
        rng = np.random.default_rng(3)
        y_full = rng.standard_normal((n, n, n))
        xs, xe = lay.X[rank]
        y = torch.tensor(y_full[xs:xe], device="cuda")
        cfg = fl.SolverConfig(alpha=0.75, beta=1e-4, precond_rank=6, residual_tol=1e-8, k_max=100)
        kind = fullsolve._control_kind(cfg)
        pre = fullsolve.kronecker_preconditioner(cfg, spec) if rank == 0 else None
        pre_cp = D.broadcast_cp(pre.diag.core if pre is not None else None)
        A = D.spectral_core(kind, spec, lay, pitch=Pp)
        P = D.spectral_cp_core(pre_cp, lay, pitch=Pp)
        yh = D.transform_fwd(y, lay, ops)
        back = D.transform_bwd(yh.clone(), lay, ops)
        rt = float((back - y).abs().max())
        u, its, hist, conv = D.pcg_slab(y, A, P, lay, ops, cfg.residual_tol, cfg.k_max)
        P_dense = None
        if rank == 0:
            P_dense = fl.cp_to_dense(pre_cp)
            P_dense = P_dense.cpu().numpy() if isinstance(P_dense, torch.Tensor) else np.asarray(P_dense)
        q.put((rank, rt, Pp, u.cpu().numpy(), its, conv, hist, P_dense))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_oracle():
    """the multi-rank slab path with the CUDA bindings (two
    processes sharing GPU 0, gloo host-staged all-to-all and all-reduce),
    configs[3]'s parameters at n = 63, against the oracle's dense PCG with the
    same (broadcast) preconditioner core: iterations +-1, solution 1e-8."""
    import socket
    import torch.multiprocessing as mp
    n, world = 63, 2
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(r[2] == 64 for r in res)  # padded spectral layout
    assert all(r[1] <= 1e-12 for r in res)
    u = np.concatenate([r[3] for r in res], axis=0)
    its = res[0][4]
    assert all(r[5] for r in res) and all(r[4] == its for r in res)
    lam = oracle.laplacian_eigenvalues(n)
    A_full = oracle.dense_core("g2", [lam] * 3, 0.75, 1e-4, 1e4)
    P_full = res[0][7]
    y_full = np.random.default_rng(3).standard_normal((n, n, n))
    x, hist, ito, ok = oracle.pcg_dense(lambda v: oracle.apply_full(A_full, v), lambda v: oracle.apply_full(P_full, v),
                                        y_full, 1e-8, 100)
    assert ok and abs(ito - its) <= 1
    assert np.linalg.norm(u - x) <= 1e-8 * np.linalg.norm(x)

"""GPU tests of the row-partitioned CG on the single available B200.

* loopback transport: P partitions of one system on this GPU, halos as device copies,
  dot partials summed in partition order -- exercises the whole decomposition
  (renumbering, halo pattern, interior/boundary SpMV views, fused dots);
* NCCL transport at world size 1 (torch.distributed + libsparseb200's own NCCL
  communicator): exercises the NCCL allreduce path end to end.
Iteration counts must match the single-GPU solver within +-2% and the reference golden
where one exists; the solution must match the single-GPU solve."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import fixtures
from paper_2510_08230_b200 import dist as D
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tests.gpu_util import host

pytestmark = pytest.mark.gpu


def _vecs(dev, parts, b_global):
    bs, xs = [], []
    for part in parts:
        lo, hi = part.pat.lo, part.pat.hi
        bs.append(sp.dense_from_array(dev, torch.tensor(b_global[lo:hi])))
        xs.append(sp.dense_create(dev, hi - lo, 1, sp.Precision.double, 0.0))
    return bs, xs


def _single(dev, a, b, rf=1e-8):
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log = sp.Cg(a, criteria=[sp.Iteration(5000), sp.ResidualNorm(rf)],
                preconditioner=sp.jacobi_create(a)).solve(sp.dense_from_array(dev, b.copy()), x)
    return log, host(x)


@pytest.mark.parametrize("p,world", [(16, 1), (16, 2), (24, 3), (32, 4)])
def test_loopback_stencil_cg(dev, p, world):
    parts = [D.stencil_partition(dev, p, r, world) for r in range(world)]
    if world > 1:
        assert all(len(part.views) >= 2 for part in parts)  # interior/boundary overlap views
    b = np.ones(p ** 3)
    bs, xs = _vecs(dev, parts, b)
    log = D.DistCg(parts, [sp.Iteration(5000), sp.ResidualNorm(1e-8)]).solve(bs, xs)
    ref_log, ref_x = _single(dev, gen.poisson3d(dev, p), b)
    golden = {16: 39, 32: 79}.get(p, ref_log.iterations)
    assert log.converged
    assert abs(log.iterations - ref_log.iterations) <= max(1, int(np.ceil(0.02 * ref_log.iterations)))
    assert abs(log.iterations - golden) <= max(1, int(np.ceil(0.02 * golden)))
    x = np.concatenate([host(v) for v in xs])
    assert np.abs(x - ref_x).max() <= 1e-7 * np.abs(ref_x).max()


def test_loopback_general_matrix(dev):
    """Random SPD-ish matrix: non-contiguous send lists (pack kernel), no overlap views."""
    rng = np.random.default_rng(8)
    n = 600
    r, c, v = fixtures.random_sparse_triplets(rng, n, n, 0.01)
    rows = np.concatenate([r, c, np.arange(n)])  # symmetrise + strong diagonal
    cols = np.concatenate([c, r, np.arange(n)])
    vals = np.concatenate([v, v, np.full(n, 20.0)])
    rp, ci, vv = fixtures.canonical_csr(n, rows, cols, vals)
    world = 3
    ghosts = {}
    for k in range(world):
        lo, hi = D.partition(n, world)[k]
        _, pat = D.localize(torch.as_tensor(rp[lo:hi + 1] - rp[lo]), torch.as_tensor(ci[rp[lo]:rp[hi]]),
                            lo, hi, D.partition(n, world), k)
        ghosts[k] = pat.ghosts
    parts = [D.csr_partition(dev, rp, ci, vv, k, world, all_patterns=ghosts) for k in range(world)]
    assert any(part._host["send_lo"][j] < 0 for part in parts for j in range(len(part.nbr)))
    b = np.random.default_rng(1).standard_normal(n)
    bs, xs = _vecs(dev, parts, b)
    log = D.DistCg(parts, [sp.Iteration(1000), sp.ResidualNorm(1e-10)]).solve(bs, xs)
    a = sp.CsrMatrix(dev, n, n, rp, ci, vv)
    ref_log, ref_x = _single(dev, a, b, rf=1e-10)
    assert log.converged and abs(log.iterations - ref_log.iterations) <= 1
    x = np.concatenate([host(v) for v in xs])
    assert np.abs(x - ref_x).max() <= 1e-8 * np.abs(ref_x).max()


def test_nccl_world1(dev):
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = D.NcclComm(0, 1)
        part = D.stencil_partition(dev, 16, 0, 1)
        bs, xs = _vecs(dev, [part], np.ones(16 ** 3))
        log = D.DistCg(part, [sp.Iteration(1000), sp.ResidualNorm(1e-8)], comm=comm).solve(bs[0], xs[0])
        assert log.converged and abs(log.iterations - 39) <= 1
        # the same communicator drives the partitioned BiCGSTAB and GMRES(30)
        cd = D.stencil_partition(dev, 16, 0, 1, c=0.5)
        bs, xs = _vecs(dev, [cd], np.ones(16 ** 3))
        lg = D.DistGmres(cd, [sp.Iteration(5000), sp.ResidualNorm(1e-8)], comm=comm, krylov_dim=30).solve(bs, xs)
        assert lg.converged and abs(lg.iterations - 81) <= 2  # reference golden 16^3
        bs, xs = _vecs(dev, [cd], np.ones(16 ** 3))
        lb = D.DistBicgstab(cd, [sp.Iteration(5000), sp.ResidualNorm(1e-8)], comm=comm).solve(bs, xs)
        ref, _ = _single_kind(dev, "bicgstab", gen.stencil_csr(dev, 16, dim=3, c=0.5), np.ones(16 ** 3))
        assert lb.converged and abs(lb.iterations - ref.iterations) <= max(1, int(np.ceil(0.02 * ref.iterations)))
        comm.close()
    finally:
        dist.destroy_process_group()


def _single_kind(dev, kind, a, b, rf=1e-8, **kw):
    cls = {"cg": sp.Cg, "bicgstab": sp.Bicgstab, "gmres": sp.Gmres}[kind]
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log = cls(a, criteria=[sp.Iteration(5000), sp.ResidualNorm(rf)], preconditioner=sp.jacobi_create(a),
              **kw).solve(sp.dense_from_array(dev, b.copy()), x)
    return log, host(x)


@pytest.mark.parametrize("p,world", [(16, 1), (16, 2), (20, 3), (24, 4)])
def test_loopback_gmres_convdiff(dev, p, world):
    """Partitioned GMRES(30)+Jacobi on the nonsymmetric conv-diff operator (config #4's
    family): same inner-iteration count as the single-GPU solver (+-2%), the reference's
    81 at 16^3, same solution."""
    parts = [D.stencil_partition(dev, p, r, world, c=0.5) for r in range(world)]
    b = np.ones(p ** 3)
    bs, xs = _vecs(dev, parts, b)
    log = D.DistGmres(parts, [sp.Iteration(5000), sp.ResidualNorm(1e-8)], krylov_dim=30).solve(bs, xs)
    ref_log, ref_x = _single_kind(dev, "gmres", gen.stencil_csr(dev, p, dim=3, c=0.5), b, krylov_dim=30)
    assert log.converged and log.stop_reason == "residual"
    assert abs(log.iterations - ref_log.iterations) <= max(1, int(np.ceil(0.02 * ref_log.iterations)))
    if p == 16:
        assert abs(log.iterations - 81) <= 2
    x = np.concatenate([host(v) for v in xs])
    assert np.abs(x - ref_x).max() <= 1e-6 * np.abs(ref_x).max()
    if world == 1:  # one partition: the identical kernels and summation order
        assert log.iterations == ref_log.iterations
        np.testing.assert_allclose(log.residual_history, ref_log.residual_history, rtol=1e-12)


@pytest.mark.parametrize("p,world", [(16, 1), (16, 2), (20, 3), (24, 4)])
def test_loopback_bicgstab(dev, p, world):
    """Partitioned BiCGSTAB+Jacobi on the conv-diff operator: iteration count within the
    single-GPU solver's +-2% band (the recurrence is rounding-sensitive)."""
    parts = [D.stencil_partition(dev, p, r, world, c=0.5) for r in range(world)]
    b = np.ones(p ** 3)
    bs, xs = _vecs(dev, parts, b)
    log = D.DistBicgstab(parts, [sp.Iteration(5000), sp.ResidualNorm(1e-8)]).solve(bs, xs)
    ref_log, ref_x = _single_kind(dev, "bicgstab", gen.stencil_csr(dev, p, dim=3, c=0.5), b)
    assert log.converged
    assert abs(log.iterations - ref_log.iterations) <= max(2, int(np.ceil(0.02 * ref_log.iterations)))
    x = np.concatenate([host(v) for v in xs])
    assert np.abs(x - ref_x).max() <= 1e-5 * np.abs(ref_x).max()
    if world == 1:
        assert log.iterations == ref_log.iterations


def test_loopback_solvers_unpreconditioned_general(dev):
    """A general (non-banded) nonsymmetric matrix, no preconditioner, 3 partitions with
    packed (non-contiguous) halos: GMRES(10) and BiCGSTAB match the single-GPU solvers."""
    rng = np.random.default_rng(9)
    n = 500
    r, c, v = fixtures.random_sparse_triplets(rng, n, n, 0.01)
    rows = np.concatenate([r, np.arange(n)])
    cols = np.concatenate([c, np.arange(n)])
    vals = np.concatenate([v, np.full(n, 8.0)])
    rp, ci, vv = fixtures.canonical_csr(n, rows, cols, vals)
    world = 3
    bounds = D.partition(n, world)
    ghosts = {}
    for k in range(world):
        lo, hi = bounds[k]
        _, pat = D.localize(torch.as_tensor(rp[lo:hi + 1] - rp[lo]), torch.as_tensor(ci[rp[lo]:rp[hi]]),
                            lo, hi, bounds, k)
        ghosts[k] = pat.ghosts
    parts = [D.csr_partition(dev, rp, ci, vv, k, world, all_patterns=ghosts) for k in range(world)]
    a = sp.CsrMatrix(dev, n, n, rp, ci, vv)
    b = np.random.default_rng(2).standard_normal(n)
    crit = [sp.Iteration(2000), sp.ResidualNorm(1e-10)]
    for name, cls, kw in (("gmres", D.DistGmres, {"krylov_dim": 10}), ("bicgstab", D.DistBicgstab, {})):
        bs, xs = _vecs(dev, parts, b)
        log = cls(parts, crit, jacobi=False, **kw).solve(bs, xs)
        single = {"gmres": sp.Gmres, "bicgstab": sp.Bicgstab}[name]
        x1 = sp.dense_create(dev, n, 1, sp.Precision.double, 0.0)
        ref = single(a, criteria=crit, **kw).solve(sp.dense_from_array(dev, b.copy()), x1)
        assert log.converged and ref.converged, name
        assert abs(log.iterations - ref.iterations) <= max(2, int(np.ceil(0.02 * ref.iterations))), name
        x = np.concatenate([host(t) for t in xs])
        xr = host(x1)
        assert np.abs(x - xr).max() <= 1e-7 * np.abs(xr).max(), name

"""Multi-process (gloo, world size 2, CPU) test of the row-partition host logic.

Each rank localises its rows of a global CSR, exchanges ghost lists over gloo, then
runs a distributed SpMV in NumPy: halo values travel with dist.send / dist.recv along
the computed pattern, and the local SpMV uses the renumbered columns.  The result must
equal the oracle's global SpMV BIT FOR BIT (the renumbering keeps each row's stored
order, so the fp64 sum order is the reference's)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fixtures, sbref


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrices():
    rng = np.random.default_rng(21)
    out = [fixtures.stencil_csr(9, dim=3), fixtures.stencil_csr(14, dim=2),
           fixtures.stencil_csr(7, dim=3, c=0.5)]
    out.append(fixtures.canonical_csr(300, *fixtures.random_sparse_triplets(rng, 300, 300, 0.02)))
    return out


def _worker(rank, world, port, results):
    from paper_2510_08230_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for mi, (rp, ci, v) in enumerate(_matrices()):
            n = rp.size - 1
            bounds = D.partition(n, world)
            lo, hi = bounds[rank]
            lrp = torch.as_tensor(rp[lo:hi + 1] - rp[lo])
            lci = torch.as_tensor(ci[rp[lo]:rp[hi]])
            local, pat = D.localize(lrp, lci, lo, hi, bounds, rank)
            D.exchange_send_lists(pat)
            b = np.random.default_rng(mi).standard_normal(n)
            # halo: send my rows that others need, receive my ghosts
            reqs = []
            for s, rows in pat.send.items():
                reqs.append(dist.isend(torch.as_tensor(b[lo:hi][rows.numpy()]), s))
            ghost_vals = np.zeros(pat.n_ghost)
            for s, (off, cnt) in pat.recv.items():
                buf = torch.zeros(cnt, dtype=torch.float64)
                dist.recv(buf, s)
                ghost_vals[off:off + cnt] = buf.numpy()
            for r in reqs:
                r.wait()
            # received ghosts are exactly the global entries they stand for
            np.testing.assert_array_equal(ghost_vals, b[pat.ghosts.numpy()])
            xe = np.concatenate([b[lo:hi], ghost_vals])
            y = sbref.csr_spmv(lrp.numpy().astype(np.int64), local.numpy().astype(np.int64),
                               v[rp[lo]:rp[hi]], xe)
            ref = sbref.csr_spmv(rp, ci, v, b)[lo:hi]
            np.testing.assert_array_equal(y, ref)
            split = pat.interior()
            if mi < 3:  # stencil slabs: boundary rows are a prefix + suffix
                assert split is not None
            results[(rank, mi)] = (pat.n_ghost, sorted(pat.send), sorted(pat.recv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_spmv_gloo(world):
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    assert len(results) == world * len(_matrices())
    # the pattern is symmetric: r sends to s  <=>  s receives from r
    for mi in range(len(_matrices())):
        for r in range(world):
            _, send_to, recv_from = results[(r, mi)]
            for s in send_to:
                assert r in results[(s, mi)][2]


# ------------------------------------------------------------------ partitioned Krylov (gloo)
class _Rank:
    """One rank's share for the partitioned-solver restatement: local rows, renumbered
    columns, halo over dist.send / dist.recv, global dots by dist.all_reduce -- the sync
    structure of csrc/dist_krylov.cu (one allreduce per reduction, halo before each SpMV)."""

    def __init__(self, rp, ci, v, rank, world):
        from paper_2510_08230_b200 import dist as D

        n = rp.size - 1
        bounds = D.partition(n, world)
        self.lo, self.hi = bounds[rank]
        lo, hi = self.lo, self.hi
        self.lrp = (rp[lo:hi + 1] - rp[lo]).astype(np.int64)
        lci = torch.as_tensor(ci[rp[lo]:rp[hi]])
        local, self.pat = D.localize(torch.as_tensor(self.lrp), lci, lo, hi, bounds, rank)
        D.exchange_send_lists(self.pat)
        self.lci = local.numpy().astype(np.int64)
        self.v = v[rp[lo]:rp[hi]]
        diag = np.zeros(hi - lo)
        for i in range(hi - lo):
            s = slice(self.lrp[i], self.lrp[i + 1])
            hit = self.lci[s] == i
            diag[i] = self.v[s][hit][0] if hit.any() else 0.0
        self.inv = 1.0 / diag

    def halo(self, own):
        reqs = [dist.isend(torch.as_tensor(own[rows.numpy()].copy()), s) for s, rows in self.pat.send.items()]
        ghosts = np.zeros(self.pat.n_ghost)
        for s, (off, cnt) in self.pat.recv.items():
            buf = torch.zeros(cnt, dtype=torch.float64)
            dist.recv(buf, s)
            ghosts[off:off + cnt] = buf.numpy()
        for r in reqs:
            r.wait()
        return np.concatenate([own, ghosts])

    def spmv(self, own):
        return sbref.csr_spmv(self.lrp, self.lci, self.v, self.halo(own))

    def dot(self, x, y):
        t = torch.tensor([sbref.dot(x, y)], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t[0])


def _bicgstab(R, b, rf, max_iters):
    """oracle/sbref.cpp bicgstab on the partition: 4 global reductions per iteration."""
    x = np.zeros_like(b)
    bnorm = np.sqrt(R.dot(b, b))
    r = b - R.spmv(x)
    rh = r.copy()
    rnorm = np.sqrt(R.dot(r, r))
    rho_prev = alpha = omega = 1.0
    p = v = None
    for it in range(1, max_iters + 1):
        rho = R.dot(rh, r)
        if it == 1:
            p = r.copy()
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = sbref.axpy(1.0, r, sbref.scal(beta, sbref.axpy(-omega, v, p)))
        ph = p * R.inv
        v = R.spmv(ph)
        alpha = rho / R.dot(rh, v)
        s = sbref.axpy(-alpha, v, r)
        snorm = np.sqrt(R.dot(s, s))
        if snorm <= rf * bnorm:
            return it
        sh = s * R.inv
        t = R.spmv(sh)
        tt, ts = R.dot(t, t), R.dot(t, s)
        omega = ts / tt
        x = sbref.axpy(omega, sh, sbref.axpy(alpha, ph, x))
        r = sbref.axpy(-omega, t, s)
        rnorm = np.sqrt(R.dot(r, r))
        if rnorm <= rf * bnorm:
            return it
        rho_prev = rho
    return max_iters


def _gmres(R, b, rf, max_iters, m):
    """solvers.py:322-399 on the partition: single-pass MGS, one allreduce per step."""
    x = np.zeros_like(b)
    bnorm = np.sqrt(R.dot(b, b))
    total = 0
    while True:
        r = b - R.spmv(x)
        beta = np.sqrt(R.dot(r, r))
        basis = [sbref.scal(1.0 / beta, r)]
        rm, g, cs, sn = np.zeros((m, m)), np.zeros(m + 1), np.zeros(m), np.zeros(m)
        g[0] = beta
        for j in range(m):
            w = R.spmv(basis[j] * R.inv)
            h = np.zeros(j + 2)
            for i in range(j + 1):
                h[i] = R.dot(basis[i], w)
                w = sbref.axpy(-h[i], basis[i], w)
            hn = np.sqrt(R.dot(w, w))
            h[j + 1] = hn
            for i in range(j):
                h[i], h[i + 1] = cs[i] * h[i] + sn[i] * h[i + 1], -sn[i] * h[i] + cs[i] * h[i + 1]
            rr = np.hypot(h[j], h[j + 1])
            cs[j], sn[j] = h[j] / rr, h[j + 1] / rr
            h[j] = rr
            rm[: j + 1, j] = h[: j + 1]
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            done = abs(g[j + 1]) <= rf * bnorm or total >= max_iters
            if done or j + 1 == m:
                k = j + 1
                y = np.zeros(k)
                for i in range(k - 1, -1, -1):
                    y[i] = (g[i] - rm[i, i + 1:k] @ y[i + 1:k]) / rm[i, i]
                z = np.zeros_like(b)
                for i in range(k):
                    z = sbref.axpy(float(y[i]), basis[i], z)
                x = sbref.axpy(1.0, z * R.inv, x)
                if done:
                    return total
                break
            basis.append(sbref.scal(1.0 / hn, w))


def _krylov_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci, v = fixtures.stencil_csr(10, dim=3, c=0.5)
        R = _Rank(rp, ci, v, rank, world)
        b = np.ones(R.hi - R.lo)
        results[("bicgstab", rank)] = _bicgstab(R, b, 1e-8, 2000)
        results[("gmres", rank)] = _gmres(R, b, 1e-8, 2000, 10)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_bicgstab_gmres_gloo(world):
    """The partitioned BiCGSTAB / GMRES(10) sync structure over a real multi-process
    backend (gloo): every rank stops at the same iteration, within +-2% of the oracle's
    single-process solve (only the dot summation order differs)."""
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_krylov_worker, args=(world, port, results), nprocs=world, join=True)
    rp, ci, v = fixtures.stencil_csr(10, dim=3, c=0.5)
    inv = sbref.jacobi_create(rp, ci, v)[0]
    b = np.ones(rp.size - 1)
    for kind, kw in (("bicgstab", {}), ("gmres", {"krylov_dim": 10})):
        its = {results[(kind, r)] for r in range(world)}
        assert len(its) == 1, (kind, its)  # identical scalars on every rank
        ref = sbref.solve(kind, rp, ci, v, b, inv_diag=inv, max_iters=2000, reduction_factor=1e-8, **kw)[0]
        assert ref.converged
        it = its.pop()
        assert abs(it - ref.iterations) <= max(1, int(np.ceil(0.02 * ref.iterations))), (kind, it, ref.iterations)

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

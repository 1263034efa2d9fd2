"""Rayleigh-Ritz on the device (test_rayleigh_ritz.py of the reference frontend)."""

import numpy as np
import pytest

import paper_2510_08230_b200.pysparseops as pg
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as core
from paper_2510_08230_b200.pysparseops.errors import OrthonormalityError
from tests.gpu_util import host

pytestmark = pytest.mark.gpu


def _basis(rng, n, k):
    q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return np.ascontiguousarray(q)


def test_diagonal_identity_basis():
    dev = pg.device("cuda")
    a = core.csr_from_dense(dev, np.diag([1.0, 2.0, 3.0]))
    values, vectors = pg.rayleigh_ritz(a, pg.as_tensor(np.eye(3), device=dev))
    np.testing.assert_array_equal(values, [1.0, 2.0, 3.0])
    np.testing.assert_allclose(np.abs(host(vectors)), np.eye(3), atol=1e-14)


def test_full_space_and_invariant_subspace():
    dev = pg.device("cuda")
    rng = np.random.default_rng(61)
    sym = rng.standard_normal((50, 50))
    sym = (sym + sym.T) / 2
    a = core.csr_from_dense(dev, sym, keep_zeros=True)
    values, _ = pg.rayleigh_ritz(a, pg.as_tensor(_basis(rng, 50, 50), device=dev))
    oracle_vals, oracle_vecs = np.linalg.eigh(sym)
    np.testing.assert_allclose(values, oracle_vals, atol=1e-8 * np.abs(oracle_vals).max())
    span = np.ascontiguousarray(oracle_vecs[:, 3:7])
    values, _ = pg.rayleigh_ritz(a, pg.as_tensor(span, device=dev))
    np.testing.assert_allclose(values, oracle_vals[3:7], atol=1e-10)


def test_large_stencil_subspace_uses_spmm():
    """3-D Poisson 32^3 (stream CSR -> one SpMM for the 6 basis vectors): Ritz values lie
    inside the spectrum (0, 12) and match the host projection."""
    dev = pg.device("cuda")
    a = gen.stencil_csr(core.create_device("cuda", 0), 32, dim=3)
    rng = np.random.default_rng(62)
    basis = _basis(rng, a.rows, 6)
    values, vectors = pg.rayleigh_ritz(a, pg.as_tensor(basis, device=dev))
    assert np.all(np.diff(values) >= 0) and values[0] > 0 and values[-1] < 12
    from oracle import sbref
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    av = np.stack([sbref.csr_spmv(rp, ci, v, basis[:, j]) for j in range(6)], axis=1)
    h = basis.T @ av
    np.testing.assert_allclose(values, np.linalg.eigh((h + h.T) / 2)[0], rtol=1e-12)
    assert host(vectors).shape == (a.rows, 6)


def test_errors():
    dev = pg.device("cuda")
    a = core.csr_from_dense(dev, np.eye(4))
    with pytest.raises(OrthonormalityError):
        pg.rayleigh_ritz(a, pg.as_tensor(np.ones((4, 2)), device=dev))
    with pytest.raises(core.errors.DimensionMismatchError):
        pg.rayleigh_ritz(a, pg.as_tensor(np.eye(3), device=dev))

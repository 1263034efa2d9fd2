"""GPU tests of the drop-in frontend (the reference's pkg/frontend/tests, restated for the
``cuda`` device): the Listing-1 / Listing-2 programs run verbatim with
``pg.device("cuda")``, dispatch reaches every typed instantiation, zero-copy torch
interop, and core error kinds cross the binding boundary unchanged."""

import numpy as np
import pytest
import torch

import paper_2510_08230_b200.pysparseops as pg
from paper_2510_08230_b200 import sparseops as core
from paper_2510_08230_b200.pysparseops import bindings
from tests.gpu_util import host

pytestmark = pytest.mark.gpu

# Listing 1 of the paper / test_pipeline_example.py:11-37 verbatim, with the CUDA device:
# ILU(0)-preconditioned GMRES(30)
PIPELINE = """
import paper_2510_08230_b200.pysparseops as pg
import numpy as np

fn = 'm1.mtx'
dev = pg.device("cuda")
mtx = pg.read(device=dev, path=fn, dtype="double", format="Csr")
n_rows = mtx.size[0]

b = pg.as_tensor(
  device=dev, dim=(n_rows,1), dtype="double", fill=1.0
)
x = pg.as_tensor(
  device=dev, dim=(n_rows,1), dtype="double", fill=0.0
)

# Create ILU preconditioner
preconditioner = pg.preconditioner.Ilu(dev, mtx)

#Setup GMRES solver
solver = pg.solver.gmres(dev, mtx, preconditioner,
    max_iters=1000, krylov_dim=30, reduction_factor=1e-06
)

#Apply
logger, result = solver.apply(b, x)
"""


@pytest.fixture
def mtx_file(tmp_path, monkeypatch):
    p = 6
    n = p * p
    trip = []
    for gy in range(p):
        for gx in range(p):
            i = gy * p + gx
            trip.append((i, i, 4.0))
            for j in (i - 1 if gx else None, i + 1 if gx < p - 1 else None,
                      i - p if gy else None, i + p if gy < p - 1 else None):
                if j is not None:
                    trip.append((i, j, -1.0))
    dev = pg.device("cuda")
    m = core.csr_from_coo(core.coo_from_triplets(dev, n, n, trip))
    core.write_matrix_market(m, tmp_path / "m1.mtx")
    monkeypatch.chdir(tmp_path)
    return m


@pytest.mark.parametrize("precond", ["Ilu", "Jacobi", "Ic"])
def test_listing1_runs_verbatim(mtx_file, precond):
    ns = {}
    exec(compile(PIPELINE.replace("preconditioner.Ilu(", f"preconditioner.{precond}("),
                 "pipeline_example", "exec"), ns)
    logger, result, x, b, mtx = ns["logger"], ns["result"], ns["x"], ns["b"], ns["mtx"]
    assert result is x
    assert logger.converged and logger.stop_reason == "residual"
    assert len(logger.residual_history) == logger.iterations >= 1
    dense = mtx.to_dense()
    bv, xv = host(b), host(result)
    assert np.linalg.norm(bv - dense @ xv) / np.linalg.norm(bv) <= 1e-6 * (1 + 1e-8)
    np.testing.assert_array_equal(bv, np.ones(mtx.rows))


def test_listing2_config_solve(mtx_file):
    dev = pg.device("cuda")
    mtx = pg.read(dev, "m1.mtx")
    args = {"type": "solver::Gmres", "krylov_dim": 30,
            "preconditioner": {"type": "preconditioner::Jacobi"},
            "criteria": [{"type": "Iteration", "max_iters": 1000},
                         {"type": "ResidualNorm", "reduction_factor": 1e-06}]}
    b = pg.as_tensor(device=dev, dim=(mtx.rows, 1), fill=1.0)
    x = pg.as_tensor(device=dev, dim=(mtx.rows, 1), fill=0.0)
    logger, result = pg.solve(args, mtx, b, x)
    assert result is x and logger.converged
    args["preconditioner"] = {"type": "preconditioner::Ilu"}
    x2 = pg.as_tensor(device=dev, dim=(mtx.rows, 1), fill=0.0)
    logger2, _ = pg.solve(args, mtx, b, x2)
    assert logger2.converged and logger2.stop_reason == "residual"


def test_dispatch_reaches_every_instantiation():
    """test_dispatch.py:19-50: each (value, index) combination routes to its binding."""
    dev = pg.device("cuda")
    rng = np.random.default_rng(3)
    dense = (rng.random((9, 7)) < 0.3) * rng.standard_normal((9, 7))
    for vname, vdt in bindings.VALUE_DTYPES.items():
        for iname, idt in bindings.INDEX_DTYPES.items():
            prec = core.Precision.from_dtype(vdt)
            iw = core.IndexWidth.from_dtype(idt)
            csr = core.csr_from_dense(dev, dense, prec, iw)
            mats = {"csr": csr, "coo": core.coo_from_csr(csr), "ell": core.ell_from_csr(csr),
                    "sellp": core.sellp_from_csr(csr), "hybrid": core.hybrid_from_csr(csr)}
            b = pg.as_tensor(rng.standard_normal(7).astype(vdt), device=dev)
            for fmt, m in mats.items():
                x = pg.as_tensor(device=dev, dim=9, dtype=vname, fill=0.0)
                pg.spmv(m, b, x)
                np.testing.assert_allclose(host(x), dense.astype(vdt) @ host(b), rtol=1e-5,
                                           atol=1e-5, err_msg=f"{fmt} {vname} {iname}")
                fn = getattr(bindings, f"{fmt}_spmv_{vname}_{iname}")
                fn(m, b, x)
                with pytest.raises(pg.InstantiationMismatchError):
                    other = "float" if vname == "double" else "double"
                    getattr(bindings, f"{fmt}_spmv_{other}_{iname}")(m, b, x)
    with pytest.raises(pg.NoMatchingInstantiationError):
        pg.spmv(csr, pg.as_tensor(np.ones(7), device=dev), pg.as_tensor(device=dev, dim=9, dtype="float", fill=0.0))


def test_zero_copy_torch_tensors():
    """test_tensor.py:11-40 with CUDA tensors: shared memory both ways, copies flagged."""
    dev = pg.device("cuda")
    src = torch.tensor([1.0, 2.0, 3.0], device="cuda")
    t = pg.as_tensor(src, device=dev)
    assert t.copied is False
    src[0] = 9.0
    assert pg.dot(t, t) == 81.0 + 4.0 + 9.0
    t.values[1] = -5.0
    assert float(src[1]) == -5.0
    f32 = torch.ones(4, dtype=torch.float32, device="cuda")
    c = pg.as_tensor(f32, device=dev, dtype="double")
    assert c.copied and c.values.dtype == torch.float64
    with pytest.raises(pg.CopyRequiredError):
        pg.as_tensor(f32, device=dev, dtype="double", copy=False)
    h = pg.as_tensor(np.arange(4.0), device=dev)  # host data crosses to the device: a copy
    assert h.copied and pg.norm2(h) == pytest.approx(np.sqrt(14.0))
    with pytest.raises(pg.CopyRequiredError):
        pg.as_tensor(np.arange(4.0), device=dev, copy=False)


def test_error_kinds_cross_the_boundary():
    """test_solve_api.py:146-152: core exception classes surface unchanged."""
    dev = pg.device("cuda")
    zero = core.csr_from_dense(dev, np.zeros((2, 2)))
    b = pg.as_tensor(np.array([1.0, 2.0]), device=dev)
    x = pg.as_tensor(device=dev, dim=2, fill=0.0)
    with pytest.raises(core.errors.BreakdownError) as exc:
        pg.solver.cg(dev, zero, None, max_iters=10).apply(b, x)
    assert exc.value.kind == "breakdown" and exc.value.iteration == 1
    with pytest.raises(core.errors.SingularDiagonalError) as exc:
        pg.preconditioner.Jacobi(dev, zero)
    assert exc.value.kind == "singular-diagonal" and exc.value.row == 0
    a = core.csr_from_dense(dev, np.eye(3))
    with pytest.raises(core.errors.DimensionMismatchError):
        pg.spmv(a, pg.as_tensor(np.ones(2), device=dev), pg.as_tensor(device=dev, dim=3, fill=0.0))
    with pytest.raises(core.errors.ConfigError) as exc:
        pg.solve({"type": "solver::Cg", "criteria": []}, a, b, x)
    assert exc.value.path == "criteria"


def test_matrix_constructors():
    import scipy.sparse as sps

    dev = pg.device("cuda")
    m = sps.random(40, 40, density=0.1, random_state=4, format="csr") + sps.eye(40) * 5
    for fmt in ("csr", "coo", "ell", "sellp", "hybrid"):
        a = pg.matrix(dev, m, format=fmt)
        np.testing.assert_allclose(a.to_dense(), m.toarray(), rtol=0, atol=1e-15)
    t = pg.matrix(dev, torch.tensor(m.toarray()).to_sparse())
    np.testing.assert_array_equal(t.to_dense(), m.toarray())
    logger, x = pg.solver.bicgstab(dev, pg.matrix(dev, m), max_iters=200,
                                   reduction_factor=1e-10).apply(
        pg.as_tensor(np.ones(40), device=dev), pg.as_tensor(device=dev, dim=40, fill=0.0))
    assert logger.converged
    np.testing.assert_allclose(m @ host(x), np.ones(40), atol=1e-8)


def test_every_reference_registry_name_runs(tmp_path):
    """All 36 reference registry names (frontend bindings.py:27-40, 81-145) execute on the
    device; none raises UnsupportedFeatureError.  The triangular solves reproduce the
    reference's ILU apply (precond.py:117-121) bit for bit from its own factors."""
    from tests import golden_io

    dev = pg.device("cuda")
    ref = [n for n, i in bindings.REGISTRY.items() if i.op in bindings.REFERENCE_OPS]
    assert len(ref) == 36
    called = set()
    (tmp_path / "m.mtx").write_text(
        "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 2\n2 2 3\n3 1 -1\n3 3 4\n")
    for vname, vdt in bindings.VALUE_DTYPES.items():
        fac = golden_io.unpack(golden_io.load(f"factor_{vdt.name}.npz"))[0]
        for iname, idt in bindings.INDEX_DTYPES.items():
            prec = core.Precision.from_dtype(vdt)
            sfx = f"{vname}_{iname}"

            def mat(p, c, v):
                n = len(p) - 1
                return core.CsrMatrix(dev, n, n, np.asarray(p, idt), np.asarray(c, idt),
                                      np.asarray(v, vdt))

            n = len(fac["ilu_l_ptrs"]) - 1
            lo = mat(fac["ilu_l_ptrs"], fac["ilu_l_cols"], fac["ilu_l_vals"])
            up = mat(fac["ilu_u_ptrs"], fac["ilu_u_cols"], fac["ilu_u_vals"])
            b = pg.as_tensor(fac["b"].astype(vdt), device=dev)
            y = core.dense_create(dev, n, 1, prec, 0.0)
            x = core.dense_create(dev, n, 1, prec, 0.0)
            getattr(bindings, f"lower_trisolve_{sfx}")(lo, b, y, unit_diag=True)
            getattr(bindings, f"upper_trisolve_{sfx}")(up, y, x)
            assert host(x).tobytes() == fac["ilu_x"].astype(vdt).tobytes()
            called |= {f"lower_trisolve_{sfx}", f"upper_trisolve_{sfx}"}
            a = getattr(bindings, f"read_csr_{sfx}")(dev, tmp_path / "m.mtx")
            c = getattr(bindings, f"read_coo_{sfx}")(dev, tmp_path / "m.mtx")
            called |= {f"read_csr_{sfx}", f"read_coo_{sfx}"}
            bb = getattr(bindings, f"dense_{vname}")(dev, np.array([1.0, 2.0, 3.0], vdt))
            xx = getattr(bindings, f"dense_create_{vname}")(dev, 3, 1, np.nan)
            getattr(bindings, f"csr_spmv_{sfx}")(a, bb, xx)
            np.testing.assert_array_equal(host(xx), [2.0, 6.0, 11.0])
            getattr(bindings, f"coo_spmv_{sfx}")(c, bb, xx)
            np.testing.assert_array_equal(host(xx), [2.0, 6.0, 11.0])
            called |= {f"csr_spmv_{sfx}", f"coo_spmv_{sfx}", f"dense_{vname}",
                       f"dense_create_{vname}"}
            assert getattr(bindings, f"dot_{vname}")(bb, bb) == 14.0
            assert getattr(bindings, f"norm2_{vname}")(bb) == pytest.approx(np.sqrt(14.0))
            getattr(bindings, f"axpy_{vname}")(2.0, bb, xx)
            getattr(bindings, f"scal_{vname}")(0.5, xx)
            np.testing.assert_array_equal(host(xx), [2.0, 5.0, 8.5])
            called |= {f"dot_{vname}", f"norm2_{vname}", f"axpy_{vname}", f"scal_{vname}"}
    assert called == set(ref)

"""CPU-side checks: the C-ABI library loads and exports exactly the declared symbols,
host-only logic (kernel selection, criteria reduction, config parsing, dispatch) and
the frontend error conventions.  No GPU needed."""

import ctypes
import re
import subprocess

import numpy as np
import pytest

from paper_2510_08230_b200 import _lib
from paper_2510_08230_b200 import pysparseops as pg
from paper_2510_08230_b200 import sparseops as sp

HEADER = "include/sparseb200.h"


def _header_symbols():
    """Function names declared by the header, after the C preprocessor expands the
    per-type declaration macros."""
    pre = subprocess.run(["gcc", "-E", "-P", "-x", "c", HEADER], capture_output=True, text=True,
                         check=True).stdout
    return set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", pre))


def test_library_exports_exactly_the_header():
    lib = _lib.load()
    declared = _header_symbols()
    assert len(declared) >= 90
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r" T (sb_[a-z0-9_]+)", nm))
    assert declared == exported, (declared ^ exported)
    assert set(_lib.all_prototypes()) == exported
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.sb_version() == 1
    assert lib.sb_status_string(6) == b"breakdown"


def test_plan_selection_host_logic():
    def select(rows, nnz, mn, mx, block, force=0, vb=8, ib=4):
        st = _lib.SbRowStats(rows, nnz, mn, mx, 0, nnz / rows, 0.0, (ctypes.c_int64 * 4)(*block))
        plan = _lib.SbCsrPlan()
        _lib.call("sb_csr_plan_select", ctypes.byref(st), vb, ib, force, ctypes.byref(plan))
        return plan

    p = select(2_097_152, 14_581_760, 4, 7, [224, 448, 896, 1792])  # Poisson 128^3
    assert p.kernel == _lib.CSR_STREAM and p.block_rows == 128 and p.nnz_cap == 896
    p = select(4_000_000, 63_958_208, 1, 11668, [20000, 20000, 20000, 20000])  # power-law
    assert p.kernel == _lib.CSR_TILE and p.num_tiles == 2 * -(-63_958_208 // 2048)
    p = select(4_000_000, 63_958_208, 1, 11668, [20000, 20000, 20000, 20000], force=_lib.CSR_MERGE)
    assert p.kernel == _lib.CSR_MERGE and p.num_tiles == -(-(4_000_000 + 63_958_208) // 1024)
    p = select(10000, 640000, 60, 70, [2240, 4480, 8960, 17920])  # long regular rows
    assert p.kernel == _lib.CSR_VECTOR and p.block_rows == 32
    p = select(100, 0, 0, 0, [0, 0, 0, 0])
    assert p.kernel == _lib.CSR_STRICT
    with pytest.raises(sp.errors.UnsupportedFeatureError):
        select(10, 10**7, 1, 10**6, [10**7] * 4, force=_lib.CSR_STREAM)


def test_workspace_sizes():
    f = _lib.fn("sb_solver_workspace_bytes")
    n = 2_097_152
    cg = f(_lib.SOLVER_CG, 8, n, 0, 1000)
    assert cg >= 5 * 8 * n
    gm = f(_lib.SOLVER_GMRES, 8, n, 30, 1000)
    assert gm >= 35 * 8 * n
    assert _lib.fn("sb_coo_from_arrays_workspace_bytes")(1000) > 6 * 8 * 1000


def test_device_names():
    with pytest.raises(sp.errors.UnsupportedBackendError):
        pg.device("omp")
    with pytest.raises(sp.errors.UnsupportedBackendError):
        pg.device("reference")
    with pytest.raises(sp.errors.UnsupportedBackendError):
        pg.device("hip")
    with pytest.raises(sp.errors.UnknownDeviceError):
        pg.device("tpu")


def test_bindings_registry_and_dispatch():
    from paper_2510_08230_b200.pysparseops import bindings, dispatch

    ref = [n for n, i in bindings.REGISTRY.items() if i.op in bindings.REFERENCE_OPS]
    assert len(ref) == 36  # the reference's 36 instantiations (test_dispatch.py:20-24)
    assert "csr_spmv_double_i32" in bindings.REGISTRY
    assert "sellp_spmv_float_i64" in bindings.REGISTRY
    assert "bicgstab_solve_double_i32" in bindings.REGISTRY
    assert dispatch.resolve("csr_spmv", np.float64, np.int32) is bindings.csr_spmv_double_i32
    with pytest.raises(pg.NoMatchingInstantiationError) as exc:
        dispatch.resolve("csr_spmv", np.float16, np.int32)
    assert "csr_spmv_double_i32" in exc.value.candidates
    with pytest.raises(pg.NoMatchingInstantiationError):
        dispatch.value_dtype("half")
    assert dispatch.value_dtype("single") == np.float32


def test_criteria_and_config():
    from paper_2510_08230_b200.sparseops.solvers import _criteria_struct

    c = _criteria_struct([sp.Iteration(50), sp.Iteration(20), sp.ResidualNorm(1e-6),
                          sp.ResidualNorm(1e-4)])
    assert (c.max_iters, c.has_residual, c.reduction_factor) == (20, 1, 1e-4)
    assert sp.check_criteria([sp.Iteration(5), sp.ResidualNorm(0.5)], 5, 1.0, 2.0) == "residual"
    assert sp.check_criteria([sp.Iteration(5)], 5, 1.0, 2.0) == "max_iters"
    assert sp.check_criteria([sp.Iteration(5), sp.ResidualNorm(0.5)], 1, 0.4, 0.0) == "residual"
    assert sp.givens_rotation(3.0, 4.0) == (0.6, 0.8, 5.0)
    with pytest.raises(sp.errors.InvalidArgumentError):
        sp.validate_criteria([sp.ResidualNorm(1e-6)])
    tree = {"type": "solver::Gmres", "preconditioner": {"type": "preconditioner::Jacobi"},
            "criteria": [{"type": "Iteration", "max_iters": 100},
                         {"type": "ResidualNorm", "reduction_factor": 1e-6}]}
    cfg = sp.parse_config(tree)
    assert cfg.krylov_dim == 30 and cfg.preconditioner.type == "preconditioner::Jacobi"
    assert sp.parse_config({"type": "solver::Bicgstab",
                            "criteria": [{"type": "Iteration", "max_iters": 3}]}).type == \
        "solver::Bicgstab"
    bad = [({"type": "solver::Cg", "criteria": [{"type": "Iteration", "max_iters": True}]},
            "criteria[0].max_iters"),
           ({"type": "solver::Cg", "krylov_dim": 3, "criteria": []}, "krylov_dim"),
           ({"type": "solver::Nope"}, "type"),
           ({"type": "solver::Cg", "criteria": [{"type": "ResidualNorm", "reduction_factor": 1}]},
            "criteria"),
           ({"type": "solver::Cg", "preconditioner": {"type": "preconditioner::Jacobi", "x": 1},
             "criteria": [{"type": "Iteration", "max_iters": 1}]}, "preconditioner.x")]
    for t, path in bad:
        with pytest.raises(sp.errors.ConfigError) as exc:
            sp.parse_config(t)
        assert exc.value.path == path, (t, exc.value.path)


def test_reference_fixture_config_parses():
    import json
    import os

    path = "/root/reference/pkg/tests/fixtures/gmres_jacobi.json"
    if not os.path.exists(path):
        pytest.skip("reference not mounted")
    cfg = sp.load_config(path)
    assert cfg.type == "solver::Gmres"
    assert cfg == sp.parse_config(json.load(open(path)))

"""Matrix Market ingest vs the REFERENCE reader (tests/golden/mmio_corpus.json).

The corpus holds the bodies of the reference's own ``pkg/tests/test_mmio.py:26-191``
plus the cases its parser distinguishes (explicit zeros in array bodies, several values
per line, non-integral / out-of-range indices, ...).  For every file the golden records
what the reference's ``read_matrix_market`` returned: the canonical integer arrays and
value bit patterns, the warning classes, or the exception class.

* CPU (``not gpu``): the host parser ``mmio.read_entries`` followed by the oracle's
  ``coo_from_arrays`` restatement must reproduce the reference bit for bit.
* GPU: the product path ``read_matrix_market`` (device canonicalisation) must too.
"""

import json
import os
import warnings

import numpy as np
import pytest

from paper_2510_08230_b200.sparseops import errors, mmio
from tests.conftest import GOLDEN

CORPUS = json.load(open(os.path.join(GOLDEN, "mmio_corpus.json")))
CASES = CORPUS["cases"]
IDS = [c["name"] for c in CASES]


def _write(tmp_path, case):
    path = tmp_path / (case["name"] + ".mtx")
    path.write_text(case["text"])
    return path


def _expected(case):
    vdt = np.float32 if case["precision"] == "single" else np.float64
    idt = np.int64 if case["index_width"] == "i64" else np.int32
    vals = np.array([float.fromhex(h) for h in case["values_hex"]], np.float64).astype(vdt)
    return vdt, idt, vals


def _read_host(path, case):
    """Host parser + oracle canonicalisation (test infrastructure, not the product)."""
    from oracle import sbref

    if case["format"].lower() not in ("csr", "coo"):
        # the target-format check precedes any parsing (reference mmio.py:206-208)
        mmio.read_matrix_market(None, path, format=case["format"])
    _, rows, cols, ri, ci, vals = mmio.read_entries(path)
    vdt, idt, _ = _expected(case)
    r, c, v = sbref.coo_canonicalize(ri, ci, vals, vdt)
    out = {"shape": [rows, cols], "col_idxs": c.astype(idt), "values": v}
    if case["format"].lower() == "csr":
        out["row_ptrs"] = sbref.csr_row_ptrs(r, rows, idt)
    else:
        out["row_idxs"] = r.astype(idt)
    return out


def _check(got, case):
    vdt, idt, vals = _expected(case)
    assert list(got["shape"]) == case["shape"]
    key = "row_ptrs" if "row_ptrs" in case else "row_idxs"
    np.testing.assert_array_equal(np.asarray(got[key]), np.asarray(case[key], idt))
    np.testing.assert_array_equal(np.asarray(got["col_idxs"]), np.asarray(case["col_idxs"], idt))
    gv = np.asarray(got["values"])
    assert gv.dtype == vdt
    assert gv.tobytes() == vals.tobytes()  # bit for bit


def _run(reader, path, case):
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        if "error" in case:
            with pytest.raises(errors.SparseOpsError) as ei:
                reader(path, case)
            assert type(ei.value).__name__ == case["error"]
            return None
        got = reader(path, case)
    names = sorted({type(w.message).__name__ for w in caught
                    if issubclass(w.category, UserWarning)})
    assert names == case["warnings"]
    return got


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_host_parse_matches_reference(tmp_path, case):
    got = _run(_read_host, _write(tmp_path, case), case)
    if got is not None:
        _check(got, case)


def test_corpus_covers_reference_suite():
    """Every body of the reference's test_mmio.py TestRead is in the corpus."""
    names = set(IDS)
    for n in ("basic", "coo_target", "symmetric", "symmetric_offdiag_only", "skew",
              "banner_case", "bad_banner", "comments_blank", "pattern", "integer_f32",
              "complex", "count_mismatch", "index_oob", "bad_size", "duplicates", "array",
              "array_symmetric", "garbage_entry"):
        assert n in names
    # explicit zeros are kept in array bodies (reference mmio.py:128-166)
    z = next(c for c in CASES if c["name"] == "array_zeros")
    assert len(z["col_idxs"]) == 9


def test_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        mmio.read_entries(tmp_path / "nope.mtx")


def test_writer_signature_is_reference_order():
    import inspect

    assert list(inspect.signature(mmio.write_matrix_market).parameters) == ["m", "path"]


def test_header_and_warning_exported():
    from paper_2510_08230_b200 import sparseops as sp

    assert sp.MatrixMarketHeader is mmio.MatrixMarketHeader
    assert issubclass(sp.DuplicateEntryWarning, UserWarning)
    assert mmio.parse_banner("%%MatrixMarket matrix array integer symmetric") == \
        mmio.MatrixMarketHeader("matrix", "array", "integer", "symmetric")


# ----------------------------------------------------------------------------- GPU


def _read_device(dev):
    from paper_2510_08230_b200 import sparseops as sp

    def reader(path, case):
        m = sp.read_matrix_market(dev, path, getattr(sp.Precision, case["precision"]),
                                  case["format"], getattr(sp.IndexWidth, case["index_width"]))
        assert type(m).__name__ == case["type"]
        out = {"shape": [m.rows, m.cols], "col_idxs": m.col_idxs.cpu().numpy(),
               "values": m.values.cpu().numpy()}
        if case["type"] == "CsrMatrix":
            out["row_ptrs"] = m.row_ptrs.cpu().numpy()
        else:
            out["row_idxs"] = m.row_idxs.cpu().numpy()
        return out

    return reader


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_device_read_matches_reference(dev, tmp_path, case):
    got = _run(_read_device(dev), _write(tmp_path, case), case)
    if got is not None:
        _check(got, case)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CORPUS["writer"]))
def test_writer_text_matches_reference(dev, tmp_path, name):
    from paper_2510_08230_b200 import sparseops as sp

    if name == "dense2":
        m = sp.csr_from_dense(dev, np.array([[1.0, 0.0], [0.0, 3.0]]))
    elif name == "awkward":
        awkward = [0.1, 1.0 / 3.0, np.pi, 1e-300, 1e300, -2.2250738585072014e-308]
        m = sp.coo_from_triplets(dev, 6, 1, [(i, 0, v) for i, v in enumerate(awkward)])
    elif name == "empty":
        m = sp.coo_from_triplets(dev, 3, 3, [])
    else:
        m = sp.csr_from_coo(sp.coo_from_triplets(dev, 2, 2, [(0, 1, 0.5), (1, 0, 0.25)],
                                                 sp.Precision.single))
    path = tmp_path / "w.mtx"
    sp.write_matrix_market(m, path)
    assert path.read_text() == CORPUS["writer"][name]
    back = sp.read_matrix_market(dev, path, m.precision, "Coo")
    np.testing.assert_array_equal(back.values.cpu().numpy(), m.values.cpu().numpy())

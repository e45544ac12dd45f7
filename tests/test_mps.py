"""MPS ingestion parity (CPU): the product's reader/writer (csrc/mps.cpp) vs
the reference's ParseMpsString / WriteMps, pinned by the committed fixtures
tests/golden/mps_golden.json (generated from the reference build by
tests/golden/make_mps_golden.py) and, where the reference build exists, live.
Bit-exact on every array; identical error messages and line numbers."""
import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import GenRandomLp, GenTransport, MpsParseError, ParseMpsFile, ParseMpsString, WriteMps

import mps_corpus

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "mps_golden.json").read_text())


def unhex(v):
    return np.array([float.fromhex(x) for x in v], dtype=np.float64)


def assert_matches(p, g):
    assert g["code"] == 0
    assert p.name == g["name"]
    assert p.num_vars() == g["n"]
    for m, gm in ((p.a, g["a"]), (p.g, g["g"])):
        assert m.rows == gm["rows"]
        np.testing.assert_array_equal(m.row_ptr, np.array(gm["row_ptr"], np.int64))
        np.testing.assert_array_equal(m.col_idx, np.array(gm["col_idx"], np.int64))
        np.testing.assert_array_equal(m.values.view(np.uint64), unhex(gm["values"]).view(np.uint64))
    for k in ("c", "b", "h", "l", "u"):
        np.testing.assert_array_equal(getattr(p, k).view(np.uint64), unhex(g[k]).view(np.uint64))
    assert float(p.objective_offset).hex() == g["offset"]
    assert int(p.negated_objective) == g["negated"]


@pytest.mark.parametrize("name", sorted(mps_corpus.GOOD))
def test_good_files_match_reference(name):
    assert_matches(ParseMpsString(mps_corpus.GOOD[name]), GOLD["good"][name])


@pytest.mark.parametrize("name", sorted(mps_corpus.FIXED))
def test_fixed_format_matches_reference(name):
    g = GOLD["fixed"][name]
    if g["code"] == 0:
        assert_matches(ParseMpsString(mps_corpus.FIXED[name], fixed_format=True), g)
    else:
        with pytest.raises(MpsParseError) as e:
            ParseMpsString(mps_corpus.FIXED[name], fixed_format=True)
        assert str(e.value) == g["error"] and e.value.line == g["line"]


@pytest.mark.parametrize("name", sorted(mps_corpus.BAD))
def test_errors_match_reference(name):
    g = GOLD["bad"][name]
    if g["code"] == 6:
        with pytest.raises(MpsParseError) as e:
            ParseMpsString(mps_corpus.BAD[name])
        assert str(e.value) == g["error"] and e.value.line == g["line"]
    else:  # LpProblem::Validate -> std::invalid_argument
        with pytest.raises(ValueError) as e:
            ParseMpsString(mps_corpus.BAD[name])
        assert str(e.value) == g["error"]


def test_writer_matches_reference():
    from golden.make_mps_golden import writer_cases
    for k, p in writer_cases().items():
        assert WriteMps(p) == GOLD["writer"][k]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_round_trip(seed, tmp_path):
    """WriteMps -> ParseMps reproduces the problem bit for bit (the
    reference's own round-trip test, test_mps.cpp)."""
    p = GenRandomLp(30, 40, 0.2, seed, equality_rows=10)
    p.l[0], p.u[0] = -np.inf, np.inf
    p.u[1] = np.inf
    p.l[2] = p.u[2] = 0.5
    p.objective_offset = -1.5
    q = ParseMpsString(WriteMps(p))
    for m1, m2 in ((p.a, q.a), (p.g, q.g)):
        np.testing.assert_array_equal(m1.row_ptr, m2.row_ptr)
        np.testing.assert_array_equal(m1.col_idx, m2.col_idx)
        np.testing.assert_array_equal(m1.values, m2.values)
    for k in ("c", "b", "h", "l", "u"):
        np.testing.assert_array_equal(getattr(p, k), getattr(q, k))
    assert q.objective_offset == p.objective_offset
    # files, plain and gzip
    f = tmp_path / "p.mps"
    rpdlp.WriteMpsFile(p, f)
    r = ParseMpsFile(f)
    np.testing.assert_array_equal(r.g.values, p.g.values)
    gz = tmp_path / "p.mps.gz"
    gz.write_bytes(gzip.compress(f.read_bytes()))
    r2 = ParseMpsFile(gz)
    np.testing.assert_array_equal(r2.a.values, p.a.values)


def test_negated_objective_round_trip():
    p = ParseMpsString(mps_corpus.GOOD["objsense_header"])
    assert p.negated_objective and p.c[0] == -3.0
    q = ParseMpsString(WriteMps(p))
    assert q.negated_objective
    np.testing.assert_array_equal(q.c, p.c)
    assert q.objective_offset == p.objective_offset


def test_missing_file():
    with pytest.raises(OSError, match="cannot open"):
        ParseMpsFile("/nonexistent/x.mps")


def test_live_reference_on_generated_files(reference):
    """Larger generated instances through both parsers (reference build only)."""
    if reference is None:
        pytest.skip("reference build absent")
    import ctypes as C
    from golden.make_mps_golden import ref_lib, ref_parse
    lib = ref_lib()
    for p in (GenTransport(20, 30, 1), GenRandomLp(50, 80, 0.1, 7, equality_rows=20)):
        text = WriteMps(p)
        assert_matches(ParseMpsString(text), ref_parse(lib, text, False))
    del C


def test_parsed_problem_solves_like_generated(restatement):
    """A problem that went through the MPS writer and reader solves to the same
    result as the in-memory one (restatement)."""
    p = GenRandomLp(20, 30, 0.3, 5, equality_rows=5)
    q = ParseMpsString(WriteMps(p))
    a = restatement.solve(p, rpdlp.SolverParams(eps=1e-6))
    b = restatement.solve(q, rpdlp.SolverParams(eps=1e-6))
    assert a.iterations == b.iterations and a.report.primal_obj == b.report.primal_obj


def _big_text():
    p = GenRandomLp(3000, 4000, 0.05, 9, equality_rows=500)
    return WriteMps(p)


def test_parallel_columns_large_file_matches_reference(reference):
    """A COLUMNS section of tens of MB is tokenised on worker threads
    (mps.cpp Reader::ColumnsBlock, >= 1 MB per chunk) and merged in file
    order: bit-identical to the reference parser."""
    if reference is None:
        pytest.skip("reference build absent")
    from golden.make_mps_golden import ref_lib, ref_parse
    text = _big_text()
    assert len(text) > 8 << 20  # several chunks
    assert_matches(ParseMpsString(text), ref_parse(ref_lib(), text, False))


@pytest.mark.parametrize("where", [0.3, 0.55, 0.97])
def test_parallel_columns_first_error_wins(where, reference):
    """Errors inside a chunked COLUMNS section: the first one in file order is
    reported, with the reference's message and line number, even when a later
    chunk fails too."""
    if reference is None:
        pytest.skip("reference build absent")
    from golden.make_mps_golden import ref_lib, ref_parse
    lines = _big_text().split("\n")
    c0 = lines.index("COLUMNS") + 1
    c1 = next(i for i in range(c0, len(lines)) if lines[i] and not lines[i][0].isspace())
    k = c0 + int(where * (c1 - c0))
    f = lines[k].split()
    lines[k] = "    " + f[0] + "  NOPE_ROW  1.0"               # unknown row
    lines[c1 - 2] = lines[c1 - 2].rsplit(None, 1)[0] + "  1.0x"  # a later bad number
    text = "\n".join(lines)
    g = ref_parse(ref_lib(), text, False)
    assert g["code"] != 0
    with pytest.raises(Exception) as ei:
        ParseMpsString(text)
    assert str(ei.value) == g["error"] or g["error"] in str(ei.value)
    assert f"line {g['line']}:" in str(ei.value)

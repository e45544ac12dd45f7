"""Device-side problem assembly: pdhg_csr_from_triplets
against the reference's own FromTriplets (oracle/_ref, sparse_matrix.cpp:25-69)."""
import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import CsrMatrix

pytestmark = pytest.mark.gpu


def _same(a: CsrMatrix, b: CsrMatrix):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_idx, b.col_idx)
    np.testing.assert_array_equal(a.values.view(np.uint64), b.values.view(np.uint64))


def _ref_or_restated(oracle_mod, rows, cols, r, c, v):
    """The reference's own FromTriplets (oracle/_ref), else the drop-in's host
    std::sort path (pinned to it in tests/test_oracle.py)."""
    ref = oracle_mod.reference()
    if ref is not None:
        return ref.from_triplets(rows, cols, r, c, v)
    import os
    os.environ["PDHG_DEVICE_ASSEMBLY"] = "0"
    try:
        return CsrMatrix.from_arrays(rows, cols, r, c, v)
    finally:
        del os.environ["PDHG_DEVICE_ASSEMBLY"]


def _triplets(seed, rows, cols, n, max_copies):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, rows, n)
    c = rng.integers(0, cols, n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)
    # exact cancellations: append negated copies of some entries
    k = rng.choice(n, n // 40, replace=False)
    r, c, v = np.concatenate([r, r[k]]), np.concatenate([c, c[k]]), np.concatenate([v, -v[k]])
    if max_copies is not None:  # keep the first `max_copies` triplets of every (row, col)
        key = r * cols + c
        order = np.argsort(key, kind="stable")
        ks = key[order]
        start = np.r_[0, np.flatnonzero(ks[1:] != ks[:-1]) + 1]
        rank = np.arange(ks.size) - np.repeat(start, np.diff(np.r_[start, ks.size]))
        keep = np.zeros(ks.size, bool)
        keep[order] = rank < max_copies
        r, c, v = r[keep], c[keep], v[keep]
    return r, c, v


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_device_assembly_matches_reference(seed, oracle_mod):
    """Device FromTriplets (stable radix sort, input-order sums) against the
    REFERENCE's FromTriplets (sparse_matrix.cpp:25-69), bit for bit, on
    inputs with duplicate pairs and exact cancellations."""
    rows, cols = 300, 200
    r, c, v = _triplets(seed, rows, cols, 20000, max_copies=2)
    _same(CsrMatrix.from_triplets_device(rows, cols, r, c, v), _ref_or_restated(oracle_mod, rows, cols, r, c, v))


def test_triple_duplicates_take_the_reference_order(oracle_mod):
    """An entry duplicated three or more times: its sum depends on the
    reference's std::sort order, so the device refuses it
    (PDHG_ORDER_DEPENDENT) and the drop-in FromTriplets -- here above the
    2^20-triplet device threshold -- assembles on the host, matching the
    reference bit for bit."""
    rows, cols = 3000, 700
    r, c, v = _triplets(7, rows, cols, (1 << 20) + 5000, max_copies=None)
    with pytest.raises(rpdlp.OrderDependent):
        CsrMatrix.from_triplets_device(rows, cols, r, c, v)
    _same(CsrMatrix.from_arrays(rows, cols, r, c, v), _ref_or_restated(oracle_mod, rows, cols, r, c, v))


def test_edge_cases():
    _same(CsrMatrix.from_triplets_device(4, 3, [], [], []), CsrMatrix.empty(4, 3))
    _same(CsrMatrix.from_triplets_device(0, 0, [], [], []), CsrMatrix.empty(0, 0))
    d = CsrMatrix.from_triplets_device(3, 3, [2, 0, 2], [1, 2, 1], [1.5, -2.0, -1.5])  # (2,1) cancels
    assert list(d.row_ptr) == [0, 1, 1, 1] and list(d.col_idx) == [2] and list(d.values) == [-2.0]
    for bad in (([3], [0]), ([0], [3]), ([-1], [0])):
        with pytest.raises(IndexError, match="triplet index out of range"):  # std::out_of_range
            CsrMatrix.from_triplets_device(3, 3, bad[0], bad[1], [1.0])


def test_generator_device_and_host_assembly_identical(monkeypatch, oracle_mod):
    """GenPagerank above the device threshold (2^20 triplets): the device
    assembly reproduces the host FromTriplets bit for bit, and both give the
    reference generator's matrix."""
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PDHG_DEVICE_ASSEMBLY", flag)
        out.append(rpdlp.GenPagerank(200_000, 0.85, 6, 3))
    a, b = out
    _same(a.g, b.g)
    _same(a.a, b.a)
    ref = oracle_mod.reference()
    if ref is not None:
        c = ref.gen_pagerank(200_000, 0.85, 6, 3)
        _same(b.g, c.g)
        _same(b.a, c.a)


def test_matrix_products_and_norms_match_serial_loops():
    """SparseMatrix products, inf-norms and power sums on the device
    (pdhg_csr_spmv / pdhg_csr_norms) against serial storage-order loops
    (sparse_matrix.cpp:114-204): bit-identical for segments <= 64."""
    p = rpdlp.GenRandomLp(60, 45, 0.25, 9)
    k = p.g
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal(k.cols), rng.standard_normal(k.rows)
    want, rinf, rp2 = np.zeros(k.rows), np.zeros(k.rows), np.zeros(k.rows)
    for r in range(k.rows):
        acc = 0.0
        for q in range(k.row_ptr[r], k.row_ptr[r + 1]):
            acc += k.values[q] * x[k.col_idx[q]]
            rinf[r] = max(rinf[r], abs(k.values[q]))
            rp2[r] += k.values[q] * k.values[q]
        want[r] = acc
    np.testing.assert_array_equal(k.multiply(x), want)
    np.testing.assert_array_equal(k.norms(), rinf)
    np.testing.assert_array_equal(k.norms(power=2.0), rp2)
    dense = k.to_dense()
    np.testing.assert_allclose(k.multiply(y, transpose=True), dense.T @ y, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(k.norms(columns=True), np.abs(dense).max(axis=0))

"""Kernel-level parity: device scaling, SpMV, power iteration, unit steps
against the oracle restatement (itself pinned to the reference), through the
C-ABI of libpdhg_b200.so."""
import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import (CsrMatrix, GenMcf, GenPagerank, GenRandomLp, GenStaircase, GenTransport,
                                         LpProblem, Session, SolverParams)

from problems import config1, empty_rows_lp, hand_dual_lp, hand_primal_lp, long_row_lp, mixed_bounds_lp, small_cases

pytestmark = pytest.mark.gpu


def uniform_columns_lp(L, n=3000, m=500, seed=4):
    """Every column holds exactly L nonzeros: the uniform-length class-S
    kernel (implicit offsets, vector loads) for L in {1, 2, 3, 4, 8}."""
    rng = np.random.default_rng(seed)
    trips = []
    for j in range(n):
        for i in rng.choice(m, size=L, replace=False):
            trips.append((int(i), j, float(rng.uniform(-1, 1)) or 0.5))
    g = CsrMatrix.from_triplets(m, n, trips)
    x = rng.uniform(0, 1, n)
    h = g.to_dense() @ x - 0.1
    return LpProblem(CsrMatrix.empty(0, n), g, rng.uniform(-1, 1, n), np.zeros(0), h, np.zeros(n), np.full(n, 2.0))


def kernel_cases():
    d = small_cases()
    d["config1"] = config1(2)
    d["long_row"] = long_row_lp()
    d["pagerank_3k"] = GenPagerank(3000, 0.85, 6, 2)
    d["transport_60x70"] = GenTransport(60, 70, 3)
    d["transport_600x40"] = GenTransport(600, 40, 2)  # 600-long demand rows: 4 rows per CTA
    d["mcf"] = GenMcf(80, 600, 6, 3)                    # columns of exactly 3
    d["staircase_d8"] = GenStaircase(5, 40, 60, 8, 2, seed=2)  # rows of exactly 8
    d["staircase_d20"] = GenStaircase(4, 50, 70, 20, 5, seed=3)  # warp-staged rows
    for L in (1, 4, 8):
        d[f"cols_len{L}"] = uniform_columns_lp(L)
    return d


CASES = kernel_cases()

# Class S bound (csrc/session.cu kThreadMax): every segment up to this length
# is summed by one thread in storage order, i.e. bit-identically with the
# reference's serial loops.
S_MAX = 64


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("scaled", [True, False])
def test_scaled_problem_bit_exact(name, scaled, restatement):
    """Ruiz x10 + Pock-Chambolle + ApplyScaling on device == reference, bit
    for bit, whenever no row/col of K exceeds S_MAX nonzeros (class S:
    storage-order sums);
    otherwise within 4 ulp-scale (PC power sums of long rows differ in order)."""
    p = CASES[name]
    prm = SolverParams()
    prm.scaling.enabled = scaled
    with Session(p, prm) as s:
        rs, cs = s.scaling()
        kv, c, l, u, q = s.scaled()
    rs0, cs0 = restatement.scaling(p, prm)
    kv0, c0, l0, u0, q0 = restatement.scaled(p, prm)
    if max_segment(p) <= S_MAX:
        for got, want in ((rs, rs0), (cs, cs0), (kv, kv0), (c, c0), (l, l0), (u, u0), (q, q0)):
            assert np.array_equal(got, want)
    else:
        for got, want in ((rs, rs0), (cs, cs0), (kv, kv0), (c, c0), (q, q0)):
            np.testing.assert_allclose(got, want, rtol=1e-15 * 8, atol=0)
        np.testing.assert_array_equal(np.isinf(l), np.isinf(l0))


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("transpose", [False, True])
def test_spmv_matches_reference_sums(name, transpose, restatement):
    """K_s x and K_s^T y: segments of <= S_MAX nonzeros are summed in storage
    order (bit-exact with sparse_matrix.cpp:114-138); longer ones with a fixed
    tree (1e-13 relative to sum |terms|)."""
    p = CASES[name]
    rng = np.random.default_rng(11)
    n, m = p.num_vars(), p.num_rows()
    vec = rng.standard_normal(m if transpose else n)
    # With segments > S_MAX the PC power sums (hence K_s) may differ in the
    # last ulp; check SpMV summation order on the unscaled K there.
    prm = SolverParams()
    prm.scaling.enabled = max_segment(p) <= S_MAX
    with Session(p, prm) as s:
        got = s.spmv(vec, transpose)
        kv = s.scaled()[0]
    want = restatement.spmv(p, vec, transpose, prm)
    rows = np.concatenate([np.repeat(np.arange(p.a.rows), np.diff(p.a.row_ptr)),
                           p.a.rows + np.repeat(np.arange(p.g.rows), np.diff(p.g.row_ptr))])
    cols = np.concatenate([p.a.col_idx, p.g.col_idx])
    if transpose:
        mag = np.bincount(cols, weights=np.abs(kv * vec[rows]), minlength=n)
        seglen = np.bincount(cols, minlength=n)
    else:
        mag = np.bincount(rows, weights=np.abs(kv * vec[cols]), minlength=m)
        seglen = np.bincount(rows, minlength=m)
    short = seglen <= S_MAX
    assert np.array_equal(got[short], want[short])
    assert np.all(np.abs(got - want) <= 1e-13 * mag + 1e-300)


def max_segment(p):
    cols = np.concatenate([p.a.col_idx, p.g.col_idx])
    lens = np.concatenate([np.diff(p.a.row_ptr), np.diff(p.g.row_ptr), np.bincount(cols, minlength=p.num_vars())])
    return int(lens.max(initial=0))


def test_spmv_deterministic_long_rows():
    p = long_row_lp()
    vec = np.random.default_rng(1).standard_normal(p.num_vars())
    with Session(p) as s:
        a = s.spmv(vec)
        b = s.spmv(vec)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["config1", "pagerank_3k", "transport_60x70", "long_row", "mixed"])
def test_opnorm(name, restatement):
    """EstimateOpNorm (solver.cpp:84-110), same libstdc++ start vector."""
    p = CASES[name]
    with Session(p) as s:
        got = s.opnorm(100, 0)
        got7 = s.opnorm(40, 7)
    want = restatement.opnorm(p, 100, 0)
    want7 = restatement.opnorm(p, 40, 7)
    assert got == pytest.approx(want, rel=1e-12)
    assert got7 == pytest.approx(want7, rel=1e-12)


def test_opnorm_known_matrices():
    """test_solver.cpp:41-57 (through the unscaled session)."""
    from paper_2312_14832_b200.rpdlp import CsrMatrix, LpProblem
    prm = SolverParams()
    prm.scaling.enabled = False

    def of(rows, cols, trips, iters, seed=1):
        g = CsrMatrix.from_triplets(rows, cols, trips)
        p = LpProblem(CsrMatrix.empty(0, cols), g, np.zeros(cols), [], np.zeros(rows), np.zeros(cols),
                      np.ones(cols))
        with Session(p, prm) as s:
            return s.opnorm(iters, seed)

    assert of(1, 1, [(0, 0, 3.0)], 50) == pytest.approx(3.0, rel=1e-12)
    est = of(3, 3, [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 5.0)], 200)
    assert 4.95 < est <= 5.0 + 1e-12
    assert of(2, 2, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 1.0)], 100) == pytest.approx(2.0, rel=1e-6)
    assert of(2, 3, [], 20) == 0.0


def test_primal_step_hand_example():
    """test_solver.cpp:65-88."""
    p = hand_primal_lp()
    assert rpdlp.PrimalStep(p, [0.2], [0.5], 0.5, 1.0)[0] == 0.0
    assert rpdlp.PrimalStep(p, [0.2], [0.5], 0.5, 2.0)[0] == pytest.approx(0.075, rel=1e-15)
    assert rpdlp.PrimalStep(p, [0.9], [5.0], 0.5, 1.0)[0] == 1.0


def test_dual_step_hand_example():
    """test_solver.cpp:90-112."""
    p = hand_dual_lp()
    y = rpdlp.DualStep(p, [1.0], [0.5], [0.1, 0.1], 0.5, 1.0)
    assert y[0] == pytest.approx(0.35, rel=1e-15) and y[1] == pytest.approx(0.35, rel=1e-15)
    y2 = rpdlp.DualStep(p, [3.0], [3.0], [0.1, 0.1], 0.5, 1.0)
    assert y2[0] == pytest.approx(-0.4, rel=1e-15) and y2[1] == 0.0


@pytest.mark.parametrize("name", ["mixed", "rand_40x30", "empty_rows", "pagerank_200"])
def test_unit_steps_vs_reference(name, restatement):
    p = CASES[name]
    rng = np.random.default_rng(5)
    n, m = p.num_vars(), p.num_rows()
    x, xo, y = rng.uniform(-1, 2, n), rng.uniform(-1, 2, n), rng.uniform(0, 1, m)
    np.testing.assert_allclose(rpdlp.PrimalStep(p, x, y, 0.3, 1.7), restatement.primal_step(p, x, y, 0.3, 1.7),
                               rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(rpdlp.DualStep(p, x, xo, y, 0.3, 1.7), restatement.dual_step(p, x, xo, y, 0.3, 1.7),
                               rtol=1e-14, atol=1e-15)


def test_scaling_api_matches_reference(restatement):
    """ComputeScaling / RuizEquilibrate / PockChambolleScale / ApplyScaling
    (scaling.hpp:49-59) through the device: the composed scales equal the
    restatement's bit for bit (segments <= 64), ApplyScaling equals the
    session's scaled problem; hand values of test_scaling.cpp:27-96."""
    p = config1(2)
    a, g = p.a, p.g  # K = [A; G] as one CSR
    K = rpdlp.CsrMatrix(a.rows + g.rows, p.num_vars(), np.concatenate([a.row_ptr[:-1], a.nnz + g.row_ptr]),
                        np.concatenate([a.col_idx, g.col_idx]), np.concatenate([a.values, g.values]))
    info = rpdlp.ComputeScaling(K)
    rs0, cs0 = restatement.scaling(p, SolverParams())
    np.testing.assert_array_equal(info.row_scale, rs0)
    np.testing.assert_array_equal(info.col_scale, cs0)
    ruiz = rpdlp.RuizEquilibrate(K, 10)
    pc = rpdlp.PockChambolleScale(K, 1.0)
    assert np.all(ruiz.row_scale > 0) and np.all(pc.col_scale > 0)
    sp = rpdlp.ApplyScaling(p, info)
    with Session(p) as s:
        kv, c, l, u, q = s.scaled()
    np.testing.assert_array_equal(np.concatenate([sp.a.values, sp.g.values]), kv)
    np.testing.assert_array_equal(sp.c, c)
    np.testing.assert_array_equal(np.concatenate([sp.b, sp.h]), q)
    one = rpdlp.CsrMatrix.from_triplets(1, 1, [(0, 0, 100.0)])
    assert rpdlp.RuizEquilibrate(one, 10).row_scale[0] == pytest.approx(0.1, rel=1e-15)
    pcs = rpdlp.PockChambolleScale(rpdlp.CsrMatrix.from_triplets(1, 2, [(0, 0, 4.0), (0, 1, 9.0)]), 1.0)
    assert pcs.row_scale[0] == pytest.approx(1 / np.sqrt(13.0), rel=1e-15)
    np.testing.assert_allclose(pcs.col_scale, [1 / 2.0, 1 / 3.0], rtol=1e-15)


@pytest.mark.parametrize("name", ["mixed", "config1", "transport_60x70", "pagerank_3k"])
def test_residuals_and_lambda_api(name, restatement):
    """ComputeResiduals / DeriveLambda (kkt.hpp:45-57) on the device against
    the reference: residuals of a CPU solution to 1e-12, lambda to 1e-12."""
    p = CASES[name]
    o = restatement.solve(p, SolverParams(eps=1e-6))
    r = rpdlp.ComputeResiduals(p, o.x, o.y)
    want = restatement.residuals(p, o.x, o.y)
    for k in ("primal_res", "dual_res", "gap_abs", "primal_obj", "dual_obj", "rel_primal", "rel_dual", "rel_gap"):
        assert getattr(r, k) == pytest.approx(getattr(want, k), rel=1e-12, abs=1e-12), k
    lam = rpdlp.DeriveLambda(p, o.y)
    np.testing.assert_allclose(lam, o.lambda_, rtol=1e-12, atol=1e-12)

"""CPU tests (no GPU): the oracle restatement pinned to the reference's golden
vectors and (where built) to the reference itself; the product's generators
pinned to the reference generators; the reference's own known-answer tests
for the host-side decision logic; the C-ABI library loading and exporting
every declared symbol."""
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2312_14832_b200 import abi, rpdlp
from paper_2312_14832_b200.rpdlp import GenPagerank, GenRandomLp, SolverParams

import problems

ROOT = Path(__file__).resolve().parents[1]
GOLD = np.load(ROOT / "tests" / "golden" / "golden.npz")
TRACE_FIELDS = ("iteration", "inner_iteration", "restarts", "omega", "eta", "kkt_candidate", "kkt_loop_start",
                "candidate_is_current", "restarted")


def digest(p) -> str:
    h = hashlib.sha256()
    for a in (p.a.row_ptr, p.a.col_idx, p.a.values, p.g.row_ptr, p.g.col_idx, p.g.values, p.c, p.b, p.h, p.l, p.u):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def golden_keys(prefix):
    return sorted(k for k in GOLD.files if k.startswith(prefix))


def solve_cases():
    d = dict(problems.small_cases())
    d["config1"] = problems.config1(1)
    d["ref_config1"] = problems.ref_config1(1)
    return d


CASES = solve_cases()


# ----------------------------------------------------------------- generators
@pytest.mark.parametrize("key", golden_keys("gen/random/"))
def test_random_generator_matches_reference(key):
    """GenRandomLp restated in csrc/instance_gen.cpp == instance_gen.cpp:143-188."""
    _, _, m, n, d, s = key.split("/")
    assert digest(GenRandomLp(int(m), int(n), float(d), int(s))) == str(GOLD[key])


@pytest.mark.parametrize("key", golden_keys("gen/pagerank/"))
def test_pagerank_generator_matches_reference(key):
    """GenPagerank restated == instance_gen.cpp:27-64, 90-141."""
    _, _, nn, dmp, att, s = key.split("/")
    assert digest(GenPagerank(int(nn), float(dmp), int(att), int(s))) == str(GOLD[key])


@pytest.mark.parametrize("name", sorted(CASES))
def test_instances_are_the_golden_ones(name):
    assert digest(CASES[name]) == str(GOLD[f"instance/{name}"])


# ------------------------------------------------- restatement vs golden vectors
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("eps", ["0.0001", "1e-08"])
def test_restatement_solve_bit_exact(name, eps, restatement):
    """The oracle restatement reproduces the reference solve bit for bit:
    status, iterations, restarts, report, x, y, lambda and the decision trace."""
    p = CASES[name]
    tr = []
    r = restatement.solve(p, SolverParams(eps=float(eps)), observer=tr.append)
    k = f"solve/{name}/{eps}"
    assert [int(r.status), r.iterations, r.restarts] == GOLD[k + "/meta"].tolist()
    rep = [getattr(r.report, f) for f in ("primal_res", "dual_res", "gap_abs", "primal_obj", "dual_obj",
                                          "rel_primal", "rel_dual", "rel_gap")]
    assert np.array_equal(np.array(rep), GOLD[k + "/report"])
    assert np.array_equal(r.x, GOLD[k + "/x"])
    assert np.array_equal(r.y, GOLD[k + "/y"])
    assert np.array_equal(r.lambda_, GOLD[k + "/lambda"])
    t = np.array([[float(getattr(e, f)) for f in TRACE_FIELDS] for e in tr]).reshape(-1, 9)
    assert np.array_equal(t, GOLD[k + "/trace"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_restatement_scaling_and_opnorm(name, restatement):
    p = CASES[name]
    rs, cs = restatement.scaling(p)
    assert np.array_equal(rs, GOLD[f"scaling/{name}/row"]) and np.array_equal(cs, GOLD[f"scaling/{name}/col"])
    got = [restatement.opnorm(p, 100, 0), restatement.opnorm(p, 40, 7)]
    assert got == GOLD[f"opnorm/{name}"].tolist()


def test_survey_decision_trace(restatement):
    """SURVEY §6 golden excerpt (reference GenRandomLp(1000,2000,.005,1), 1e-4)."""
    tr = []
    r = restatement.solve(GenRandomLp(1000, 2000, 0.005, 1), SolverParams(eps=1e-4), observer=tr.append)
    assert (int(r.status), r.iterations, r.restarts) == (0, 1088, 5)
    assert r.report.primal_obj == -380.16081970365025 and r.report.dual_obj == -380.17125406000321
    e = tr[0]
    assert (e.iteration, e.omega, e.eta, e.kkt_candidate, e.kkt_loop_start) == (
        64, 2.3959378656901058, 1.1089245806836978, 5.1042179725561301, 503.70198792768861)
    assert [x.iteration for x in tr if x.restarted] == [64, 128, 256, 448, 704]


# ----------------------------------------- restatement vs the reference build
def random_lps():
    rng = np.random.default_rng(20260826)
    out = []
    for t in range(12):
        m, n = int(rng.integers(2, 40)), int(rng.integers(2, 30))
        p = GenRandomLp(m, n, float(rng.uniform(0.1, 0.9)), int(rng.integers(1, 1 << 40)),
                        equality_rows=int(rng.integers(0, m)))
        if t % 3 == 0:
            p.l[0], p.u[0] = -np.inf, np.inf
        if t % 4 == 1:
            p.l[-1], p.u[-1] = -np.inf, 5.0
        out.append(p)
    return out


@pytest.mark.parametrize("i", range(12))
def test_restatement_vs_reference_random(i, restatement, reference):
    if reference is None:
        pytest.skip("reference build (oracle/_ref) not present")
    p = random_lps()[i]
    # Free / upper-only columns can make an instance unbounded: cap iterations.
    for prm in (SolverParams(eps=1e-6, iter_limit=4000), SolverParams(eps=1e-7, adaptive_step=True, iter_limit=4000),
                SolverParams(eps=1e-6, check_every=17, restart_enabled=(i % 2 == 0), iter_limit=4000)):
        a, b = restatement.solve(p, prm), reference.solve(p, prm)
        assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and np.array_equal(a.lambda_, b.lambda_)


def test_restatement_vs_reference_kernels(restatement, reference):
    if reference is None:
        pytest.skip("reference build (oracle/_ref) not present")
    rng = np.random.default_rng(3)
    for p in [problems.mixed_bounds_lp(), GenPagerank(500, 0.85, 3, 9), problems.empty_rows_lp()]:
        x, xo, y = rng.standard_normal(p.num_vars()), rng.standard_normal(p.num_vars()), rng.random(p.num_rows())
        assert np.array_equal(restatement.spmv(p, x), reference.spmv(p, x))
        assert np.array_equal(restatement.spmv(p, y, True), reference.spmv(p, y, True))
        assert np.array_equal(restatement.primal_step(p, x, y, .3, 1.7), reference.primal_step(p, x, y, .3, 1.7))
        assert np.array_equal(restatement.dual_step(p, x, xo, y, .3, 1.7),
                              reference.dual_step(p, x, xo, y, .3, 1.7))
        for a, b in zip(restatement.scaled(p), reference.scaled(p)):
            assert np.array_equal(a, b)
        ra, rb = restatement.residuals(p, x, y), reference.residuals(p, x, y)
        assert ra == rb


def test_restatement_limits_and_errors(restatement):
    p = GenRandomLp(5, 5, 0.6, 7)
    r = restatement.solve(p, SolverParams(eps=1e-16, iter_limit=10))
    assert r.status == rpdlp.SolveStatus.kIterLimit and r.iterations == 10
    t = restatement.solve(p, SolverParams(time_limit=0.0))
    assert t.status == rpdlp.SolveStatus.kTimeLimit and t.iterations == 0
    with pytest.raises(ValueError, match="eps must be positive"):
        restatement.solve(p, SolverParams(eps=0.0))
    q = problems.tiny_lp()
    q.l, q.u = np.array([2.0]), np.array([1.0])
    with pytest.raises(ValueError, match="crossed bounds"):
        restatement.solve(q)


def test_dense_residual_oracle(restatement):
    """Residuals vs a dense numpy re-derivation (test_kkt.cpp:82-101 style)."""
    rng = np.random.default_rng(31)
    for trial in range(5):
        p = GenRandomLp(5, 5, 0.7, 100 + trial, equality_rows=2)
        x, y = rng.uniform(-2, 2, 5), np.abs(rng.uniform(-2, 2, 5))
        r = restatement.residuals(p, x, y)
        A, G = p.a.to_dense(), p.g.to_dense()
        pr = np.sqrt(np.sum((A @ x - p.b) ** 2) + np.sum(np.maximum(p.h - G @ x, 0) ** 2))
        red = p.c - A.T @ y[:2] - G.T @ y[2:]
        lam = red.copy()  # boxed [0, 1]
        assert r.primal_res == pytest.approx(pr, rel=1e-12)
        assert r.dual_res == pytest.approx(np.linalg.norm(red - lam), abs=1e-12)
        dual = p.b @ y[:2] + p.h @ y[2:] + np.sum(np.where(lam > 0, p.l * lam, np.where(lam < 0, p.u * lam, 0)))
        assert r.dual_obj == pytest.approx(dual, rel=1e-12)
        assert r.primal_obj == pytest.approx(p.c @ x, rel=1e-12)


# ------------------------------------------- host decision logic of the product
def test_restart_truth_table():
    """test_solver.cpp:155-183 / acceptance C3 against the product's host code."""
    inf = float("inf")
    cases = [(1, 100, .10, 1., .05, True), (1, 100, .20, 1., .05, True), (1, 100, .50, 1., .40, True),
             (1, 100, .50, 1., .60, False), (1, 100, .79, 1., .79, False), (1, 100, .81, 1., .50, False),
             (36, 100, .90, 1., inf, True), (35, 100, .90, 1., inf, False), (1, 100, .80, 1., .70, True),
             (1, 100, .50, 1., inf, False), (35, 100, .15, 1., .01, True), (50, 100, 1.5, 1., .20, True)]
    for t, k, cand, start, prev, want in cases:
        assert rpdlp.ShouldRestart(SolverParams(), t, k, cand, start, prev) == want, (t, cand, prev)


def test_primal_weight_update():
    """test_solver.cpp:185-196."""
    assert rpdlp.UpdatePrimalWeight(1.0, 1.0, 4.0) == pytest.approx(2.0, rel=1e-15)
    assert rpdlp.UpdatePrimalWeight(3.0, 2.0, 2.0) == pytest.approx(np.sqrt(3.0), rel=1e-15)
    assert rpdlp.UpdatePrimalWeight(2.5, 0.0, 1.0) == 2.5
    assert rpdlp.UpdatePrimalWeight(2.5, 1.0, 1e-12) == 2.5


def test_kkt_error_hand_values():
    """test_kkt.cpp:127-173."""
    assert rpdlp.KktError(3.0, 4.0, 0.0, 1.0) == pytest.approx(5.0, rel=1e-15)
    assert rpdlp.KktError(3.0, 4.0, 0.0, 2.0) == pytest.approx(np.sqrt(40.0), rel=1e-15)
    assert rpdlp.KktError(0.0, 0.0, 0.0, 7.0) == 0.0
    rng = np.random.default_rng(77)
    for _ in range(100):
        pr, du, gap, w = rng.uniform(0, 50), rng.uniform(0, 50), rng.uniform(0, 50), rng.uniform(0.05, 20)
        ref = np.sqrt(w * w * pr * pr + du * du / (w * w) + gap * gap)
        assert rpdlp.KktError(pr, du, gap, w) == pytest.approx(ref, rel=1e-12)


def test_check_termination():
    """test_kkt.cpp:113-125."""
    r = rpdlp.ResidualReport()
    assert rpdlp.CheckTermination(r, 1e-12)
    r.rel_gap = 2e-4
    assert not rpdlp.CheckTermination(r, 1e-4)
    r.rel_primal = r.rel_dual = r.rel_gap = 9e-5
    assert rpdlp.CheckTermination(r, 1e-4) and rpdlp.CheckTermination(r, 1e-3)
    assert not rpdlp.CheckTermination(r, 1e-5)


def test_params_defaults_match_reference():
    """pdhg_params_default == SolverParams{} (solver.hpp:33-54)."""
    c = abi.default_params()
    py = SolverParams().to_c()
    for f, _ in abi.Params._fields_:
        assert getattr(c, f) == getattr(py, f), f


# ------------------------------------------------------------ library / ABI
def declared_symbols():
    text = (ROOT / "include" / "pdhg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdhg_[a-z0-9_]+)\s*\(", text)) - {"pdhg_eval_cb"})


def test_library_exports_every_declared_symbol():
    lib = abi.load()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(abi.SIGNATURES), set(syms) ^ set(abi.SIGNATURES)
    assert lib.pdhg_abi_version() == 1
    assert b"sm_100a" in lib.pdhg_build_info()


def test_library_is_sm100a_cubin():
    import subprocess
    so = ROOT / "paper_2312_14832_b200" / "libpdhg_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    import ctypes as C
    assert C.sizeof(abi.Params) == 104
    assert C.sizeof(abi.Report) == 64
    assert C.sizeof(abi.Csr) == 40
    assert C.sizeof(abi.EvalInfo) == 7 * 8 + 8 + 64 + 8


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = ROOT / "paper_2312_14832_b200"
    for f in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*")):
        txt = f.read_text(errors="replace")
        assert "oracle" not in txt.replace("ORACLE", "").lower() or f.name == "build.py", f


def test_gpu_entry_fails_loudly_without_device():
    """No CPU fallback: with no CUDA device the solve raises."""
    if abi.load().pdhg_device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(rpdlp.CudaError):
        rpdlp.Solve(problems.tiny_lp())


def test_from_triplets_semantics():
    """sparse_matrix.cpp:25-69 (duplicates summed, zeros dropped, sorted)."""
    m = rpdlp.CsrMatrix.from_triplets(2, 3, [(1, 2, 1.0), (0, 1, 2.0), (1, 2, -1.0), (0, 0, 3.0), (0, 1, 1.0)])
    assert m.row_ptr.tolist() == [0, 2, 2] and m.col_idx.tolist() == [0, 1] and m.values.tolist() == [3.0, 3.0]
    with pytest.raises(IndexError):
        rpdlp.CsrMatrix.from_triplets(1, 1, [(0, 1, 1.0)])


# ------------------------------------------- round-2 pins (residual view, transport, triplets)
@pytest.mark.parametrize("name", sorted(CASES))
def test_residuals_view_bit_identical(name, restatement, reference):
    """oracle_residuals_view (CSR-only, no host matrix copies; used for the
    1e9-nnz staircase) == the restated ResidualEvaluator and, where built,
    the reference's ComputeResiduals (kkt.cpp:143-145), bit for bit."""
    p = CASES[name]
    rng = np.random.default_rng(5)
    x, y = rng.uniform(-1, 2, p.num_vars()), rng.uniform(-1, 2, p.num_rows())
    a = restatement.residuals_view(p, x, y)
    b = restatement.residuals(p, x, y)
    assert a == b
    if reference is not None:
        assert a == reference.residuals(p, x, y)


def test_reference_side_transport_generator(reference):
    """oracle/ref_shim.cpp ref_gen_transport (built through the reference's
    FromTriplets, used by bench.py's reference arm) == the product's
    GenTransport, array for array."""
    if reference is None:
        pytest.skip("reference build absent")
    for (s, t, seed) in [(3, 4, 1), (12, 9, 5), (100, 80, 2)]:
        assert digest(reference.gen_transport(s, t, seed)) == digest(rpdlp.GenTransport(s, t, seed))


def test_fullscale_fixtures_are_reference_runs():
    """tests/golden/fullscale_*.json (make_fullscale.py, reference build):
    consistent shape, and config 2 is the reference's 13,056-iteration solve."""
    import json
    fx = json.loads((ROOT / "tests" / "golden" / "fullscale_transport.json").read_text())
    assert fx["status"] == 0 and fx["iterations"] == 13056 and fx["restarts"] == 13
    assert len(fx["restart_iterations"]) == 13 and fx["restart_iterations"][:3] == [64, 128, 256]
    # the terminating check returns before the observer (solver.cpp:405-412)
    assert len(fx["trace"]) == fx["iterations"] // 64 - 1
    assert fx["digest"] == digest(rpdlp.GenTransport(1000, 1000, 1))


def test_from_triplets_duplicate_order_matches_reference(reference):
    """Entries duplicated three or more times: FromTriplets sums them in the
    reference's std::sort order (sparse_matrix.cpp:35), which can differ
    from input order in the last bit; the drop-in (pdhg_from_triplets, host
    std::sort) reproduces the reference's values exactly."""
    if reference is None:
        pytest.skip("reference build absent")
    rng = np.random.default_rng(11)
    rows, cols = 7, 5
    trips = [(int(rng.integers(rows)), int(rng.integers(cols)),
              float(rng.uniform(-1, 1)) * 10.0 ** int(rng.integers(-8, 8))) for _ in range(400)]
    trips.sort(key=lambda t: t[0])  # row-grouped, input order inside a row: what ref_shim's FromCsr feeds
    m = rpdlp.CsrMatrix.from_triplets(rows, cols, trips)
    z = np.zeros(cols)
    raw = rpdlp.LpProblem(rpdlp.CsrMatrix.empty(0, cols), rpdlp.CsrMatrix(rows, cols, *_raw_csr(rows, trips)), z,
                          np.zeros(0), np.zeros(rows), z, z + 1)
    kv = reference.scaled(raw, SolverParams(scaling=rpdlp.ScalingConfig(enabled=False)))[0]
    assert np.array_equal(kv[:m.values.size], m.values)
    # and the input-order sum really differs for some entry (the case matters)
    naive = {}
    for r, c, v in trips:
        naive[(r, c)] = naive.get((r, c), 0.0) + v
    dense = m.to_dense()
    assert any(dense[r, c] != v for (r, c), v in naive.items())


def _raw_csr(rows, trips):
    """Triplets as an (unsorted, duplicate-carrying) CSR in input order per
    row: the reference's FromTriplets (via ref_shim FromCsr) re-sorts them."""
    per = [[] for _ in range(rows)]
    for r, c, v in trips:
        per[r].append((c, v))
    ptr = np.zeros(rows + 1, np.int64)
    idx, val = [], []
    for r in range(rows):
        ptr[r + 1] = ptr[r] + len(per[r])
        for c, v in per[r]:
            idx.append(c)
            val.append(v)
    return ptr, np.asarray(idx, np.int64), np.asarray(val, np.float64)

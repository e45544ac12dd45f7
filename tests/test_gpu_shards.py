"""The sharded solver on one GPU: K split into P balanced row
blocks (K x) and column blocks (K^T y) held by one session, exchanges in place.
Each shard owns whole rows / columns and sums them exactly as the unsharded
path does, so the matrix passes agree bit for bit; only the order of the
check reductions changes (per-shard partials, then a fixed shard order). The
solve must meet the same parity bar against the CPU oracle."""
import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import (GenMcf, GenPagerank, GenStaircase, GenTransport, Shards, SolveStatus,
                                         SolverParams)

from problems import config1, empty_rows_lp, long_row_lp, mixed_bounds_lp, small_cases

pytestmark = pytest.mark.gpu


def check(p, params, restatement, world, iter_tol=0.05):
    g = rpdlp.Solve(p, params, shards=Shards(world=world))
    o = restatement.solve(p, params)
    assert g.status == o.status
    assert abs(g.report.primal_obj - o.report.primal_obj) <= 1e-6 * (1.0 + abs(o.report.primal_obj))
    assert abs(g.report.dual_obj - o.report.dual_obj) <= 1e-6 * (1.0 + abs(o.report.dual_obj))
    assert abs(g.iterations - o.iterations) <= iter_tol * o.iterations
    if g.status == SolveStatus.kOptimal:
        r = restatement.residuals(p, g.x, g.y)
        assert max(r.rel_primal, r.rel_dual, r.rel_gap) <= params.eps
    return g, o


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("seed", [1, 2])
def test_config1_sharded(world, seed, restatement):
    check(config1(seed), SolverParams(eps=1e-4), restatement, world)


@pytest.mark.parametrize("world", [2, 4])
def test_config1_sharded_tight(world, restatement):
    check(config1(3), SolverParams(eps=1e-8), restatement, world)


@pytest.mark.parametrize("world", [2, 5])
def test_edge_cases_sharded(world, restatement):
    for p in (mixed_bounds_lp(), empty_rows_lp()):
        check(p, SolverParams(eps=1e-6), restatement, world)


def test_more_shards_than_rows(restatement):
    """Empty blocks: 8 shards over a 7-row, 6-column problem."""
    check(empty_rows_lp(), SolverParams(eps=1e-6), restatement, 8)


def test_long_rows_sharded(restatement):
    check(long_row_lp(), SolverParams(eps=1e-4, iter_limit=3000), restatement, 4)


def test_pagerank_sharded(restatement):
    g, _ = check(GenPagerank(3000, 0.85, 3, 2), SolverParams(eps=1e-6), restatement, 4)
    assert abs(g.x.sum() - 1.0) <= 1e-4


def test_transport_sharded(restatement):
    check(GenTransport(40, 60, 3), SolverParams(eps=1e-4), restatement, 3)


def test_mcf_sharded(restatement):
    check(GenMcf(60, 400, 5, 2), SolverParams(eps=1e-4), restatement, 4)


def test_staircase_sharded(restatement):
    check(GenStaircase(6, 40, 50, 8, 2, seed=4), SolverParams(eps=1e-4), restatement, 6)


@pytest.mark.parametrize("name", ["pagerank_200", "transport_12x9"])
def test_adaptive_sharded(name, restatement):
    """Per-iteration adaptive step: per-shard partials, shard sum, on-device
    eta update (only the shapes the reference's adaptive rule converges on;
    its trajectory is chaotic, see test_gpu_solve.py::test_adaptive_step)."""
    p = small_cases()[name]
    check(p, SolverParams(eps=1e-6, adaptive_step=True, iter_limit=20000), restatement, 3, iter_tol=0.5)


@pytest.mark.parametrize("world", [2, 4, 7])
def test_matrix_passes_match_unsharded(world):
    """Scaling factors, scaled data and both SpMV directions: the sharded
    session reproduces the single-shard one bit for bit on rows/columns the
    one-pass kernels handle (<= 16384 nonzeros), and to 1e-13 elsewhere."""
    p = long_row_lp(n=30000)
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(p.num_vars()), rng.standard_normal(p.num_rows())
    with rpdlp.Session(p) as s1, rpdlp.Session(p, shards=Shards(world=world)) as sp:
        r1, c1 = s1.scaling()
        rp, cp = sp.scaling()
        short_r = np.diff(np.concatenate([p.a.row_ptr[:-1], p.a.nnz + p.g.row_ptr])) <= 16384
        np.testing.assert_array_equal(rp[short_r], r1[short_r])
        np.testing.assert_allclose(rp, r1, rtol=1e-13)
        np.testing.assert_array_equal(cp, c1)
        for a, b in zip(s1.scaled(), sp.scaled()):
            np.testing.assert_allclose(b, a, rtol=1e-13)
        kx1, kxp = s1.spmv(x), sp.spmv(x)
        np.testing.assert_array_equal(kxp[short_r], kx1[short_r])
        np.testing.assert_allclose(kxp, kx1, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(sp.spmv(y, transpose=True), s1.spmv(y, transpose=True))
        assert sp.opnorm(50) == pytest.approx(s1.opnorm(50), rel=1e-12)
        rb, cb = sp.blocks()
        assert rb[0] == 0 and rb[-1] == p.num_rows() and cb[0] == 0 and cb[-1] == p.num_vars()
        assert np.all(np.diff(rb) >= 0) and np.all(np.diff(cb) >= 0)
        st = sp.stats()
        assert st.world == world and st.local_shards == world


def test_session_resolve_sharded(restatement):
    """Resident sharded session: repeated solves are bitwise identical."""
    p = config1(2)
    with rpdlp.Session(p, shards=Shards(world=3)) as s:
        a = s.solve(SolverParams(eps=1e-6))
        b = s.solve(SolverParams(eps=1e-6))
    assert a.iterations == b.iterations
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)


def test_sharded_limits():
    p = config1(1)
    r = rpdlp.Solve(p, SolverParams(eps=1e-10, iter_limit=100), shards=Shards(world=3))
    assert r.status == SolveStatus.kIterLimit and r.iterations == 100
    r = rpdlp.Solve(p, SolverParams(eps=1e-10, time_limit=0.0), shards=Shards(world=3))
    assert r.status == SolveStatus.kTimeLimit and r.iterations == 0


@pytest.mark.parametrize("gen", ["staircase", "pagerank", "transport"])
def test_ghost_plan_counts(gen):
    """The ghost plan (entries each block reads from every other block) equals
    a numpy count from the original matrix and the balanced blocks."""
    p = {"staircase": lambda: GenStaircase(8, 60, 70, 6, 2, seed=3),
         "pagerank": lambda: GenPagerank(2000, 0.85, 3, 2),
         "transport": lambda: GenTransport(20, 30, 1)}[gen]()
    world = 4
    K = np.vstack([p.a.to_dense(), p.g.to_dense()]) != 0
    with rpdlp.Session(p, shards=Shards(world=world)) as s:
        rb, cb = s.blocks()
        xc, yc, use = s.ghost_counts()
    assert use == (False, False)  # one process: exchanges are in place
    for r in range(world):
        for b in range(world):
            rows, cols = slice(rb[r], rb[r + 1]), slice(cb[b], cb[b + 1])
            want_x = 0 if r == b else int(K[rows, cols].any(axis=0).sum())
            crow, ccol = slice(cb[r], cb[r + 1]), slice(rb[b], rb[b + 1])
            want_y = 0 if r == b else int(K[ccol, crow].any(axis=1).sum())
            assert xc[r, b] == want_x, (r, b)
            assert yc[r, b] == want_y, (r, b)
    if gen == "staircase":  # a stage block reads only its neighbour's boundary
        assert xc.sum() < 0.5 * (world - 1) * K.shape[1]


def test_nccl_path_single_rank(restatement):
    """The one-shard-per-process NCCL path on one GPU (world = 1): in-place
    all-gathers, the check all-reduce, rank 0's clock in the pack and the
    observer-abort all-reduce, all captured in the block graphs -- same
    trajectory as the default session."""
    p = config1(1)
    prm = SolverParams(eps=1e-6)
    tr_a, tr_b = [], []
    a = rpdlp.Solve(p, prm, observer=tr_a.append)
    b = rpdlp.Solve(p, prm, observer=tr_b.append, shards=Shards.nccl_single())
    assert a.status == b.status and a.iterations == b.iterations and a.restarts == b.restarts
    np.testing.assert_array_equal(a.x, b.x)
    assert [(e.iteration, e.restarted) for e in tr_a] == [(e.iteration, e.restarted) for e in tr_b]
    r = rpdlp.Solve(p, SolverParams(eps=1e-10, iter_limit=200), shards=Shards.nccl_single())
    assert r.iterations == 200
    with pytest.raises(RuntimeError):
        def stop(_):
            raise RuntimeError("stop")
        rpdlp.Solve(p, prm, observer=stop, shards=Shards.nccl_single())

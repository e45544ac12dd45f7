"""The reference's end-to-end acceptance criteria (proj/tests/acceptance.cpp)
run through the B200 solve path. C3 (restart truth table), C4 (KKT formula)
and C6 (SGM closed form) are host logic and live in test_oracle.py /
test_suite_cli.py; C9 (byte-identical redacted bench reports) in
test_suite_cli.py. The vertex-enumeration oracle of C1 is replaced by an
exact LP solve (scipy HiGHS) -- test infrastructure only."""
import math
import time

import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp, suite
from paper_2312_14832_b200.rpdlp import GenPagerank, GenRandomLp, SolverParams, SolveStatus

pytestmark = pytest.mark.gpu


def _mt19937_64(seed):
    """std::mt19937_64 (the C++ standard's parameters): the seed stream of
    acceptance.cpp:67."""
    n, m, a = 312, 156, 0xB5026F5AA96619E9
    up, lo, mask = 0xFFFFFFFF80000000, 0x7FFFFFFF, (1 << 64) - 1
    mt = [seed & mask]
    for i in range(1, n):
        mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & mask)
    idx = n
    while True:
        if idx >= n:
            for i in range(n):
                y = (mt[i] & up) | (mt[(i + 1) % n] & lo)
                mt[i] = mt[(i + m) % n] ^ (y >> 1) ^ (a if y & 1 else 0)
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & mask
        y ^= (y << 37) & 0xFFF7EEE000000000 & mask
        y ^= y >> 43
        yield y & mask


def _exact_optimum(p):
    from scipy.optimize import linprog
    g = p.g.to_dense()
    a = p.a.to_dense() if p.a.rows else None
    res = linprog(p.c, A_ub=-g if p.g.rows else None, b_ub=-p.h if p.g.rows else None,
                  A_eq=a, b_eq=p.b if p.a.rows else None, bounds=list(zip(p.l, p.u)), method="highs")
    assert res.status == 0
    return res.fun + p.objective_offset


def test_c1_c2_random_lps_match_exact_optimum(restatement):
    """C1: 50 seeded random LPs at eps 1e-8 reach the exact optimum to 1e-6
    relative within 60 s; C2: every Optimal result has all three relative
    residuals (recomputed on the host, kkt.cpp) below eps."""
    seeds = _mt19937_64(20260826)
    t0 = time.perf_counter()
    solved = []
    for _ in range(50):
        s = next(seeds)
        m, n = 2 + s % 7, 2 + (s >> 8) % 5
        p = GenRandomLp(m, n, 0.7, s)
        r = rpdlp.Solve(p, SolverParams(eps=1e-8))
        assert r.status == SolveStatus.kOptimal, p.name
        best = _exact_optimum(p)
        assert abs(r.report.primal_obj - best) / (1.0 + abs(best)) <= 1e-6, p.name
        solved.append((p, r))
    assert time.perf_counter() - t0 < 60.0
    for p, r in solved:
        rep = restatement.residuals(p, r.x, r.y)
        assert rep.rel_primal <= 1e-8 and rep.rel_dual <= 1e-8 and rep.rel_gap <= 1e-8, p.name


def test_c5_pagerank_shapes_and_solutions():
    """C5: n + 1 rows; Optimal at eps 1e-6 within 120 s at n = 10000;
    sum(x) within 1e-4 of 1, x >= 0."""
    for n in (100, 1000, 10000):
        p = GenPagerank(n, 0.85, 3, 2026)
        assert p.num_rows() == n + 1 and p.num_vars() == n
        t0 = time.perf_counter()
        r = rpdlp.Solve(p, SolverParams(eps=1e-6, time_limit=120.0))
        assert r.status == SolveStatus.kOptimal
        assert time.perf_counter() - t0 <= 120.0
        assert abs(r.x.sum() - 1.0) <= 1e-4 and r.x.min() >= 0.0


def test_c7_sgm_tolerance_ordering(tmp_path):
    """C7: on a 10-instance suite SGM10 at 1e-8 is at least SGM10 at 1e-4."""
    for i in range(5):
        rpdlp.WriteMpsFile(GenPagerank(400 + 100 * i, 0.85, 3, 50 + i), tmp_path / f"pagerank_{i}.mps")
        rpdlp.WriteMpsFile(GenRandomLp(40, 30, 0.3, 60 + i), tmp_path / f"random_{i}.mps")
    loose = suite.RunSuite(str(tmp_path), SolverParams(eps=1e-4))
    tight = suite.RunSuite(str(tmp_path), SolverParams(eps=1e-8))
    assert len(loose.records) == len(tight.records) == 10
    assert tight.sgm10 >= loose.sgm10


def test_c8_restart_benefit():
    """C8: across 10 PageRank seeds at n = 2000 the median iteration count
    with restarts is at most 0.8x the median without."""
    with_r, without = [], []
    for seed in range(1, 11):
        p = GenPagerank(2000, 0.85, 3, seed)
        r = rpdlp.Solve(p, SolverParams(eps=1e-6, time_limit=120.0))
        assert r.status == SolveStatus.kOptimal
        with_r.append(r.iterations)
        q = rpdlp.Solve(p, SolverParams(eps=1e-6, time_limit=120.0, restart_enabled=False))
        assert q.status == SolveStatus.kOptimal
        without.append(q.iterations)
    med = lambda v: float(np.median(v))  # noqa: E731
    assert med(with_r) <= 0.8 * med(without), (med(with_r), med(without))
    assert math.isfinite(med(without))

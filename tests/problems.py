"""Problem factories shared by the tests (mirrors the reference test fixtures)."""
from __future__ import annotations

import numpy as np

from paper_2312_14832_b200.rpdlp import CsrMatrix, LpProblem, GenPagerank, GenRandomLp, GenTransport

INF = float("inf")


def lp(a, g, c, b, h, l, u, n=None, offset=0.0) -> LpProblem:
    n = len(c) if n is None else n
    return LpProblem(a, g, np.asarray(c, float), np.asarray(b, float), np.asarray(h, float), np.asarray(l, float),
                     np.asarray(u, float), offset)


def tiny_lp() -> LpProblem:
    """min x s.t. x >= 1, x >= 0; optimum (1, 1) (test_solver.cpp:29-39)."""
    return lp(CsrMatrix.empty(0, 1), CsrMatrix.from_triplets(1, 1, [(0, 0, 1.0)]), [1.0], [], [1.0], [0.0], [INF])


def hand_primal_lp() -> LpProblem:
    """test_solver.cpp:65-75."""
    return lp(CsrMatrix.empty(0, 1), CsrMatrix.from_triplets(1, 1, [(0, 0, 1.0)]), [1.0], [], [0.0], [0.0], [1.0])


def hand_dual_lp() -> LpProblem:
    """test_solver.cpp:90-99."""
    return lp(CsrMatrix.from_triplets(1, 1, [(0, 0, 1.0)]), CsrMatrix.from_triplets(1, 1, [(0, 0, 1.0)]), [0.0],
              [2.0], [2.0], [0.0], [INF])


def mixed_bounds_lp(seed=7) -> LpProblem:
    """Random LP with all four bound classes, equality rows and an objective
    offset (exercises every branch of the residual/lambda code)."""
    p = GenRandomLp(30, 40, 0.2, seed, equality_rows=8)
    p.l[0], p.u[0] = -INF, INF
    p.l[1], p.u[1] = -INF, 2.0
    p.l[2], p.u[2] = 0.0, INF
    p.l[3], p.u[3] = -1.0, 3.0
    p.objective_offset = 1.5
    return p


def empty_rows_lp() -> LpProblem:
    """Empty rows and columns in K (zero-length segments in both layouts)."""
    g = CsrMatrix.from_triplets(5, 6, [(0, 0, 1.0), (0, 2, -1.0), (2, 1, 2.0), (2, 2, 1.0), (4, 0, 1.0), (4, 1, 1.0)])
    a = CsrMatrix.from_triplets(2, 6, [(1, 0, 1.0), (1, 1, 1.0), (1, 2, 1.0)])
    return lp(a, g, [1.0, 2.0, 0.5, 0.0, 0.0, 1.0], [0.0, 1.0], [-1.0, -5.0, 0.5, -2.0, 0.2], [0.0] * 6,
              [4.0, 4.0, 4.0, 1.0, INF, 2.0])


def long_row_lp(n=20000, seed=3) -> LpProblem:
    """One dense equality row of length n (spans ~10 tiles), plus a
    power-law set of long G rows and short rows: the PageRank shape in small."""
    rng = np.random.default_rng(seed)
    trips = [(0, j, 1.0) for j in range(n)]
    a = CsrMatrix.from_triplets(1, n, trips)
    g_tr = []
    rows = 300
    for i in range(rows):
        ln = int(min(n, 1 + rng.pareto(1.1) * 3)) if i % 50 else 2500 + 37 * i
        cols = rng.choice(n, size=min(ln, n), replace=False)
        for j in cols:
            g_tr.append((i, int(j), float(rng.uniform(-1, 1))))
    g = CsrMatrix.from_triplets(rows, n, g_tr)
    x_hat = rng.uniform(0, 1, n)
    x_hat /= x_hat.sum()
    dense_h = np.array([sum(v * x_hat[c] for (r, c, v) in []) for _ in range(0)])
    gx = np.zeros(rows)
    for r in range(rows):
        for k in range(g.row_ptr[r], g.row_ptr[r + 1]):
            gx[r] += g.values[k] * x_hat[g.col_idx[k]]
    h = gx - 0.1 * rng.uniform(0, 1, rows)
    c = rng.uniform(-1, 1, n)
    del dense_h
    return lp(a, g, c, [1.0], h, np.zeros(n), np.full(n, INF))


def config1(seed=1) -> LpProblem:
    """GenRandomLp(1000, 2000, 0.005, s), first 300 rows
    moved into A with b = A x_hat."""
    return GenRandomLp(1000, 2000, 0.005, seed, equality_rows=300)


def ref_config1(seed=1) -> LpProblem:
    """The reference's own GenRandomLp(1000, 2000, 0.005, s) (all >= rows)."""
    return GenRandomLp(1000, 2000, 0.005, seed)


def small_cases():
    return {
        "tiny": tiny_lp(),
        "mixed": mixed_bounds_lp(),
        "empty_rows": empty_rows_lp(),
        "rand_6x8": GenRandomLp(6, 8, 0.5, 55),
        "rand_40x30": GenRandomLp(40, 30, 0.3, 60),
        "pagerank_200": GenPagerank(200, 0.85, 3, 4),
        "transport_12x9": GenTransport(12, 9, 5),
    }

"""Randomised parity sweep: feasible LPs whose row and column lengths span
every length class (thread / warp / CTA / tile engine), with equality and
inequality rows, all four bound classes and an objective offset, solved on
the B200 path and by the CPU oracle (restatement pinned to the reference).
The north_star bar per instance: same status, objectives within 1e-6
relative, host-recomputed residuals below eps, iterations within 5 %."""
import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import CsrMatrix, LpProblem, SolverParams, SolveStatus

pytestmark = pytest.mark.gpu

INF = float("inf")


def _random_lp(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    m = int(rng.integers(20, 400))
    # heavy-tailed row lengths: most short, a few across the class bounds
    lens = np.minimum(n, np.maximum(1, (rng.pareto(1.2, m) * 4).astype(int)))
    lens[rng.integers(0, m)] = min(n, int(rng.choice([40, 80, 700, 2000, 2900])))
    rows, cols = [], []
    for r, k in enumerate(lens):
        rows += [r] * int(k)
        cols += list(rng.choice(n, int(k), replace=False))
    vals = rng.uniform(-1, 1, len(rows))
    x_hat = rng.uniform(0, 1, n)
    k_all = CsrMatrix.from_triplets(m, n, zip(rows, cols, vals))
    kx = k_all.to_dense() @ x_hat
    m1 = int(rng.integers(0, m // 3 + 1))
    dense = k_all.to_dense()

    def block(lo, hi):
        r, c = np.nonzero(dense[lo:hi])
        return CsrMatrix.from_triplets(hi - lo, n, zip(r, c, dense[lo:hi][r, c]))

    a, g = block(0, m1), block(m1, m)
    b = kx[:m1]
    h = kx[m1:] - np.abs(rng.uniform(0, 0.3, m - m1))
    c = rng.uniform(-1, 1, n)
    l, u = np.zeros(n), np.ones(n)
    kinds = rng.integers(0, 4, n)  # free / upper-only / lower-only / boxed around x_hat
    l[kinds == 0], u[kinds == 0] = -INF, INF
    l[kinds == 1], u[kinds == 1] = -INF, 2.0
    l[kinds == 2], u[kinds == 2] = -0.5, INF
    c[kinds == 0] = 0.0  # keep free variables from making the LP unbounded
    c[kinds == 1] = -np.abs(c[kinds == 1])
    c[kinds == 2] = np.abs(c[kinds == 2])
    return LpProblem(a, g, c, b, h, l, u, float(rng.uniform(-5, 5)))


@pytest.mark.parametrize("seed", range(12))
def test_random_class_mix_parity(seed, restatement):
    p = _random_lp(1000 + seed)
    prm = SolverParams(eps=1e-6, iter_limit=60000)
    g = rpdlp.Solve(p, prm)
    o = restatement.solve(p, prm)
    assert g.status == o.status
    if o.status != SolveStatus.kOptimal:
        return  # identical limit status is the bar there
    rel = abs(g.report.primal_obj - o.report.primal_obj) / (1.0 + abs(o.report.primal_obj))
    assert rel <= 1e-6
    r = restatement.residuals(p, g.x, g.y)
    assert r.rel_primal <= prm.eps and r.rel_dual <= prm.eps and r.rel_gap <= prm.eps
    assert abs(g.iterations - o.iterations) <= 0.05 * o.iterations

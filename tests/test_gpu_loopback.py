"""The multi-rank (one shard per process) code path with world 2..8 on ONE GPU.

Every rank is a one-shard Session in this process on its own host thread,
created with a loopback id (rpdlp.Shards.loopback, csrc/comm.cuh
LoopbackComm): the session runs exactly its NCCL-mode path -- padded slices,
ghost-only exchanges (pack, per-peer send/recv segments, unpack), per-rank
check packs summed over ranks, rank 0's clock in the pack, the
observer-abort reduction -- with device copies and event barriers in place
of NCCL's transport.

Device ordering between the ranks' streams uses CUDA events exchanged
through the host rendezvous (no spinning kernels), so the ranks' sessions run
their blocks eagerly instead of as CUDA graphs (Comm::graphs); the kernels
are the same.

Parity bar: every rank returns the same result, and it is bit-identical to
the in-process shard mode (all shards in one session), which the
CPU-oracle parity tests of test_gpu_shards.py pin. Only NCCL's own data
movement is not exercised here (one GPU per call in this environment).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp
from paper_2312_14832_b200.rpdlp import GenMcf, GenPagerank, GenStaircase, GenTransport, Shards, SolverParams

from problems import config1, empty_rows_lp, mixed_bounds_lp

pytestmark = pytest.mark.gpu


def run_ranks(p, params, world, observers=None, ghost=False):
    """Construct and solve one session per rank concurrently; returns the
    per-rank results (or exceptions) and, with ghost=True, the ghost use flags."""
    specs = Shards.loopback(world)
    out = [None] * world
    use = [None] * world

    def rank(r):
        try:
            with rpdlp.Session(p, params, shards=specs[r]) as s:
                if ghost:
                    use[r] = s.ghost_counts()[2]
                out[r] = s.solve(params, (observers or {}).get(r))
        except BaseException as e:  # noqa: BLE001 - reported per rank
            out[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a loopback rank hung"
    return out, use


def same(a, b):
    assert a.status == b.status
    assert a.iterations == b.iterations and a.restarts == b.restarts
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and np.array_equal(a.lambda_, b.lambda_)
    assert a.report.primal_obj == b.report.primal_obj and a.report.dual_obj == b.report.dual_obj


CASES = {
    "config1": lambda: config1(2),
    "transport": lambda: GenTransport(40, 60, 3),
    "pagerank": lambda: GenPagerank(3000, 0.85, 3, 2),
    "mcf": lambda: GenMcf(60, 400, 5, 2),
    "staircase": lambda: GenStaircase(6, 40, 50, 8, 2, seed=4),
    "mixed_bounds": mixed_bounds_lp,
    "empty_rows": empty_rows_lp,
}


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_loopback_ranks_match_shard_mode(name, world):
    p = CASES[name]()
    params = SolverParams(eps=1e-5, iter_limit=20000)
    ref = rpdlp.Solve(p, params, shards=Shards(world=world))
    res, _ = run_ranks(p, params, world)
    errs = [(r, repr(g)) for r, g in enumerate(res) if isinstance(g, BaseException)]
    assert not errs, errs
    for g in res:
        same(g, ref)


def test_loopback_eight_ranks_ghost_exchange():
    """World 8 on the staircase: the ghost-only exchange (only boundary
    stages cross ranks) is chosen and reproduces the shard mode bit for bit."""
    p = GenStaircase(16, 60, 60, 8, 2, seed=5)
    params = SolverParams(eps=1e-6, iter_limit=20000)
    ref = rpdlp.Solve(p, params, shards=Shards(world=8))
    res, use = run_ranks(p, params, 8, ghost=True)
    errs = [repr(g) for g in res if isinstance(g, BaseException)]
    assert not errs, errs
    assert all(u is not None and u[0] and u[1] for u in use), use
    for g in res:
        same(g, ref)


def test_loopback_observer_on_rank0_only_aborts_every_rank():
    """only rank 0 has an observer (as under torchrun); its abort
    at the third check stops every rank -- the abort reduction stays paired."""
    p = config1(1)
    params = SolverParams(eps=1e-10, iter_limit=100000)
    seen = []

    class Stop(Exception):
        pass

    def obs(info):
        seen.append(info.iteration)
        if len(seen) == 3:
            raise Stop()

    res, _ = run_ranks(p, params, 3, observers={0: obs})
    assert isinstance(res[0], Stop)
    for g in res[1:]:
        assert isinstance(g, BaseException) and "aborted" in str(g), g
    assert len(seen) == 3


def test_loopback_limits_and_restarts_match():
    """Iteration limit in the middle of a block, and a time limit decided by
    rank 0's clock: every rank stops after the same iteration."""
    p = GenTransport(30, 50, 2)
    params = SolverParams(eps=1e-9, iter_limit=1000)
    ref = rpdlp.Solve(p, params, shards=Shards(world=3))
    res, _ = run_ranks(p, params, 3)
    for g in res:
        same(g, ref)
    assert ref.status == rpdlp.SolveStatus.kIterLimit and ref.iterations == 1000
    res, _ = run_ranks(p, SolverParams(eps=1e-12, time_limit=0.2), 3)
    its = {g.iterations for g in res}
    assert len(its) == 1 and all(g.status == rpdlp.SolveStatus.kTimeLimit for g in res), res

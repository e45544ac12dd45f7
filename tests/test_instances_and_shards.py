"""CPU tests of the new instance builders and of
the host side of the sharded solver: the balanced block split
every rank computes, and -- with a world_size-2 gloo process group -- the
exchange pattern of a row/column-sharded PDHG iteration (slice updates,
all-gather of x+ and y+, all-reduce of the check sums) against the unsharded
iteration."""
import os
import socket

import numpy as np
import pytest

from paper_2312_14832_b200 import rpdlp  # noqa: E402
from paper_2312_14832_b200.rpdlp import GenMcf, GenStaircase, PartitionBlocks, SolverParams, SolveStatus


def dense(m):
    return m.to_dense()


# ----------------------------------------------------------- generators
def test_mcf_shape_and_feasibility():
    V, E, K = 80, 500, 6
    p = GenMcf(V, E, K, 3)
    assert p.num_vars() == E * K and p.num_eq_rows() == V * K and p.num_ineq_rows() == E
    assert p.nnz() == 3 * E * K
    rl = np.diff(p.a.row_ptr)
    assert rl.max() > 5 * max(rl.mean(), 1)  # heavy-tailed conservation rows
    assert np.all(np.diff(p.g.row_ptr) == K)
    # every column appears exactly 3 times (tail +1, head -1, capacity -1)
    cnt = np.bincount(np.concatenate([p.a.col_idx, p.g.col_idx]), minlength=p.num_vars())
    assert np.all(cnt == 3)
    w = p.witness
    assert np.allclose(dense(p.a) @ w, p.b, atol=1e-12)
    assert np.all(dense(p.g) @ w >= p.h)
    assert np.all(w >= 0)
    for m in (p.a, p.g):  # strictly increasing columns per row
        for r in range(m.rows):
            seg = m.col_idx[m.row_ptr[r]:m.row_ptr[r + 1]]
            assert np.all(np.diff(seg) > 0)


def test_mcf_deterministic():
    a, b = GenMcf(50, 300, 4, 9), GenMcf(50, 300, 4, 9)
    for k in ("row_ptr", "col_idx", "values"):
        np.testing.assert_array_equal(getattr(a.a, k), getattr(b.a, k))
    np.testing.assert_array_equal(a.c, b.c)
    np.testing.assert_array_equal(a.h, b.h)
    assert not np.array_equal(a.c, GenMcf(50, 300, 4, 10).c)


def test_staircase_shape_and_feasibility():
    T, R, C, D, Dl = 5, 30, 40, 7, 2
    p = GenStaircase(T, R, C, D, Dl, seed=2)
    assert p.num_rows() == T * R and p.num_vars() == T * C and p.nnz() == T * R * D
    assert p.num_eq_rows() == T * (R // 2)
    w = p.witness
    assert np.allclose(dense(p.a) @ w, p.b, atol=1e-12)
    assert np.all(dense(p.g) @ w >= p.h)
    assert np.all((p.l <= w) & (w <= p.u))
    # staircase structure: a row of stage t touches stages t-1 and t only
    for m, per in ((p.a, R // 2), (p.g, R - R // 2)):
        for r in range(m.rows):
            t = r // per
            cols = m.col_idx[m.row_ptr[r]:m.row_ptr[r + 1]]
            assert np.all(np.diff(cols) > 0)
            assert cols.min() >= max(t - 1, 0) * C and cols.max() < (t + 1) * C
            if t > 0:
                assert np.sum(cols < t * C) == Dl


def test_staircase_thread_count_invariant():
    a = GenStaircase(9, 20, 25, 6, 2, seed=5, threads=1)
    b = GenStaircase(9, 20, 25, 6, 2, seed=5, threads=4)
    for x, y in ((a.a, b.a), (a.g, b.g)):
        for k in ("row_ptr", "col_idx", "values"):
            np.testing.assert_array_equal(getattr(x, k), getattr(y, k))
    for k in ("c", "b", "h", "l", "u", "witness"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))


def test_generator_argument_errors():
    with pytest.raises(ValueError):
        GenMcf(1, 10, 2, 1)
    with pytest.raises(ValueError):
        GenStaircase(2, 10, 5, 8, 1)  # D - Dl > C


@pytest.mark.parametrize("gen", ["mcf", "staircase"])
def test_new_instances_solve_on_reference(gen, reference):
    p = GenMcf(40, 200, 3, 1) if gen == "mcf" else GenStaircase(4, 20, 25, 6, 2, seed=1)
    r = reference.solve(p, SolverParams(eps=1e-6))
    assert r.status == SolveStatus.kOptimal
    assert max(r.report.rel_primal, r.report.rel_dual, r.report.rel_gap) <= 1e-6


def test_instance_views_are_zero_copy_and_owned():
    """Generated arrays are views into the C++ instance, which lives as long
    as any of them does."""
    p = GenStaircase(3, 10, 12, 4, 1, seed=1)
    vals = p.a.values
    ref = vals.copy()
    del p
    import gc
    gc.collect()
    np.testing.assert_array_equal(vals, ref)


# ------------------------------------------------------------ partition
def block_weights(ptr, begin, w):
    return [(ptr[begin[b + 1]] - ptr[begin[b]]) + w * (begin[b + 1] - begin[b]) for b in range(len(begin) - 1)]


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 64])
def test_partition_blocks_balanced(parts):
    rng = np.random.default_rng(parts)
    lens = rng.zipf(1.8, size=5000).clip(max=20000)
    ptr = np.concatenate([[0], np.cumsum(lens)])
    b = PartitionBlocks(ptr, parts, 6)
    assert b[0] == 0 and b[-1] == len(lens) and np.all(np.diff(b) >= 0) and len(b) == parts + 1
    wts = block_weights(ptr, b, 6)
    total = ptr[-1] + 6 * len(lens)
    assert sum(wts) == total
    assert max(wts) <= total / parts + lens.max() + 6


def test_partition_blocks_degenerate():
    ptr = np.array([0, 0, 0, 10])  # one heavy segment, empty ones
    b = PartitionBlocks(ptr, 4, 0)
    assert b[0] == 0 and b[-1] == 3 and np.all(np.diff(b) >= 0)
    assert list(PartitionBlocks(np.array([0]), 3, 6)) == [0, 0, 0, 0]


# ------------------------------------------- gloo world_size-2 exchange test
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pdhg_iters(K, q, c, l, u, eq, eta, omega, iters, shard=None):
    """Unscaled PDHG iterations (solver.cpp:284-306) with K x and K^T y either
    whole or split by the blocks of `shard` = (dist, rank, row_begin, col_begin),
    exchanging x+ / y+ slices with all_gather and the check sums with
    all_reduce, as the sharded device loop does."""
    import torch
    m, n = K.shape
    x = np.clip(np.zeros(n), l, u)
    y = np.zeros(m)
    kx = K @ x
    sums = []
    for _ in range(iters):
        if shard is None:
            xn = np.clip(x - (eta / omega) * (c - K.T @ y), l, u)
            kxn = K @ xn
        else:
            dist, rank, rb, cb = shard
            c0, c1 = cb[rank], cb[rank + 1]
            part = np.clip(x[c0:c1] - (eta / omega) * (c[c0:c1] - K[:, c0:c1].T @ y), l[c0:c1], u[c0:c1])
            xn = _all_gather(dist, torch, part, cb)
            r0, r1 = rb[rank], rb[rank + 1]
            kxn = np.zeros(m)
            kxn[r0:r1] = K[r0:r1] @ xn
        v = y + eta * omega * (q - (2.0 * kxn - kx))
        yn = np.where(eq, v, np.maximum(v, 0.0))
        if shard is not None:
            dist, rank, rb, cb = shard
            r0, r1 = rb[rank], rb[rank + 1]
            yn = _all_gather(dist, torch, yn[r0:r1], rb)
            kxn = _all_gather(dist, torch, kxn[r0:r1], rb)
            s = np.array([np.sum((K[r0:r1] @ xn - q[r0:r1]) ** 2), np.sum(c[cb[rank]:cb[rank + 1]] * xn[cb[rank]:cb[rank + 1]])])
            t = torch.from_numpy(s)
            dist.all_reduce(t)
            sums.append(t.numpy())
        else:
            sums.append(np.array([np.sum((K @ xn - q) ** 2), np.sum(c * xn)]))
        x, y, kx = xn, yn, kxn
    return x, y, np.array(sums)


def _all_gather(dist, torch, part, begin):
    world = len(begin) - 1
    slice_ = int(max(np.diff(begin)))
    buf = torch.zeros(slice_, dtype=torch.float64)
    buf[:len(part)] = torch.from_numpy(np.ascontiguousarray(part))
    outs = [torch.zeros(slice_, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(outs, buf)
    return np.concatenate([outs[b][:begin[b + 1] - begin[b]].numpy() for b in range(world)])


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = GenStaircase(4, 12, 15, 5, 2, seed=7)
        K = np.vstack([p.a.to_dense(), p.g.to_dense()])
        q = np.concatenate([p.b, p.h])
        eq = np.arange(K.shape[0]) < p.num_eq_rows()
        kptr = np.concatenate([p.a.row_ptr[:-1], p.a.nnz + p.g.row_ptr])
        rb = PartitionBlocks(kptr, world, 6)
        cptr = np.concatenate([[0], np.cumsum(np.count_nonzero(K, axis=0))])
        cb = PartitionBlocks(cptr, world, 6)
        args = (K, q, p.c, p.l, p.u, eq, 0.05, 1.0, 25)
        xs, ys, ss = _pdhg_iters(*args, shard=(dist, rank, rb, cb))
        x1, y1, s1 = _pdhg_iters(*args)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), rb=rb, cb=cb, xs=xs, ys=ys, ss=ss, x1=x1, y1=y1, s1=s1)
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_sharded_iteration(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    np.testing.assert_array_equal(r[0]["rb"], r[1]["rb"])  # every rank computes the same split
    np.testing.assert_array_equal(r[0]["cb"], r[1]["cb"])
    assert r[0]["rb"][1] > 0 and r[0]["cb"][1] > 0
    for k in range(world):
        # slice-wise updates + all-gather reproduce the unsharded iterates exactly
        np.testing.assert_array_equal(r[k]["xs"], r[k]["x1"])
        np.testing.assert_array_equal(r[k]["ys"], r[k]["y1"])
        np.testing.assert_allclose(r[k]["ss"], r[k]["s1"], rtol=1e-12)
    np.testing.assert_array_equal(r[0]["ss"], r[1]["ss"])  # all-reduced sums agree across ranks


# ------------------------------------------- power-iteration start vector
@pytest.mark.parametrize("seed", [0, 1, 12345])
@pytest.mark.parametrize("n", [1, 7, 32768, 40000, 100001, 262147])
def test_parallel_normal_vector_is_bit_exact(seed, n):
    """The pipelined multi-threaded start vector (csrc/normal_rng.h) equals the
    sequential libstdc++ std::normal_distribution / std::mt19937_64 draw bit
    for bit, for every worker count (1 worker, odd counts, the host's)."""
    import ctypes as C
    from paper_2312_14832_b200 import abi
    lib = abi.load()
    dp = lambda v: v.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    ref = np.empty(n)
    assert lib.pdhg_normal_vector(seed, n, 1, dp(ref)) == 0
    for threads in (-1, 2, 3, 8):
        out = np.full(n, np.nan)
        assert lib.pdhg_normal_vector(seed, n, threads, dp(out)) == 0
        np.testing.assert_array_equal(out.view(np.uint64), ref.view(np.uint64))


# ------------------------------- gloo world_size-3 ghost-only exchange test
def _ghost_lists(K, row_begin, col_begin, me):
    """Entries block `me` reads from every other column block (recv) and the
    entries of block `me`'s slice every other block reads (send) -- the
    definition csrc/session.cu BuildGhostPlan implements."""
    world = len(row_begin) - 1
    nz = K != 0
    recv, send = {}, {}
    for b in range(world):
        if b == me:
            continue
        cols = np.arange(col_begin[b], col_begin[b + 1])
        recv[b] = cols[nz[row_begin[me]:row_begin[me + 1], col_begin[b]:col_begin[b + 1]].any(axis=0)]
        mine = np.arange(col_begin[me], col_begin[me + 1])
        send[b] = mine[nz[row_begin[b]:row_begin[b + 1], col_begin[me]:col_begin[me + 1]].any(axis=0)]
    return recv, send


def _ghost_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = GenStaircase(6, 14, 16, 5, 2, seed=11)
        K = np.vstack([p.a.to_dense(), p.g.to_dense()])
        kptr = np.concatenate([p.a.row_ptr[:-1], p.a.nnz + p.g.row_ptr])
        rb = PartitionBlocks(kptr, world, 6)
        cb = PartitionBlocks(np.concatenate([[0], np.cumsum(np.count_nonzero(K, axis=0))]), world, 6)
        # K x with rows of block `rank`, x exchanged ghost-only (x_full NaN elsewhere)
        rng = np.random.default_rng(3)
        x = rng.standard_normal(K.shape[1])
        x_full = np.full(K.shape[1], np.nan)
        x_full[cb[rank]:cb[rank + 1]] = x[cb[rank]:cb[rank + 1]]
        recv, send = _ghost_lists(K, rb, cb, rank)
        reqs = []
        bufs = {}
        for b in range(world):
            if b == rank:
                continue
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x_full[send[b]])), dst=b))
            bufs[b] = torch.zeros(len(recv[b]), dtype=torch.float64)
            reqs.append(dist.irecv(bufs[b], src=b))
        for r in reqs:
            r.wait()
        for b, t in bufs.items():
            x_full[recv[b]] = t.numpy()
        rows = slice(rb[rank], rb[rank + 1])
        sub = K[rows]
        kx = np.array([np.sum(sub[i][sub[i] != 0] * x_full[sub[i] != 0]) for i in range(sub.shape[0])])
        ghost = sum(len(v) for v in recv.values())
        np.savez(os.path.join(out_dir, f"g{rank}.npz"), kx=kx, want=K[rows] @ x, ghost=ghost,
                 full=(world - 1) * int(max(np.diff(cb))))
    finally:
        dist.destroy_process_group()


def test_gloo_three_rank_ghost_exchange(tmp_path):
    """Ghost-only exchange (send/recv of just the entries each row block
    reads) reproduces the row products exactly; everything outside the own
    slice and the ghost lists stays NaN, so a missing ghost would show."""
    import torch.multiprocessing as mp
    world = 3
    mp.spawn(_ghost_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for k in range(world):
        r = np.load(tmp_path / f"g{k}.npz")
        assert np.all(np.isfinite(r["kx"]))
        np.testing.assert_allclose(r["kx"], r["want"], rtol=1e-13, atol=1e-13)
        assert r["ghost"] < r["full"]  # staircase: far less than an all-gather


# ------------------------------------------------ LpProblem::Validate (C-ABI)
def _big_lp(n=600_000):
    """A 1-row LP large enough for the threaded validation scan."""
    from paper_2312_14832_b200.rpdlp import CsrMatrix, LpProblem
    a = CsrMatrix(0, n, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    g = CsrMatrix(1, n, np.array([0, 2], np.int64), np.array([0, n - 1], np.int64), np.ones(2))
    return LpProblem(a, g, np.ones(n), np.zeros(0), np.zeros(1), np.zeros(n), np.ones(n))


@pytest.mark.parametrize("where", [0, 299_999, 599_999])
def test_validation_precedence_on_large_inputs(where):
    """lp_problem.cpp:22-58 order and messages, through the threaded scan the
    C-ABI runs before any device work (no GPU needed): NaN in c beats an
    infinite c and a crossed bound anywhere; the FIRST bad bound index is
    reported; NaN bound beats crossed at the same index."""
    from paper_2312_14832_b200 import rpdlp
    p = _big_lp()
    n = p.c.size
    p.l[n - 1] = 5.0  # a crossed bound at the end ...
    p.l[where] = 3.0  # ... and the first one here
    with pytest.raises(ValueError, match=f"crossed bounds: l > u at index {where}$"):
        rpdlp.Solve(p)
    p.u[where] = np.nan
    with pytest.raises(ValueError, match="NaN bound"):
        rpdlp.Solve(p)
    p.c[n - 1 - where] = np.inf
    with pytest.raises(ValueError, match="infinite entry in c"):
        rpdlp.Solve(p)
    p.c[where // 2] = np.nan
    with pytest.raises(ValueError, match="NaN in c"):
        rpdlp.Solve(p)


# ------------------------------- PageRank graph / LP builder / edge lists
@pytest.mark.parametrize("seed", [0, 3])
def test_pagerank_graph_then_build_equals_generator(seed):
    """GenPagerank == BuildPagerankLp(GenPagerankGraph) (instance_gen.cpp:139-141),
    bit for bit; edge count core + (n - core) * attachment."""
    e = rpdlp.GenPagerankGraph(3000, 0.85, 4, seed)
    assert e.shape == (5 + (3000 - 5) * 4, 2)
    a, b = rpdlp.BuildPagerankLp(e, 3000, 0.85), rpdlp.GenPagerank(3000, 0.85, 4, seed)
    for m in ("a", "g"):
        x, y = getattr(a, m), getattr(b, m)
        np.testing.assert_array_equal(x.row_ptr, y.row_ptr)
        np.testing.assert_array_equal(x.col_idx, y.col_idx)
        np.testing.assert_array_equal(x.values.view(np.uint64), y.values.view(np.uint64))
    np.testing.assert_array_equal(a.h, b.h)


def test_edge_list_reader_and_builder(tmp_path):
    """instance_gen.cpp:66-137: comments / blank lines skipped, sparse ids
    compacted in first-appearance order, dangling nodes get self-loops,
    malformed lines and out-of-range endpoints rejected."""
    f = tmp_path / "g.txt"
    f.write_text("# a comment\n\n10 20\n  20 30\n\t# indented comment\n30 10 extra\n40 20\n")
    e, n = rpdlp.ReadEdgeList(f)
    assert n == 4 and e.tolist() == [[0, 1], [1, 2], [2, 0], [3, 1]]
    p = rpdlp.BuildPagerankLp(e, n, 0.5)
    d = p.g.to_dense()
    # node 3 has in-degree 0 but out-degree 1; no dangling node here
    np.testing.assert_allclose(np.diag(d), [1.0, 1.0, 1.0, 1.0])
    assert d[1, 0] == -0.5 and d[1, 3] == -0.5 and d[2, 1] == -0.5 and d[0, 2] == -0.5
    np.testing.assert_allclose(p.h, [0.125] * 4)
    assert p.a.to_dense().tolist() == [[1.0, 1.0, 1.0, 1.0]] and list(p.b) == [1.0]
    dang = rpdlp.BuildPagerankLp(np.array([[0, 1]]), 2, 0.85).g.to_dense()
    assert dang[1, 1] == pytest.approx(1.0 - 0.85)  # dangling node 1: self-loop
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2\n3\n")
    with pytest.raises(RuntimeError, match="malformed edge line"):
        rpdlp.ReadEdgeList(bad)
    with pytest.raises(ValueError, match="edge endpoint out of range"):
        rpdlp.BuildPagerankLp(np.array([[0, 5]]), 3, 0.85)
    with pytest.raises(ValueError, match="empty graph"):
        rpdlp.BuildPagerankLp(np.zeros((0, 2), np.int64), 0, 0.85)

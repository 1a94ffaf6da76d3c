"""Multi-process host logic of the multi-GPU drivers (paper_1004_3719_b200/dist.py),
world_size 2 over gloo on CPU.  The per-rank compute is an exact reference
backend built on the oracle (test infrastructure), so these tests check the
partitioning, the per-step all-gather, and the assembly of S -- the parts the
GPU path shares -- against the single-process oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


class RefBackend:
    device = torch.device("cpu")

    def __init__(self, m):
        import oracle
        self.o = oracle
        self.m = m

    def tensor(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32).copy())

    def empty(self, shape):
        return torch.zeros(shape, dtype=torch.int32)

    def to_numpy(self, t):
        return t.contiguous().numpy().view(np.uint32)

    def create(self, rows, cols, ri, ci, v, m):
        return (rows, cols, np.asarray(ri), np.asarray(ci), np.asarray(v))

    def sequence(self, A, X, L, U):
        rows, cols, ri, ci, v = A
        S = self.o.sequence(rows, ri, ci, v, self.m, self.to_numpy(X), L, self.to_numpy(U))
        return self.tensor(S)

    def apply_block(self, A, X, out):
        rows, cols, ri, ci, v = A
        Y = self.o.apply_block(rows, cols, ri, ci, v, self.m, self.to_numpy(X))
        out.copy_(self.tensor(Y))
        return out

    def project(self, A, V, U, out):
        n = V.shape[0]
        z = np.zeros(0, np.uint32)
        S = self.o.sequence(n, z, z, np.zeros(0, np.int64), self.m, self.to_numpy(V), 1,
                            self.to_numpy(U))
        out.copy_(self.tensor(S[0]))
        return out

    def sum_mod(self, A, parts, out):
        s = self.to_numpy(parts).astype(np.uint64).sum(axis=0) % self.m
        out.copy_(self.tensor(s.astype(np.uint32)))
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, case, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1004_3719_b200 import dist as fd
        n, ri, ci, v, m, X, U, L = case
        be = RefBackend(m)
        if mode == "rows":
            S, V = fd.sequence_rows(n, ri, ci, v, m, X, L, U, be, want_vout=True)
            result_q.put((rank, S, V))
        elif mode.startswith("2d"):
            pr, pc = (int(t) for t in mode[2:].split("x"))
            seen = []
            S, V = fd.sequence_2d(n, ri, ci, v, m, X, L, U, be, pr, pc, want_vout=True, on_step=seen.append)
            assert seen == list(range(L + 1)), seen       # the bench's timing hook
            result_q.put((rank, S, V))
        else:
            S = fd.sequence_columns(n, ri, ci, v, m, X, L, U, be)
            result_q.put((rank, S, None))
    finally:
        dist.destroy_process_group()


def _run(mode, case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def _case(n=70, k=5, ku=3, L=6, m=65521, seed=3):
    g = synth.rng(seed)
    ri, ci, v = synth.random_coo(g, n, n, 6 * n, m, dup=0.05)
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, ku), m)
    return (n, ri, ci, v, m, X, U, L)


@pytest.mark.parametrize("mode", ["rows", "columns"])
def test_sequence_world2_matches_oracle(oracle_mod, mode):
    case = _case()
    n, ri, ci, v, m, X, U, L = case
    want, Vw = oracle_mod.sequence(n, ri, ci, v, m, X, L, U, want_vout=True)
    res = _run(mode, case)
    for rank, S, V in res:
        assert np.array_equal(np.asarray(S).reshape(want.shape), want), f"rank {rank}"
        if V is not None:
            assert np.array_equal(V, Vw)


def test_partitioning_edge_cases():
    from paper_1004_3719_b200 import dist as fd
    # nnz-balanced bands cover every row exactly once, also with empty rows,
    # more ranks than rows, and N not divisible by P
    for rows, world in ((10, 3), (3, 8), (1000, 7)):
        ri = np.repeat(np.arange(rows), np.arange(rows) % 5)
        b = fd.row_bands(ri, rows, world)
        assert b[0] == 0 and b[-1] == rows and np.all(np.diff(b) >= 0) and len(b) == world + 1
    c = fd.column_shards(16, 3)
    assert c.tolist() == [0, 5, 10, 16]
    c = fd.column_shards(2, 4)
    assert c[0] == 0 and c[-1] == 2 and np.all(np.diff(c) >= 0)
    # band re-basing
    r2, c2, v2 = fd.band_triples(np.array([0, 3, 5]), np.array([1, 2, 3]), np.array([7, 8, 9]), 3, 6)
    assert r2.tolist() == [0, 2] and c2.tolist() == [2, 3] and v2.tolist() == [8, 9]


def test_rows_mode_uneven_world2(oracle_mod):
    # all nonzeros in the first rows: one band carries nearly everything
    n, m = 40, 251
    g = synth.rng(9)
    ri = g.integers(0, 5, size=120).astype(np.uint32)
    ci = g.integers(0, n, size=120).astype(np.uint32)
    v = g.integers(-m, m, size=120)
    X = synth.uniform(g, (n, 2), m)
    case = (n, ri, ci, v, m, X, None, 5)
    want = oracle_mod.sequence(n, ri, ci, v, m, X, 5)
    for rank, S, V in _run("rows", case):
        assert np.array_equal(np.asarray(S).reshape(want.shape), want)


@pytest.mark.parametrize("grid", ["2d2x2", "2d1x2", "2d2x1", "2d4x1"])
def test_sequence_2d_matches_oracle(oracle_mod, grid):
    # P_r x P_c grid (world 4 or 2): row bands x column blocks, all-gather of
    # the iterate within each column block, projections summed over bands
    pr, pc = (int(t) for t in grid[2:].split("x"))
    case = _case(n=53, k=5, ku=3, L=5, m=2147483647, seed=11)
    n, ri, ci, v, m, X, U, L = case
    want, Vw = oracle_mod.sequence(n, ri, ci, v, m, X, L, U, want_vout=True)
    for rank, S, V in _run(grid, case, world=pr * pc):
        assert np.array_equal(np.asarray(S).reshape(want.shape), want), f"rank {rank}"
        assert np.array_equal(V, Vw), f"rank {rank}"


def test_grid_shape():
    from paper_1004_3719_b200 import dist as fd
    # c5 sizes (N = 2^21, ~21 M nnz, k = 16, u16 iterate): the byte model of
    # SURVEY §8e picks 2 x 4 at P = 8 (NVLink-bound 8 x 1, matrix-bound 1 x 8)
    assert fd.grid_shape(8, 16, n=1 << 21, nnz=21_000_000) == (2, 4)
    for w in (1, 2, 4, 8):
        pr, pc = fd.grid_shape(w, 16, n=1 << 21, nnz=21_000_000)
        assert pr * pc == w and pc <= 16
    assert fd.grid_shape(8, 1, n=1 << 21, nnz=21_000_000) == (8, 1)    # one column: rows only
    assert fd.grid_shape(4, 16) == (1, 4)                              # no sizes: columns first

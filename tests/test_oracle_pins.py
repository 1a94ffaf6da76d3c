"""Pins for the CPU oracle (``oracle/``) against things other than itself.

Each test fixes the oracle to a value the paper prints, a closed form, an
invariant of the mathematics, or dense big-integer brute force on tiny
inputs -- chosen so a dropped term, a wrong sign/index or a transposed
operand in oracle.c fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def dense(rows, cols, ri, ci, val):
    """Dense expansion with Python big integers (no residues taken)."""
    D = [[0] * cols for _ in range(rows)]
    for r, c, v in zip(ri.tolist(), ci.tolist(), val.tolist()):
        D[r][c] += int(v)
    return D


def brute_apply(D, m, x, y, alpha, beta):
    out = []
    for i, row in enumerate(D):
        s = sum(a * int(xj) for a, xj in zip(row, x))
        out.append((alpha * s + beta * int(y[i])) % m)
    return np.array(out, dtype=np.uint64).astype(np.uint32)


def transpose_dense(D, cols):
    return [[D[i][j] for i in range(len(D))] for j in range(cols)]


# --------------------------------------------------------------------------
# 1. The paper's worked example, golden fixture.
# --------------------------------------------------------------------------

def load_golden():
    with open(os.path.join(HERE, "golden", "paper_2x2_mod27.json")) as f:
        return json.load(f)


def test_paper_listing(oracle_mod):
    g = load_golden()
    t = np.array(g["triples"], dtype=np.int64)
    ri, ci, val = t[:, 0].astype(np.uint32), t[:, 1].astype(np.uint32), t[:, 2]
    for case in g["cases"]:
        y = oracle_mod.apply(2, 2, ri, ci, val, g["m"], case["x"], case["y"],
                             case["alpha"], case["beta"])
        assert y.tolist() == case["expect"], case["what"]
    for case in g["transpose_cases"]:
        y = oracle_mod.apply_transpose(2, 2, ri, ci, val, g["m"], case["x"])
        assert y.tolist() == case["expect"], case["what"]


def test_paper_powers_and_sequence(oracle_mod):
    g = load_golden()
    t = np.array(g["triples"], dtype=np.int64)
    ri, ci, val = t[:, 0].astype(np.uint32), t[:, 1].astype(np.uint32), t[:, 2]
    x = np.array(g["powers"]["x"], np.uint32)
    for n, want in enumerate(g["powers"]["expect"]):
        S, V = oracle_mod.sequence(2, ri, ci, val, g["m"], x.reshape(2, 1), n, want_vout=True)
        assert V.ravel().tolist() == want
    s = g["sequence"]
    S = oracle_mod.sequence(2, ri, ci, val, g["m"], np.array(s["Y"], np.uint32), s["L"])
    assert S.ravel().tolist() == s["expect"]


# --------------------------------------------------------------------------
# 2. Dense big-integer brute force on tiny random matrices.
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m", synth.MODULI)
def test_bruteforce_apply_and_transpose(oracle_mod, m):
    g = synth.rng(7 + m % 1000)
    for trial in range(12):
        rows, cols = int(g.integers(0, 24)), int(g.integers(0, 24))
        nnz = int(g.integers(0, 1 + rows * cols)) if rows * cols else 0
        ri, ci, val = synth.random_coo(g, rows, cols, nnz, m, dup=0.2, big=True)
        D = dense(rows, cols, ri, ci, val)
        x = synth.uniform(g, cols, m)
        y = synth.uniform(g, rows, m)
        alpha, beta = int(g.integers(0, 1 << 32)), int(g.integers(0, 1 << 32))
        got = oracle_mod.apply(rows, cols, ri, ci, val, m, x, y, alpha, beta)
        assert np.array_equal(got, brute_apply(D, m, x, y, alpha, beta))
        xt = synth.uniform(g, rows, m)
        yt = synth.uniform(g, cols, m)
        got_t = oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, xt, yt, alpha, beta)
        assert np.array_equal(got_t, brute_apply(transpose_dense(D, cols), m, xt, yt, alpha, beta))


@pytest.mark.parametrize("m", [2, 3, 65521, (1 << 31) - 1, (1 << 32) - 1])
def test_bruteforce_block(oracle_mod, m):
    g = synth.rng(99 + m % 997)
    for k in (1, 2, 3, 8):
        rows, cols = 9, 13
        ri, ci, val = synth.random_coo(g, rows, cols, 40, m, dup=0.1)
        D = dense(rows, cols, ri, ci, val)
        X = synth.uniform(g, (cols, k), m)
        Y = synth.uniform(g, (rows, k), m)
        got = oracle_mod.apply_block(rows, cols, ri, ci, val, m, X, Y, alpha=5, beta=7)
        for c in range(k):
            assert np.array_equal(got[:, c], brute_apply(D, m, X[:, c], Y[:, c], 5, 7))


def test_bruteforce_sequence(oracle_mod):
    for m in (3, 251, 65521, (1 << 32) - 5):
        g = synth.rng(m % 1013)
        n, k, ku, L = 7, 3, 2, 6
        ri, ci, val = synth.random_coo(g, n, n, 20, m)
        D = dense(n, n, ri, ci, val)
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, ku), m)
        S, V = oracle_mod.sequence(n, ri, ci, val, m, X, L, U, want_vout=True)
        Vt = [[int(v) for v in row] for row in X]
        for t in range(L):
            for a in range(ku):
                for b in range(k):
                    want = sum(int(U[r, a]) * Vt[r][b] for r in range(n)) % m
                    assert int(S[t, a, b]) == want
            Vt = [[sum(D[i][j] * Vt[j][b] for j in range(n)) % m for b in range(k)]
                  for i in range(n)]
        assert V.tolist() == Vt


# --------------------------------------------------------------------------
# 3. Closed forms.
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m", [2, 65521, (1 << 31) - 1, (1 << 32) - 1])
def test_identity_permutation_diagonal_zero(oracle_mod, m):
    g = synth.rng(5)
    n = 50
    x = synth.uniform(g, n, m)
    y = synth.uniform(g, n, m)
    idx = np.arange(n, dtype=np.uint32)
    a, b = 123456789, 987654321
    # identity -> alpha x + beta y
    got = oracle_mod.apply(n, n, idx, idx, np.ones(n, np.int64), m, x, y, a, b)
    want = [(a * int(xi) + b * int(yi)) % m for xi, yi in zip(x, y)]
    assert got.tolist() == want
    # permutation pi: (P x)_i = x_{pi(i)}; transpose gives the inverse
    pi = g.permutation(n).astype(np.uint32)
    got = oracle_mod.apply(n, n, idx, pi, np.ones(n, np.int64), m, x)
    assert got.tolist() == [int(x[p]) for p in pi]
    inv = np.empty(n, np.int64)
    inv[pi] = np.arange(n)
    got_t = oracle_mod.apply_transpose(n, n, idx, pi, np.ones(n, np.int64), m, x)
    assert got_t.tolist() == [int(x[p]) for p in inv]
    # diagonal d
    d = g.integers(-(1 << 40), 1 << 40, size=n)
    got = oracle_mod.apply(n, n, idx, idx, d, m, x)
    assert got.tolist() == [(int(di) * int(xi)) % m for di, xi in zip(d, x)]
    # zero matrix -> beta y ; empty triple list
    got = oracle_mod.apply(n, n, idx[:0], idx[:0], d[:0], m, x, y, a, b)
    assert got.tolist() == [(b * int(yi)) % m for yi in y]


@pytest.mark.parametrize("m", [3, 65521, (1 << 31) - 1, (1 << 32) - 5, (1 << 32) - 1])
@pytest.mark.parametrize("R", [1, 2, 3, 4, 5, 1000, 100000])
def test_overflow_worst_case(oracle_mod, m, R):
    """A row of R entries m-1 times x = m-1: (Ax)_0 = R (m-1)^2 = R (mod m);
    with y = m-1 and beta = 1 the result is R - 1 (mod m).  R (m-1)^2 exceeds
    2^64 for large m, so a 64-bit accumulator would fail here."""
    cols = R
    ri = np.zeros(R, np.uint32)
    ci = np.arange(R, dtype=np.uint32)
    val = np.full(R, m - 1, np.int64)
    x = np.full(cols, m - 1, np.uint32)
    got = oracle_mod.apply(1, cols, ri, ci, val, m, x)
    assert int(got[0]) == R % m
    got = oracle_mod.apply(1, cols, ri, ci, val, m, x, np.array([m - 1], np.uint32), 1, 1)
    assert int(got[0]) == (R - 1) % m
    # +-1 rows with x = 0 exercise the (m - x) = m addend of a -1 entry
    got = oracle_mod.apply(1, cols, ri, ci, np.full(R, -1, np.int64), m, np.zeros(cols, np.uint32))
    assert int(got[0]) == 0


# --------------------------------------------------------------------------
# 4. Invariants.
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m", [2, 3, 251, 65521, (1 << 32) - 1])
def test_transpose_duality(oracle_mod, m):
    """(A x) . y == x . (A^T y)  (mod m)."""
    g = synth.rng(11)
    for _ in range(10):
        rows, cols = int(g.integers(1, 60)), int(g.integers(1, 60))
        ri, ci, val = synth.random_coo(g, rows, cols, int(g.integers(0, 200)), m, dup=0.1)
        x = synth.uniform(g, cols, m)
        y = synth.uniform(g, rows, m)
        Ax = oracle_mod.apply(rows, cols, ri, ci, val, m, x)
        Aty = oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, y)
        lhs = sum(int(a) * int(b) for a, b in zip(Ax, y)) % m
        rhs = sum(int(a) * int(b) for a, b in zip(x, Aty)) % m
        assert lhs == rhs


@pytest.mark.parametrize("m", [3, 65521, (1 << 32) - 5])
def test_linearity_and_split(oracle_mod, m):
    """A(x + x') = Ax + Ax'; (A1 + A2) x = A1 x + A2 x for any split of the
    triples (pins the +-1 / valued / format piece decomposition)."""
    g = synth.rng(13)
    rows, cols = 40, 30
    ri, ci, val = synth.random_coo(g, rows, cols, 300, m, dup=0.1)
    x1 = synth.uniform(g, cols, m)
    x2 = synth.uniform(g, cols, m)
    xs = ((x1.astype(np.uint64) + x2) % m).astype(np.uint32)
    a = oracle_mod.apply(rows, cols, ri, ci, val, m, x1).astype(np.uint64)
    b = oracle_mod.apply(rows, cols, ri, ci, val, m, x2).astype(np.uint64)
    c = oracle_mod.apply(rows, cols, ri, ci, val, m, xs)
    assert np.array_equal(((a + b) % m).astype(np.uint32), c)
    cut = g.random(ri.size) < 0.5
    p1 = oracle_mod.apply(rows, cols, ri[cut], ci[cut], val[cut], m, x1).astype(np.uint64)
    p2 = oracle_mod.apply(rows, cols, ri[~cut], ci[~cut], val[~cut], m, x1).astype(np.uint64)
    assert np.array_equal(((p1 + p2) % m).astype(np.uint32), a.astype(np.uint32))
    # y <- Ax + y equals apply then add
    y = synth.uniform(g, rows, m)
    got = oracle_mod.apply(rows, cols, ri, ci, val, m, x1, y, 1, 1)
    assert np.array_equal(got, ((a + y) % m).astype(np.uint32))


def test_block_columns_and_identity(oracle_mod):
    m = 65521
    g = synth.rng(17)
    rows, cols = 25, 20
    ri, ci, val = synth.random_coo(g, rows, cols, 120, m, dup=0.1)
    X = np.eye(cols, dtype=np.uint32)
    Y = oracle_mod.apply_block(rows, cols, ri, ci, val, m, X)
    D = dense(rows, cols, ri, ci, val)
    assert Y.tolist() == [[v % m for v in row] for row in D]


def test_sequence_closed_forms(oracle_mod):
    m = 65521
    g = synth.rng(19)
    n, k, ku = 12, 3, 2
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, ku), m)
    idx = np.arange(n, dtype=np.uint32)
    L = 9
    # A = c I  ->  S_t = c^t S_0
    c = 12345
    S = oracle_mod.sequence(n, idx, idx, np.full(n, c, np.int64), m, X, L, U)
    for t in range(L):
        assert np.array_equal(S[t].astype(np.uint64),
                              (S[0].astype(np.uint64) * pow(c, t, m)) % m)
    # diagonal d  ->  S_t[a][b] = sum_r U[r][a] d_r^t X[r][b]
    d = g.integers(0, m, size=n)
    S = oracle_mod.sequence(n, idx, idx, d, m, X, L, U)
    for t in range(L):
        for a in range(ku):
            for b in range(k):
                want = sum(int(U[r, a]) * pow(int(d[r]), t, m) * int(X[r, b]) for r in range(n)) % m
                assert int(S[t, a, b]) == want
    # nilpotent shift (row i <- x_{i+1})  ->  S_t = 0 for t >= n
    S = oracle_mod.sequence(n, idx[:-1], idx[1:], np.ones(n - 1, np.int64), m, X, n + 3, U)
    assert not S[n:].any() and S[:n].any()
    # permutation of order q  ->  S_{t+q} = S_t
    q = 5
    cyc = np.arange(n)
    cyc[:q] = (np.arange(q) + 1) % q
    S = oracle_mod.sequence(n, idx, cyc.astype(np.uint32), np.ones(n, np.int64), m, X, 3 * q, U)
    assert np.array_equal(S[:q], S[q:2 * q]) and np.array_equal(S[:q], S[2 * q:])
    # U = None means U = X (the paper's Y^T A^i Y)
    ri, ci, val = synth.random_coo(g, n, n, 40, m)
    S1 = oracle_mod.sequence(n, ri, ci, val, m, X, 4)
    S2 = oracle_mod.sequence(n, ri, ci, val, m, X, 4, X)
    assert np.array_equal(S1, S2)


def test_sequence_chaining(oracle_mod):
    """S over [0, L1+L2) = concat(S(X, L1), S(A^L1 X, L2)); A^i x = i applies."""
    m = 251
    g = synth.rng(23)
    n, k = 15, 2
    ri, ci, val = synth.random_coo(g, n, n, 60, m)
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, 3), m)
    S, V = oracle_mod.sequence(n, ri, ci, val, m, X, 7, U, want_vout=True)
    S1, V1 = oracle_mod.sequence(n, ri, ci, val, m, X, 3, U, want_vout=True)
    S2, V2 = oracle_mod.sequence(n, ri, ci, val, m, V1, 4, U, want_vout=True)
    assert np.array_equal(S, np.concatenate([S1, S2])) and np.array_equal(V, V2)
    v = X[:, 0].copy()
    for _ in range(7):
        v = oracle_mod.apply(n, n, ri, ci, val, m, v)
    assert np.array_equal(v, V[:, 0])


def test_preconditions(oracle_mod):
    idx = np.zeros(1, np.uint32)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.apply(1, 1, idx + 1, idx, np.ones(1, np.int64), 5, [0])   # row out of range
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.apply(1, 1, idx, idx, np.ones(1, np.int64), 5, [5])       # x not canonical
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.apply(1, 1, idx, idx, np.ones(1, np.int64), 1, [0])       # m < 2


# --------------------------------------------------------------------------
# 6. Threaded timing mode: pinned to dense brute force
#    on tiny inputs and to the serial functions on larger ones, for thread
#    counts that leave threads empty and cut keys at every boundary.
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m", [2, 3, 65521, (1 << 31) - 1, (1 << 32) - 1])
def test_threaded_mode_bruteforce(oracle_mod, m):
    g = synth.rng(404 + m % 991)
    for trial in range(8):
        rows, cols = int(g.integers(0, 20)), int(g.integers(0, 20))
        nnz = int(g.integers(0, 1 + rows * cols)) if rows * cols else 0
        ri, ci, val = synth.random_coo(g, rows, cols, nnz, m, dup=0.2, big=True)
        D = dense(rows, cols, ri, ci, val)
        x, y = synth.uniform(g, cols, m), synth.uniform(g, rows, m)
        alpha, beta = int(g.integers(0, 1 << 32)), int(g.integers(0, 1 << 32))
        r_s, c_s, v_s = oracle_mod.sort_triples(ri, ci, val)
        for T in (1, 3, 64):
            got = oracle_mod.apply_mt(rows, cols, r_s, c_s, v_s, m, x, y, alpha, beta, nthreads=T)
            assert np.array_equal(got, brute_apply(D, m, x, y, alpha, beta))
        xt, yt = synth.uniform(g, rows, m), synth.uniform(g, cols, m)
        c_t, r_t, v_t = oracle_mod.sort_triples(ci, ri, val)
        for T in (2, 5):
            got = oracle_mod.apply_transpose_mt(rows, cols, c_t, r_t, v_t, m, xt, yt, alpha, beta,
                                                nthreads=T)
            assert np.array_equal(got, brute_apply(transpose_dense(D, cols), m, xt, yt, alpha, beta))


def test_threaded_mode_matches_serial(oracle_mod):
    g = synth.rng(4242)
    M = synth.config_matrix("c2", scale=1 / 64)
    m, n = M["m"], M["rows"]
    r_s, c_s, v_s = oracle_mod.sort_triples(M["row"], M["col"], M["val"])
    X = synth.uniform(g, (n, 5), m)
    U = synth.uniform(g, (n, 3), m)
    for T in (1, 4, 7):
        assert np.array_equal(oracle_mod.apply_block_mt(n, n, r_s, c_s, v_s, m, X, nthreads=T),
                              oracle_mod.apply_block(n, n, M["row"], M["col"], M["val"], m, X))
        S1, V1 = oracle_mod.sequence_mt(n, r_s, c_s, v_s, m, X, 4, U, want_vout=True, nthreads=T)
        S0, V0 = oracle_mod.sequence(n, M["row"], M["col"], M["val"], m, X, 4, U, want_vout=True)
        assert np.array_equal(S1, S0) and np.array_equal(V1, V0)
    with pytest.raises(oracle_mod.OracleError):            # unsorted input is refused
        oracle_mod.apply_mt(n, n, M["row"][::-1], M["col"][::-1], M["val"][::-1], m, X[:, 0])

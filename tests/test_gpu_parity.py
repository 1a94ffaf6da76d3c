"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, bit-exact (integer arithmetic: tolerance zero).

Covers every operation of SURVEY §8(a) (apply, transpose, block, sequence),
every band format, forced accumulator widths, the moduli that cross every
u8/u16/u32 storage and u32/u64/u96 accumulator boundary, ragged/empty edge
cases, and the BASELINE configs (c1 full; c2-c5 full size on the launch
configuration bench.py times, sampled where the oracle would be too slow).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

MODS = [2, 3, 27, 251, 256, 257, 65521, 65536, 65537, (1 << 20) + 7, (1 << 31) - 1,
        (1 << 32) - 5, (1 << 32) - 1]
OPTS = [dict(), dict(force_format=1), dict(force_format=2), dict(force_format=3),
        dict(segregate_pm1=-1), dict(band_rows=32, long_row=6), dict(force_acc_bits=96),
        dict(force_acc_bits=64, force_format=2, long_row=3),
        dict(strategy=2), dict(strategy=2, panel_rows=32, panel_cols=64),
        dict(strategy=2, panel_rows=96, panel_cols=32, segregate_pm1=-1),
        dict(strategy=3), dict(strategy=3, panel_rows=32, panel_cols=64),
        dict(strategy=3, panel_rows=8, panel_cols=64, segregate_pm1=-1, panel_xbits=32),
        dict(strategy=3, panel_rows=12, panel_cols=128, panel_xbits=16)]


def dev(a):
    import torch
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def rand_case(g, m, rows=None, cols=None, long_rows=False):
    rows = int(g.integers(0, 300)) if rows is None else rows
    cols = int(g.integers(0, 300)) if cols is None else cols
    nnz = int(g.integers(0, 6 * max(rows, 1) + 1))
    ri, ci, val = synth.random_coo(g, rows, cols, nnz, m, dup=0.05, big=True)
    if long_rows and rows and cols:
        for L in (40, 700, 20000):
            r = int(g.integers(0, rows))
            ri = np.concatenate([ri, np.full(L, r, np.uint32)])
            ci = np.concatenate([ci, g.integers(0, cols, size=L).astype(np.uint32)])
            val = np.concatenate([val, g.integers(-m, m, size=L)])
    return rows, cols, ri, ci, val


@pytest.mark.parametrize("m", MODS)
@pytest.mark.parametrize("opt", range(len(OPTS)))
def test_apply_transpose_parity(ff, oracle_mod, cuda, m, opt):
    g = synth.rng(31 * opt + m % 9973)
    for trial in range(3):
        rows, cols, ri, ci, val = rand_case(g, m, long_rows=(trial == 2))
        A = ff.ffspmv_create(rows, cols, ri, ci, val, m, **OPTS[opt])
        for (alpha, beta) in ((1, 0), (1, 1), (int(g.integers(0, 1 << 32)), int(g.integers(0, 1 << 32)))):
            x = synth.uniform(g, cols, m)
            y0 = synth.uniform(g, rows, m)
            want = oracle_mod.apply(rows, cols, ri, ci, val, m, x, y0, alpha, beta)
            yd = dev(y0)
            ff.ffspmv_apply(A, alpha, dev(x), beta, yd)
            assert np.array_equal(host(yd), want)
            xt = synth.uniform(g, rows, m)
            yt0 = synth.uniform(g, cols, m)
            want_t = oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, xt, yt0, alpha, beta)
            ytd = dev(yt0)
            ff.ffspmv_apply_transpose(A, alpha, dev(xt), beta, ytd)
            assert np.array_equal(host(ytd), want_t)


@pytest.mark.parametrize("m", [2, 3, 251, 65521, 65537, (1 << 31) - 1, (1 << 32) - 1])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8, 16, 17, 32, 33, 64])
def test_block_parity(ff, oracle_mod, cuda, m, k):
    g = synth.rng(1000 * k + m % 997)
    for opt in (dict(), dict(force_format=2), dict(force_format=3, long_row=5)):
        rows, cols, ri, ci, val = rand_case(g, m, long_rows=True)
        A = ff.ffspmv_create(rows, cols, ri, ci, val, m, **opt)
        X = synth.uniform(g, (cols, k), m)
        Y0 = synth.uniform(g, (rows, k), m)
        alpha, beta = int(g.integers(0, m)), int(g.integers(0, m))
        want = oracle_mod.apply_block(rows, cols, ri, ci, val, m, X, Y0, alpha, beta)
        Yd = dev(Y0)
        ff.ffspmv_apply_block(A, k, alpha, dev(X), beta, Yd)
        assert np.array_equal(host(Yd), want)


def test_block_leading_dimension(ff, oracle_mod, cuda):
    import torch
    m, k = 65521, 5
    g = synth.rng(77)
    rows, cols, ri, ci, val = rand_case(g, m, rows=120, cols=90)
    A = ff.ffspmv_create(rows, cols, ri, ci, val, m)
    Xw = synth.uniform(g, (cols, 9), m)
    Yw = synth.uniform(g, (rows, 7), m)
    Xd, Yd = dev(Xw), dev(Yw)
    ff.ffspmv_apply_block(A, k, 3, Xd[:, 2:2 + k], 4, Yd[:, 1:1 + k])
    want = oracle_mod.apply_block(rows, cols, ri, ci, val, m, Xw[:, 2:2 + k], Yw[:, 1:1 + k], 3, 4)
    got = host(Yd)
    assert np.array_equal(got[:, 1:1 + k], want)
    assert np.array_equal(got[:, :1], Yw[:, :1]) and np.array_equal(got[:, 1 + k:], Yw[:, 1 + k:])


@pytest.mark.parametrize("m", [3, 251, 65521, 65536, 65537, (1 << 31) - 1, (1 << 32) - 5])
def test_sequence_parity(ff, oracle_mod, cuda, m):
    import torch
    g = synth.rng(m % 10007)
    for (n, k, ku, L, useU, opt) in ((50, 3, 2, 7, True, dict()), (200, 16, 16, 9, False, dict()),
                                      (97, 1, 4, 5, True, dict(force_format=2)),
                                      (130, 8, 33, 4, True, dict(force_format=3, long_row=4)),
                                      (64, 40, 5, 3, True, dict()), (10, 2, 2, 0, False, dict())):
        ri, ci, val = synth.random_coo(g, n, n, 6 * n, m, dup=0.05)
        A = ff.ffspmv_create(n, n, ri, ci, val, m, **opt)
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, ku), m) if useU else None
        Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, L, U, want_vout=True)
        S, V = A.sequence(dev(X), L, dev(U) if useU else None, want_vout=True)
        assert np.array_equal(host(S).reshape(Sw.shape), Sw)
        assert np.array_equal(host(V), Vw)


def test_sequence_paper_example(ff, oracle_mod, cuda):
    # P:249-261 example: S_i = 2*3^i mod 27
    A = ff.ffspmv_create(2, 2, np.array([0, 0, 1], np.uint32), np.array([0, 1, 1], np.uint32),
                         np.array([2, 1, 3], np.int64), 27)
    S = A.sequence(dev(np.ones((2, 1), np.uint32)), 5)
    assert host(S).ravel().tolist() == [2, 6, 18, 0, 0]


def test_empty_and_degenerate(ff, oracle_mod, cuda):
    import torch
    m = 65521
    z = np.zeros(0, np.uint32)
    e = np.zeros(0, np.int64)
    # 0 x 0 matrix
    A = ff.ffspmv_create(0, 0, z, z, e, m)
    ff.ffspmv_apply(A, 1, dev(z), 0, dev(z))
    # rows but no entries: y <- beta y
    A = ff.ffspmv_create(70, 0, z, z, e, m)
    y0 = synth.uniform(synth.rng(1), 70, m)
    yd = dev(y0)
    ff.ffspmv_apply(A, 5, dev(z), 3, yd)
    assert np.array_equal(host(yd), (y0.astype(np.uint64) * 3 % m).astype(np.uint32))
    # every triple cancels (1 + (m-1) = 0) -> zero matrix
    A = ff.ffspmv_create(3, 3, np.array([1, 1], np.uint32), np.array([2, 2], np.uint32),
                         np.array([1, m - 1], np.int64), m)
    assert A.info()["nnz"] == 0
    yd = dev(np.full(3, 9, np.uint32))
    ff.ffspmv_apply(A, 1, dev(np.ones(3, np.uint32)), 0, yd)
    assert host(yd).tolist() == [0, 0, 0]


def test_errors_on_device(ff, cuda):
    import torch
    m = 65521
    g = synth.rng(2)
    ri, ci, val = synth.random_coo(g, 20, 30, 100, m)
    A = ff.ffspmv_create(20, 30, ri, ci, val, m, no_transpose=True, check_inputs=True)
    x = dev(synth.uniform(g, 30, m))
    y = dev(np.zeros(20, np.uint32))
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_apply(A, 1, x[:29], 0, y)
    assert e.value.status == ff.ERR_DIM
    bad = dev(np.full(30, m, np.uint32))
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_apply(A, 1, bad, 0, y)
    assert e.value.status == ff.ERR_INVALID_ARG
    with pytest.raises(ff.FFSPMVError) as e:          # aliasing
        big = dev(np.zeros(64, np.uint32))
        B = ff.ffspmv_create(30, 30, ci, ci, val, m)
        ff.ffspmv_apply(B, 1, big[:30], 0, big[10:40])
    assert e.value.status == ff.ERR_INVALID_ARG
    with pytest.raises(ff.FFSPMVError) as e:
        A.sequence(dev(np.zeros((20, 2), np.uint32)), 3)
    assert e.value.status == ff.ERR_NONSQUARE
    B = ff.ffspmv_create(30, 30, ci, ci, val, m)
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_sequence(B, 2, dev(np.zeros((30, 2), np.uint32)), 2, None, 3,
                           dev(np.zeros(12, np.uint32)), None, ws)
    assert e.value.status == ff.ERR_NOMEM


def test_apply_host_end_to_end(ff, oracle_mod, cuda):
    m = 65521
    g = synth.rng(8)
    rows, cols, ri, ci, val = rand_case(g, m, rows=500, cols=400)
    A = ff.ffspmv_create(rows, cols, ri, ci, val, m)
    x = synth.uniform(g, cols, m)
    y = synth.uniform(g, rows, m)
    want = oracle_mod.apply(rows, cols, ri, ci, val, m, x, y, 7, 11)
    ff.ffspmv_apply_host(A, ff.OP_APPLY, 7, x, 11, y)
    assert np.array_equal(y, want)
    xt = synth.uniform(g, rows, m)
    yt = np.zeros(cols, np.uint32)
    ff.ffspmv_apply_host(A, ff.OP_TRANSPOSE, 1, xt, 0, yt)
    assert np.array_equal(yt, oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, xt))


def test_overflow_adversarial(ff, oracle_mod, cuda):
    """Rows of R entries m-1 (valued path: use m-2 and -2) times x = m-1, for
    every accumulator boundary (SURVEY §8c 'Overflow worst case')."""
    for m in (65521, (1 << 31) - 1, (1 << 32) - 5, (1 << 32) - 1):
        for R in (1, 2, 3, 4, 5, 33, 1000, 20000):
            for v in (m - 2, m - 1):
                cols = R
                ri = np.zeros(R, np.uint32)
                ci = np.arange(R, dtype=np.uint32)
                val = np.full(R, v, np.int64)
                x = np.full(cols, m - 1, np.uint32)
                A = ff.ffspmv_create(2, cols, ri, ci, val, m)
                yd = dev(np.array([m - 1, m - 1], np.uint32))
                ff.ffspmv_apply(A, 1, dev(x), 1, yd)
                assert np.array_equal(host(yd), oracle_mod.apply(2, cols, ri, ci, val, m, x,
                                                                  np.array([m - 1, m - 1]), 1, 1))


@pytest.mark.parametrize("k", [8, 16, 32])
@pytest.mark.parametrize("m", [65521, (1 << 31) - 1, (1 << 31) + 11, (1 << 32) - 5])
def test_block_overflow_adversarial(ff, oracle_mod, cuda, m, k):
    """Block apply (cp.async slice walk) on rows of R maximal products
    (m-1)(m-1) and -1 entries with x = m-1, R crossing every fold of the
    folded u64 accumulator (m = 2^31-1: 4 addends per fold) and the u96
    regime (m with a large 2^32 mod m), all in one SELL band."""
    g = synth.rng(m % 1009 + k)
    rows, cols = 96, 4096
    ri, ci, val = [], [], []
    for r in range(rows):
        R = (r % 48) + 1 if r < 64 else 300 + r
        c = g.choice(cols, size=R, replace=False).astype(np.uint32)
        v = np.where(g.random(R) < 0.3, -1, m - 1).astype(np.int64)
        ri.append(np.full(R, r, np.uint32)); ci.append(c); val.append(v)
    ri, ci, val = np.concatenate(ri), np.concatenate(ci), np.concatenate(val)
    X = np.full((cols, k), m - 1, np.uint32)
    X[::7] = g.integers(0, m, size=(len(X[::7]), k), dtype=np.uint64).astype(np.uint32)
    A = ff.ffspmv_create(rows, cols, ri, ci, val, m, long_row=4096)
    Yd = dev(np.zeros((rows, k), np.uint32))
    ff.ffspmv_apply_block(A, k, 1, dev(X), 0, Yd)
    assert np.array_equal(host(Yd), oracle_mod.apply_block(rows, cols, ri, ci, val, m, X))


@pytest.mark.parametrize("strategy", [2, 3])
@pytest.mark.parametrize("m", [251, 65521, 65536])
def test_panel_overflow_adversarial(ff, oracle_mod, cuda, m, strategy):
    """Panel tiles whose row sums approach 2^32: one dense row per section
    kind (+1, -1 with x = 0, valued m-2 with x = m-1), long enough that the
    lazy Barrett remainders (< 2m) would overflow a u32 and, for m = 65536,
    that even exact residues would (the builder then keeps the rows layout)."""
    for n, v, xv in ((65536, 1, m - 1), (65536, m - 1, 0), (40000, m - 2, m - 1),
                     (65536, m - 2, m - 1)):
        cols = n
        ri = np.zeros(n, np.uint32)
        ci = np.arange(n, dtype=np.uint32)
        val = np.full(n, v, np.int64)
        x = np.full(cols, xv, np.uint32)
        A = ff.ffspmv_create(3, cols, ri, ci, val, m, strategy=strategy)
        y0 = np.array([m - 1, 1, 0], np.uint32)
        yd = dev(y0)
        ff.ffspmv_apply(A, 1, dev(x), 1, yd)
        assert np.array_equal(host(yd), oracle_mod.apply(3, cols, ri, ci, val, m, x, y0, 1, 1))


@pytest.mark.parametrize("strategy", [2, 3])
@pytest.mark.parametrize("m", [3, 65521, 65537])
def test_panel_pipeline_many_tiles(ff, oracle_mod, cuda, m, strategy):
    """Panel schedule edge cases: > 64 tiles per CTA (header-cache reloads,
    tiny 32 x 32 tiles) and tiles with more quads than the register ring
    (> 16384 entries in one tile, the overflow loop)."""
    g = synth.rng(77 + m % 1000)
    for rows, cols, nnz, kw in ((6000, 6000, 60000, dict(panel_rows=32, panel_cols=32)),
                                (20000, 20000, 120000, dict())):
        ri, ci, val = synth.random_coo(g, rows, cols, nnz, m, dup=0.0, big=True)
        A = ff.ffspmv_create(rows, cols, ri, ci, val, m, strategy=strategy, **kw)
        assert A.info()["strategy_apply"] == strategy
        x = synth.uniform(g, cols, m)
        y0 = synth.uniform(g, rows, m)
        yd = dev(y0)
        ff.ffspmv_apply(A, 7, dev(x), 3, yd)
        assert np.array_equal(host(yd), oracle_mod.apply(rows, cols, ri, ci, val, m, x, y0, 7, 3))
        xt = synth.uniform(g, rows, m)
        ytd = dev(np.zeros(cols, np.uint32))
        ff.ffspmv_apply_transpose(A, 1, dev(xt), 0, ytd)
        assert np.array_equal(host(ytd), oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, xt,
                                                                    np.zeros(cols, np.uint32), 1, 0))


def test_determinism_and_streams(ff, cuda):
    import torch
    m = 65521
    M = synth.config_matrix("c2", scale=1 / 16)
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], m)
    g = synth.rng(9)
    x = dev(synth.uniform(g, M["cols"], m))
    outs = []
    for i in range(3):
        s = torch.cuda.Stream()
        y = torch.empty(M["rows"], dtype=torch.int32, device="cuda")
        with torch.cuda.stream(s):
            ff.ffspmv_apply(A, 1, x, 0, y, stream=s)
        s.synchronize()
        outs.append(host(y))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


# ------------------------------------------------------ BASELINE configs ---

def _cfg_vectors(name, M, m):
    g = synth.rng(synth.CONFIGS[name]["vseed"])
    return g


def test_config_c1_full(ff, oracle_mod, cuda):
    M = synth.config_matrix("c1")
    m = M["m"]
    g = _cfg_vectors("c1", M, m)
    x = synth.uniform(g, M["cols"], m)
    y = synth.uniform(g, M["rows"], m)
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], m)
    yd = dev(y)
    ff.ffspmv_apply(A, 1, dev(x), 1, yd)     # y <- A x + y (BASELINE configs[0])
    assert np.array_equal(host(yd), oracle_mod.apply(M["rows"], M["cols"], M["row"], M["col"],
                                                     M["val"], m, x, y, 1, 1))


@pytest.mark.parametrize("strategy", [0, 2])
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_full_apply_transpose(ff, oracle_mod, cuda, name, strategy):
    """Full-size c2 / c3, the exact launch bench.py times (alpha=1, beta=0,
    default strategy), compared on every output element (the oracle finishes
    in seconds); also the PANELS layout."""
    M = synth.config_matrix(name)
    m = M["m"]
    g = _cfg_vectors(name, M, m)
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], m, strategy=strategy)
    x = synth.uniform(g, M["cols"], m)
    import torch
    yd = torch.empty(M["rows"], dtype=torch.int32, device="cuda")
    ff.ffspmv_apply(A, 1, dev(x), 0, yd)
    assert np.array_equal(host(yd), oracle_mod.apply(M["rows"], M["cols"], M["row"], M["col"],
                                                     M["val"], m, x))
    xt = synth.uniform(g, M["rows"], m)
    ytd = torch.empty(M["cols"], dtype=torch.int32, device="cuda")
    ff.ffspmv_apply_transpose(A, 1, dev(xt), 0, ytd)
    assert np.array_equal(host(ytd), oracle_mod.apply_transpose(M["rows"], M["cols"], M["row"],
                                                                M["col"], M["val"], m, xt))


@pytest.mark.parametrize("k", [8, 16, 32])
def test_config_c4_block_full(ff, oracle_mod, cuda, k):
    M = synth.config_matrix("c4")
    m = M["m"]
    g = _cfg_vectors("c4", M, m)
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], m)
    X = synth.uniform(g, (M["cols"], k), m)
    import torch
    Yd = torch.empty((M["rows"], k), dtype=torch.int32, device="cuda")
    ff.ffspmv_apply_block(A, k, 1, dev(X), 0, Yd)
    got = host(Yd)
    # every row for k = 8; a seeded sample of rows (whole row blocks) otherwise
    if k == 8:
        assert np.array_equal(got, oracle_mod.apply_block(M["rows"], M["cols"], M["row"], M["col"],
                                                          M["val"], m, X))
    else:
        rows = np.sort(synth.rng(4).choice(M["rows"], size=4096, replace=False))
        sel = np.isin(M["row"], rows)
        sub = oracle_mod.apply_block(M["rows"], M["cols"], M["row"][sel], M["col"][sel],
                                     M["val"][sel], m, X)
        assert np.array_equal(got[rows], sub[rows])


@pytest.mark.parametrize("m", [2, 3, 251, 65521, 65537, (1 << 31) - 1, (1 << 32) - 1])
def test_transpose_without_store(ff, oracle_mod, cuda, m):
    """no_transpose: A^T x by scattering A's rows (u64 atomics),
    every format and long / split rows; the scratch is cleared between calls."""
    g = synth.rng(606 + m % 1000)
    for opt in (dict(), dict(force_format=2), dict(force_format=3, long_row=4), dict(segregate_pm1=-1)):
        for trial in range(3):
            rows, cols, ri, ci, val = rand_case(g, m, long_rows=(trial == 2))
            A = ff.ffspmv_create(rows, cols, ri, ci, val, m, no_transpose=True, **opt)
            for alpha, beta in ((1, 0), (int(g.integers(0, m)), int(g.integers(0, m)))):
                xt = synth.uniform(g, rows, m)
                yt0 = synth.uniform(g, cols, m)
                want = oracle_mod.apply_transpose(rows, cols, ri, ci, val, m, xt, yt0, alpha, beta)
                ytd = dev(yt0)
                ff.ffspmv_apply_transpose(A, alpha, dev(xt), beta, ytd)
                assert np.array_equal(host(ytd), want), (opt, trial)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_transpose_without_store(ff, oracle_mod, cuda, name):
    M = synth.config_matrix(name)
    m = M["m"]
    g = synth.rng(synth.CONFIGS[name]["vseed"] + 1)
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], m, no_transpose=True)
    import torch
    for rep in range(2):
        xt = synth.uniform(g, M["rows"], m)
        ytd = torch.empty(M["cols"], dtype=torch.int32, device="cuda")
        ff.ffspmv_apply_transpose(A, 1, dev(xt), 0, ytd)
        assert np.array_equal(host(ytd), oracle_mod.apply_transpose(M["rows"], M["cols"], M["row"],
                                                                    M["col"], M["val"], m, xt))

"""GPU parity of the block Wiedemann sequence path (
P:438 §3 step 1, §2.5.2) against the CPU oracle, bit-exact.

Every sequence kernel the dispatcher in csrc/seq.cu can reach is exercised:

* u16 iterate (m <= 65536), tensor-core projection (k % 4 == 0, 4 <= k <= 16,
  ku <= 16): the half-slice kernels k = 8, 16 and the 4-column kernels
  k = 4, 12, with u8 (m <= 256) and u16 stored values;
* the fused scalar step k_seq_step for every KP (k in 1..32: 1, 2, 4, 8, 16,
  32 lanes per row) and KUP (ku <= 16, ku in 17..32), u16 and u32 iterates;
* the unfused path (k or ku > 32);

each on SELL-only, CSR-only and COO_S-only operators and on matrices with
long rows (default threshold and a tiny one, so the out-of-line scalar path
and the shared-memory projection atomics run).  Also: ffspmv_project and
ffspmv_sum_mod directly, chaining compared with the oracle, and the c5
protocol of SURVEY §8(c) (16-term prefix at full size, 8 spot checks, a
scaled c5 over the full L = 2 ceil(N/k) + 2).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

SEQ_MODS = [3, 251, 65521, 65536, 65537, (1 << 31) - 1]
SEQ_K = [2, 4, 5, 8, 12, 16, 24, 32]
SEQ_KU = [1, 3, 16, 24]
FORMATS = {
    "sell": dict(force_format=1),
    "csr": dict(force_format=2),
    "coos": dict(force_format=3),
    "long": dict(),
    "tinylong": dict(long_row=6, band_rows=32),
}


def dev(a):
    import torch
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def _matrix(g, m, fmt):
    if fmt == "long":
        # a few rows longer than the default long_row (512) threshold
        n = 1500
        ri, ci, val = synth.random_coo(g, n, n, 5 * n, m, dup=0.02)
        extra = []
        for L in (600, 900, 1400):
            r = int(g.integers(0, n))
            extra.append((np.full(L, r, np.uint32), g.permutation(n)[:L].astype(np.uint32),
                          g.integers(-m, m, size=L)))
        ri = np.concatenate([ri] + [e[0] for e in extra])
        ci = np.concatenate([ci] + [e[1] for e in extra])
        val = np.concatenate([val] + [e[2] for e in extra])
        return n, ri, ci, val
    n = 180
    nnz = 6 * n
    ri, ci, val = synth.random_coo(g, n, n, nnz, m, dup=0.05)
    if fmt == "coos":
        keep = ri % 3 == 0                      # two rows in three empty
        ri, ci, val = ri[keep], ci[keep], val[keep]
    return n, ri, ci, val


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("m", SEQ_MODS)
def test_sequence_kernel_matrix(ff, oracle_mod, cuda, m, fmt):
    """k x ku grid over every reachable step kernel, U given and U = X."""
    g = synth.rng(7 * m % 100003 + len(fmt))
    n, ri, ci, val = _matrix(g, m, fmt)
    A = ff.ffspmv_create(n, n, ri, ci, val, m, **FORMATS[fmt])
    L = 5
    ks = SEQ_K if fmt != "long" else [2, 4, 8, 12, 16, 32]
    kus = SEQ_KU if fmt != "long" else [3, 16, 24]
    for k in ks:
        X = synth.uniform(g, (n, k), m)
        for ku in kus:
            U = synth.uniform(g, (n, ku), m)
            Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, L, U, want_vout=True)
            S, V = A.sequence(dev(X), L, dev(U), want_vout=True)
            assert np.array_equal(host(S).reshape(Sw.shape), Sw), (k, ku)
            assert np.array_equal(host(V), Vw), (k, ku)
        Sw = oracle_mod.sequence(n, ri, ci, val, m, X, L)
        assert np.array_equal(host(A.sequence(dev(X), L)).reshape(Sw.shape), Sw), (k, "U=X")


@pytest.mark.parametrize("m", [3, 65521, (1 << 31) - 1])
def test_sequence_wide_blocks(ff, oracle_mod, cuda, m):
    """The unfused path (k or ku > 32) and the u32 iterate at the edges."""
    g = synth.rng(m % 9999 + 3)
    n, ri, ci, val = _matrix(g, m, "sell")
    A = ff.ffspmv_create(n, n, ri, ci, val, m)
    for k, ku in ((33, 1), (1, 33), (40, 40), (64, 7)):
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, ku), m)
        Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, 4, U, want_vout=True)
        S, V = A.sequence(dev(X), 4, dev(U), want_vout=True)
        assert np.array_equal(host(S).reshape(Sw.shape), Sw), (k, ku)
        assert np.array_equal(host(V), Vw), (k, ku)


@pytest.mark.parametrize("m", [3, 251, 65521, 65537, (1 << 31) - 1])
def test_sequence_chaining_vs_oracle(ff, oracle_mod, cuda, m):
    """sequence(L1) then sequence(L2) from V_out == the oracle's L1 + L2 terms
    (R14: V_out = A^L X makes chaining exact)."""
    g = synth.rng(5 + m % 1000)
    n = 300
    ri, ci, val = synth.random_coo(g, n, n, 2000, m)
    A = ff.ffspmv_create(n, n, ri, ci, val, m)
    for k, ku in ((4, 3), (8, 8), (12, 16), (16, 16), (5, 2)):
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, ku), m)
        Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, 9, U, want_vout=True)
        S1, V1 = A.sequence(dev(X), 4, dev(U), want_vout=True)
        S2, V2 = A.sequence(V1, 5, dev(U), want_vout=True)
        assert np.array_equal(np.concatenate([host(S1), host(S2)]).reshape(Sw.shape), Sw), (k, ku)
        assert np.array_equal(host(V2), Vw), (k, ku)


@pytest.mark.parametrize("m", [65521, (1 << 31) - 1, (1 << 32) - 5])
def test_project_parity(ff, oracle_mod, cuda, m):
    """ffspmv_project (k_project_t register tiles, vec and non-vec staging,
    the generic k_project for k or ku > 64, the Acc96 'wide' branch for
    m > 2^16) against the oracle's S_0 = U^T V; rows not a multiple of the
    tile, and 16-byte-misaligned V / U views."""
    import torch
    g = synth.rng(m % 777)
    z = np.zeros(0, np.uint32)
    for n in (1, 63, 1000, 70001):
        A = ff.ffspmv_create(n, n, z, z, np.zeros(0, np.int64), m)
        for k, ku in ((1, 1), (3, 4), (4, 3), (16, 16), (33, 64), (64, 65), (100, 3)):
            V = synth.uniform(g, (n, k), m)
            U = synth.uniform(g, (n, ku), m)
            want = oracle_mod.sequence(n, z, z, np.zeros(0, np.int64), m, V, 1, U)[0]
            ws = torch.empty(max(1, ff.ffspmv_workspace_size(A, ff.OP_PROJECT, k, ku)),
                             dtype=torch.uint8, device="cuda")
            S = dev(np.zeros((ku, k), np.uint32))
            ff.ffspmv_project(A, k, dev(V), ku, dev(U), S, ws)
            assert np.array_equal(host(S), want), (n, k, ku)
            # misaligned: views one element into a larger buffer
            Vb = dev(np.concatenate([[0], V.ravel()]))
            Ub = dev(np.concatenate([[0], U.ravel()]))
            S2 = dev(np.zeros((ku, k), np.uint32))
            ff.ffspmv_project(A, k, Vb[1:].view(n, k), ku, Ub[1:].view(n, ku), S2, ws)
            assert np.array_equal(host(S2), want), (n, k, ku, "misaligned")


@pytest.mark.parametrize("m", [2, 65521, (1 << 32) - 1])
def test_sum_mod_parity(ff, cuda, m):
    g = synth.rng(m % 313)
    z = np.zeros(0, np.uint32)
    A = ff.ffspmv_create(1, 1, z, z, np.zeros(0, np.int64), m)
    for count, nparts in ((1, 1), (7, 3), (1000, 8), (4097, 1)):
        parts = synth.uniform(g, (nparts, count), m)
        out = dev(np.zeros(count, np.uint32))
        ff.ffspmv_sum_mod(A, count, nparts, dev(parts), out)
        want = (parts.astype(object).sum(axis=0) % m).astype(np.uint32)
        assert np.array_equal(host(out), want)


def test_sequence_dim_limit(ff, cuda):
    """n * k >= 2^32 is refused (32-bit iterate offsets) before any launch."""
    import torch
    z = np.zeros(0, np.uint32)
    n, k = 1 << 22, 1024
    A = ff.ffspmv_create(n, n, z, z, np.zeros(0, np.int64), 65521, no_transpose=True)
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_sequence(A, k, dev(np.zeros(16, np.uint32)), 1, dev(np.zeros(16, np.uint32)), 1,
                           dev(np.zeros(256, np.uint32)), None,
                           torch.empty(16, dtype=torch.uint8, device="cuda"))
    assert e.value.status == ff.ERR_DIM


# ------------------------------------------------------------ c5 protocol ---

def test_config_c5_prefix_and_spot_checks(ff, oracle_mod, cuda):
    """c5 at full size (N = 2^21, k = ku = 16, m = 65521), SURVEY §8(c):
    the first 16 terms S_0..S_15 and V_16 against the oracle; then 8 spot
    checks: the device run continues to 8 seeded depths j, V_j is downloaded
    and the oracle's S_j, S_{j+1} (from V_j) are compared with the device's."""
    M = synth.config_matrix("c5")
    m, n, k = M["m"], M["rows"], 16
    g = synth.rng(synth.CONFIGS["c5"]["vseed"])
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, k), m)
    A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], m, no_transpose=True)
    Ud = dev(U)
    S, V = A.sequence(dev(X), 16, Ud, want_vout=True)
    Sw, Vw = oracle_mod.sequence(n, M["row"], M["col"], M["val"], m, X, 16, U, want_vout=True)
    assert np.array_equal(host(S).reshape(Sw.shape), Sw)
    assert np.array_equal(host(V), Vw)
    depth = 16
    for j in sorted(synth.rng(55).choice(np.arange(20, 400), size=8, replace=False)):
        _, V = A.sequence(V, int(j) - depth, Ud, want_vout=True)       # V = V_j
        depth = int(j)
        S_dev, V_next = A.sequence(V, 2, Ud, want_vout=True)           # S_j, S_{j+1}
        Sw2, Vw2 = oracle_mod.sequence(n, M["row"], M["col"], M["val"], m, host(V), 2, U,
                                       want_vout=True)
        assert np.array_equal(host(S_dev).reshape(Sw2.shape), Sw2), j
        assert np.array_equal(host(V_next), Vw2), j


def test_config_c5_scaled_full_length(ff, oracle_mod, cuda):
    """Scaled c5 (N = 2^14, same recipe) over the full L = 2 ceil(N/k) + 2 =
    2050 steps, U given, compared term by term, plus V_L."""
    M = synth.config_matrix("c5", scale=1 / 128)
    m, n, k = M["m"], M["rows"], 16
    assert n == 1 << 14
    g = synth.rng(2005)
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, k), m)
    L = 2 * ((n + k - 1) // k) + 2
    A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], m)
    S, V = A.sequence(dev(X), L, dev(U), want_vout=True)
    Sw, Vw = oracle_mod.sequence(n, M["row"], M["col"], M["val"], m, X, L, U, want_vout=True)
    assert np.array_equal(host(S).reshape(Sw.shape), Sw)
    assert np.array_equal(host(V), Vw)


def test_c3_square_sequence_u8_iterate(ff, oracle_mod, cuda):
    """m = 3 (every nonzero +-1): the iterate is stored as u8 (SURVEY a-8,
    P:631).  A square GL7d-shaped matrix at full size (1,911,130 rows, the
    c3 recipe with cols = rows): the first 4 terms and V_4 against the
    oracle; a scaled one over the full L = 2 ceil(N/k) + 2."""
    M = synth.config_matrix("c3", square=True)
    m, n, k = M["m"], M["rows"], 16
    A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], m, no_transpose=True)
    assert A.info()["iterate_bytes"] == 1
    g = synth.rng(2033)
    X = synth.uniform(g, (n, k), m)
    U = synth.uniform(g, (n, k), m)
    S, V = A.sequence(dev(X), 4, dev(U), want_vout=True)
    rs, cs, vs = oracle_mod.sort_triples(M["row"], M["col"], M["val"])
    Sw, Vw = oracle_mod.sequence_mt(n, rs, cs, vs, m, X, 4, U, want_vout=True)
    assert np.array_equal(host(S).reshape(Sw.shape), Sw)
    assert np.array_equal(host(V), Vw)
    Ms = synth.config_matrix("c3", scale=1 / 256, square=True)
    ns = Ms["rows"]
    Xs = synth.uniform(g, (ns, k), m)
    L = 2 * ((ns + k - 1) // k) + 2
    As = ff.ffspmv_create(ns, ns, Ms["row"], Ms["col"], Ms["val"], m)
    Ss = As.sequence(dev(Xs), L)
    assert np.array_equal(host(Ss).reshape(L, k, k), oracle_mod.sequence(ns, Ms["row"], Ms["col"], Ms["val"], m, Xs, L))

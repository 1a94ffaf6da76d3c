"""CPU tests of the C ABI library: it loads, exports every declared symbol,
validates arguments, and its host format builder packs
exactly A -- the triples rebuilt from every slot of every piece sum back to
the canonical matrix ("A is split into smaller submatrices")."""
import os
import re
from collections import defaultdict

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1004_3719_b200 import build
    build.build()
    import paper_1004_3719_b200 as ff
    ff.load()
    return ff


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ffspmv.h")).read()
    return sorted(set(re.findall(r"FFSPMV_API[^;]*?\b(ffspmv_\w+)\s*\(", txt, re.S)))


def test_exports_every_declared_symbol(lib):
    declared = header_symbols()
    assert len(declared) >= 14
    L = lib.load()
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(lib.EXPORTS) == declared
    info = lib.ffspmv_analyze(1, 1, np.zeros(1, np.uint32), np.zeros(1, np.uint32),
                              np.ones(1, np.int64), 7)
    import ctypes
    assert info["struct_size"] == ctypes.sizeof(lib.ffspmv_info)
    assert lib.ffspmv_version() >= 100
    assert lib.ffspmv_status_string(lib.ERR_NONSQUARE) == "FFSPMV_ERR_NONSQUARE"


def canonical(rows, cols, ri, ci, val, m, transpose=False):
    acc = defaultdict(int)
    for r, c, v in zip(ri.tolist(), ci.tolist(), val.tolist()):
        key = (c, r) if transpose else (r, c)
        acc[key] = (acc[key] + int(v)) % m
    return {k: v for k, v in acc.items() if v}


def rebuilt(rec):
    rr, rc, rv = rec
    out = {}
    for r, c, v in zip(rr.tolist(), rc.tolist(), rv.tolist()):
        assert (r, c) not in out, "entry packed twice"
        out[(r, c)] = v
    return out


OPTION_SETS = [
    dict(),
    dict(force_format=1), dict(force_format=2), dict(force_format=3),
    dict(segregate_pm1=-1), dict(segregate_pm1=1, force_format=3),
    dict(band_rows=32, long_row=4), dict(band_rows=64, long_row=8, force_format=2),
    dict(force_acc_bits=96), dict(force_acc_bits=64, force_format=3),
    dict(strategy=2), dict(strategy=2, panel_rows=32, panel_cols=32),
    dict(strategy=2, panel_rows=64, panel_cols=96, segregate_pm1=-1),
    dict(strategy=3), dict(strategy=3, panel_rows=32, panel_cols=64),
    dict(strategy=3, panel_rows=8, panel_cols=64, segregate_pm1=-1, panel_xbits=32),
    dict(strategy=3, panel_rows=12, panel_cols=128, panel_xbits=16),
]


@pytest.mark.parametrize("m", [2, 3, 251, 65521, 65537, (1 << 31) - 1, (1 << 32) - 1])
@pytest.mark.parametrize("opt", range(len(OPTION_SETS)))
def test_pack_reconstructs_canonical(lib, m, opt):
    g = synth.rng(1000 + opt * 31 + m % 1000)
    kw = OPTION_SETS[opt]
    for trial in range(3):
        rows, cols = int(g.integers(0, 150)), int(g.integers(0, 150))
        nnz = int(g.integers(0, 4 * max(rows, 1)))
        ri, ci, val = synth.random_coo(g, rows, cols, nnz, m, dup=0.1, big=True)
        if rows and cols and trial == 2:   # a few long rows for the tail
            extra = g.integers(0, cols, size=300).astype(np.uint32)
            ri = np.concatenate([ri, np.full(300, rows - 1, np.uint32)])
            ci = np.concatenate([ci, extra])
            val = np.concatenate([val, g.integers(-m, m, size=300)])
        want = canonical(rows, cols, ri, ci, val, m)
        for tr in (False, True):
            info, rec = lib.ffspmv_analyze(rows, cols, ri, ci, val, m, transpose=tr,
                                           reconstruct=True, **kw)
            got = rebuilt(rec)
            exp = canonical(rows, cols, ri, ci, val, m, transpose=tr)
            assert got == exp
        assert info["nnz"] == len(want)
        assert info["nnz_pm1"] + info["nnz_valued"] == len(want)
        pm = sum(1 for v in want.values() if v == 1 or (m > 2 and v == m - 1))
        if kw.get("segregate_pm1") == -1:
            assert info["nnz_pm1"] == 0
        elif kw.get("segregate_pm1") == 1:
            assert info["nnz_pm1"] == pm
        assert info["has_transpose"] == 1


def test_chooser_and_regimes(lib):
    m = 65521
    n = 4096
    # constant row length 8, valued entries 2..m-2 -> SELL bands, u64
    ri = np.repeat(np.arange(n, dtype=np.uint32), 8)
    ci = (np.arange(n * 8, dtype=np.uint32) * 7919) % n
    val = np.full(n * 8, 5, np.int64)
    info = lib.ffspmv_analyze(n, n, ri, ci, val, m)
    assert info["bands_sell"] == info["bands"] and info["slices"] == n // 32
    assert info["padded_slots"] == n * 8          # uniform rows: no padding
    assert info["acc_bits_max"] == 64
    # m = 65521: one valued product (<= 65520^2 < 2^32) fits u32
    info = lib.ffspmv_analyze(n, n, ri[::8], ci[::8], val[::8], m)
    assert info["acc_bits_max"] == 32
    # m = 2^31 - 1: five products of (m-2)*(m-1) exceed 2^64 -> u96; four do not
    P = (1 << 31) - 1
    for r, bits in ((4, 64), (5, 96)):
        info = lib.ffspmv_analyze(1, 8, np.zeros(r, np.uint32), np.arange(r, dtype=np.uint32),
                                  np.full(r, P - 2, np.int64), P)
        assert info["acc_bits_max"] == bits
    # m = 3, all entries +-1 -> index-only stream, u32 adds
    ri2, ci2, v2 = synth.random_coo(synth.rng(3), 500, 500, 5000, 3, pm=1.0)
    info = lib.ffspmv_analyze(500, 500, ri2, ci2, v2, 3)
    assert info["nnz_valued"] == 0 and info["acc_bits_max"] == 32 and info["value_bytes"] == 1
    # long rows go to the tail; rows > 2^14 entries are split
    cols = 40000
    ri3 = np.zeros(cols, np.uint32)
    ci3 = np.arange(cols, dtype=np.uint32)
    info = lib.ffspmv_analyze(2, cols, ri3, ci3, np.full(cols, 7, np.int64), m)
    assert info["long_rows"] == 1 and info["split_rows"] == 1
    # forced formats are honoured band by band
    for fmt, key in ((1, "bands_sell"), (2, "bands_csr"), (3, "bands_coos")):
        info = lib.ffspmv_analyze(n, n, ri, ci, val, m, force_format=fmt, band_rows=1024)
        assert info[key] == info["bands"] == 4


def test_panel_strategy_choice(lib):
    import synth as sy
    M = sy.config_matrix("c2", scale=1 / 2)        # random columns, 524k x 524k
    info = lib.ffspmv_analyze(M["rows"], M["cols"], M["row"], M["col"], M["val"], M["m"])
    assert info["gather_locality"] > 0.7
    assert info["strategy_apply"] == lib.STRATEGY_PANELS == info["strategy_transpose"]
    assert info["panels"] == 8 and info["panel_bands"] == -(-M["rows"] // 8160)
    # m = 3: RUNS, x staged at 2 bits -> one panel; ~6.7 entries per row
    # (a third of the values vanish mod 3) -> 256-row units (>= 1024 entries)
    info = lib.ffspmv_analyze(M["rows"], M["cols"], M["row"], M["col"], M["val"], 3)
    assert info["strategy_apply"] == lib.STRATEGY_RUNS and info["panel_xbits"] == 2
    assert info["panels"] == 1 and info["panel_bands"] == M["rows"] // 256
    # banded matrix: columns local -> rows layout
    n = 1 << 19
    ri = np.repeat(np.arange(n, dtype=np.uint32), 4)
    ci = (ri.astype(np.int64) + np.tile(np.arange(4), n)) % n
    info = lib.ffspmv_analyze(n, n, ri, ci.astype(np.uint32), np.full(4 * n, 3, np.int64), 65521)
    assert info["gather_locality"] < 0.2 and info["strategy_apply"] == lib.STRATEGY_ROWS


def test_algorithmic_bytes(lib):
    m = 65521
    ri, ci, val = synth.random_coo(synth.rng(5), 300, 200, 3000, m, pm=0.3, dup=0.0)
    info = lib.ffspmv_analyze(300, 200, ri, ci, val, m)
    assert info["alg_bytes_apply"] == 4 * info["nnz_pm1"] + 6 * info["nnz_valued"] + 4 * 200 + 4 * 300


@pytest.mark.parametrize("case", ["modulus", "index", "dim", "options", "null"])
def test_argument_errors(lib, case):
    z = np.zeros(1, np.uint32)
    one = np.ones(1, np.int64)
    with pytest.raises(lib.FFSPMVError) as e:
        if case == "modulus":
            lib.ffspmv_analyze(1, 1, z, z, one, 1)
        elif case == "index":
            lib.ffspmv_analyze(1, 1, z + 1, z, one, 7)
        elif case == "dim":
            lib.ffspmv_analyze(1 << 31, 1, z, z, one, 7)
        elif case == "options":
            lib.ffspmv_analyze(1, 1, z, z, one, 7, band_rows=33)
        else:
            lib.ffspmv_analyze(1, 1, z[:0], z[:0], one[:0], 7, force_acc_bits=48)
    want = {"modulus": lib.ERR_MODULUS, "index": lib.ERR_INDEX, "dim": lib.ERR_DIM,
            "options": lib.ERR_INVALID_ARG, "null": lib.ERR_INVALID_ARG}[case]
    assert e.value.status == want
    assert lib.ffspmv_last_error()


def test_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    z = np.zeros(1, np.uint32)
    with pytest.raises(lib.FFSPMVError) as e:
        lib.ffspmv_create(1, 1, z, z, np.ones(1, np.int64), 7)
    assert e.value.status == lib.ERR_CUDA

"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module only *draws* inputs (triples, vectors, blocks).  It holds none of
the method's arithmetic: no residues, no products, no reductions.  Both the
tests/bench (which feed ``oracle``) and the product path (which feeds the C
ABI) take their inputs from here, so the two sides see identical data.

Recipes follow DESIGN.md §"Input recipe", shaped like the
paper's sparse-integer-collection workloads (Table 1):

* c1  2000 x 2000, Poisson(8) row lengths, 30% +-1, mod 65521, 1% duplicates
* c2  2^20 x 2^20, Poisson(10), 30% +-1, mod 65521
* c3  1,911,130 x 1,955,309, skewed "c + r" rows:
      max(1, round(LogNormal(2.725, 0.7))) capped at 4096, 0.01% rows forced
      to 1000-4000; values +-1 w.p. .96, +-2 w.p. .03, +-3 w.p. .01; mod 3
* c4  2^20 x 2^20, Poisson(10), 30% +-1, mod 2^31-1, k in {8, 16, 32}
* c5  2^21 x 2^21, Poisson(10), 30% +-1, mod 65521, k = ku = 16

All generators use numpy ``Generator(PCG64(seed))``; the matrix seed of
config c is 1000+c and its vector seed 2000+c.
"""
from __future__ import annotations

import numpy as np

P31 = (1 << 31) - 1

CONFIGS = {
    "c1": dict(rows=2000, cols=2000, m=65521, lengths=("poisson", 8.0), pm=0.30, dup=0.01,
               seed=1001, vseed=2001),
    "c2": dict(rows=1 << 20, cols=1 << 20, m=65521, lengths=("poisson", 10.0), pm=0.30, dup=0.0,
               seed=1002, vseed=2002),
    "c3": dict(rows=1911130, cols=1955309, m=3, lengths=("lognormal", 2.725, 0.7, 4096), pm=None,
               dup=0.0, seed=1003, vseed=2003),
    "c4": dict(rows=1 << 20, cols=1 << 20, m=P31, lengths=("poisson", 10.0), pm=0.30, dup=0.0,
               seed=1004, vseed=2004, k=(8, 16, 32)),
    "c5": dict(rows=1 << 21, cols=1 << 21, m=65521, lengths=("poisson", 10.0), pm=0.30, dup=0.0,
               seed=1005, vseed=2005, k=16),
}


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _row_lengths(g, rows, cols, spec):
    kind = spec[0]
    if kind == "poisson":
        r = g.poisson(spec[1], size=rows)
    elif kind == "lognormal":
        mu, sigma, cap = spec[1], spec[2], spec[3]
        r = np.maximum(1, np.rint(g.lognormal(mu, sigma, size=rows))).astype(np.int64)
        r = np.minimum(r, cap)
        nlong = max(1, rows // 10000)                      # 0.01% long rows
        idx = g.choice(rows, size=nlong, replace=False)
        r[idx] = g.integers(1000, 4001, size=nlong)
    elif kind == "fixed":
        r = np.full(rows, spec[1])
    else:
        raise ValueError(kind)
    return np.minimum(r.astype(np.int64), cols)


def _distinct_columns(g, lengths, cols):
    """Uniform columns, distinct within a row, sorted by (row, col)."""
    rows = lengths.size
    ri = np.repeat(np.arange(rows, dtype=np.int64), lengths)
    ci = g.integers(0, cols, size=ri.size, dtype=np.int64)
    key = np.sort(ri * cols + ci)
    keep = np.ones(key.size, bool)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    return (key // cols).astype(np.uint32), (key % cols).astype(np.uint32)


def _values_mixed(g, n, m, pm):
    """pm fraction of +-1 (half +1, half written as -1), the rest uniform in
    [2, m-2] (m >= 5) -- the "mixed +-1 and random values" of configs 1,2,4,5."""
    v = np.empty(n, np.int64)
    u = g.random(n)
    is_pm = u < pm
    plus = g.random(n) < 0.5
    v[is_pm & plus] = 1
    v[is_pm & ~plus] = -1
    nv = int((~is_pm).sum())
    if m >= 5:
        v[~is_pm] = g.integers(2, m - 1, size=nv, dtype=np.int64)
    else:
        v[~is_pm] = g.integers(0, m, size=nv, dtype=np.int64)
    return v


def _values_gl7d(g, n):
    """c3: +-1 w.p. 0.96, +-2 w.p. 0.03, +-3 w.p. 0.01 (integers; mod 3 every
    nonzero is +-1 and the +-3 entries vanish)."""
    u = g.random(n)
    mag = np.where(u < 0.96, 1, np.where(u < 0.99, 2, 3)).astype(np.int64)
    sign = np.where(g.random(n) < 0.5, 1, -1).astype(np.int64)
    return mag * sign


def config_matrix(name: str, scale: float = 1.0, square: bool = False):
    """Triples of config ``name``; ``scale`` < 1 shrinks rows and cols
    (same recipe, smaller shape) for oracle-sized parity cases; ``square``
    sets cols = rows (e.g. a GL7d-shaped square matrix for the sequence)."""
    c = CONFIGS[name]
    rows = max(1, int(round(c["rows"] * scale)))
    cols = rows if square else max(1, int(round(c["cols"] * scale)))
    g = rng(c["seed"])
    lengths = _row_lengths(g, rows, cols, c["lengths"])
    ri, ci = _distinct_columns(g, lengths, cols)
    if c["pm"] is None:
        val = _values_gl7d(g, ri.size)
    else:
        val = _values_mixed(g, ri.size, c["m"], c["pm"])
    if c["dup"]:
        nd = int(round(ri.size * c["dup"]))
        pick = g.choice(ri.size, size=nd, replace=False)
        ri = np.concatenate([ri, ri[pick]])
        ci = np.concatenate([ci, ci[pick]])
        val = np.concatenate([val, _values_mixed(g, nd, c["m"], c["pm"])])
    return dict(name=name, rows=rows, cols=cols, m=c["m"], row=ri, col=ci, val=val)


def uniform(g, shape, m):
    """Canonical uniform residues in [0, m) as uint32."""
    return g.integers(0, m, size=shape, dtype=np.uint64).astype(np.uint32)


def random_coo(g, rows, cols, nnz, m, *, pm=0.3, dup=0.0, negative=True, shuffle=True,
               big=False):
    """Small random test matrix.  Values: pm fraction +-1, otherwise uniform
    residues, optionally negative or >= m (``big``) to exercise input
    canonicalisation.  May contain duplicates and explicit zeros."""
    nnz = int(nnz)
    ri = g.integers(0, max(rows, 1), size=nnz, dtype=np.int64).astype(np.uint32)
    ci = g.integers(0, max(cols, 1), size=nnz, dtype=np.int64).astype(np.uint32)
    if rows == 0 or cols == 0:
        ri = ri[:0]; ci = ci[:0]; nnz = 0
    v = g.integers(0, m, size=nnz, dtype=np.uint64).astype(np.int64)
    u = g.random(nnz)
    v[u < pm / 2] = 1
    v[(u >= pm / 2) & (u < pm)] = -1 if negative else m - 1
    if negative:
        flip = g.random(nnz) < 0.2
        v[flip] = v[flip] - m
    if big:
        lift = g.random(nnz) < 0.2
        v[lift] = v[lift] + m * g.integers(1, 1 << 20, size=int(lift.sum()))
    if dup and nnz:
        nd = max(1, int(nnz * dup))
        pick = g.integers(0, nnz, size=nd)
        ri = np.concatenate([ri, ri[pick]])
        ci = np.concatenate([ci, ci[pick]])
        v = np.concatenate([v, g.integers(-m, m, size=nd, dtype=np.int64)])
    if shuffle and ri.size:
        p = g.permutation(ri.size)
        ri, ci, v = ri[p], ci[p], v[p]
    return ri.astype(np.uint32), ci.astype(np.uint32), v.astype(np.int64)


MODULI = [2, 3, 27, 251, 256, 257, 65521, 65536, 65537, (1 << 20) + 7, P31, (1 << 32) - 5,
          (1 << 32) - 1]

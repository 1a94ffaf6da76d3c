"""Multi-GPU drivers: one process per GPU, torch.distributed for
the plumbing (NCCL over NVLink on the GPU box; gloo in the CPU tests).

The partitioning is host logic; every product runs in the C ABI kernels of
the calling rank.  Two modes of the block Wiedemann sequence:

* ``sequence_columns``  -- the paper's "ship independent set of vector blocks
  of V to different cores ... then gather the results": rank r
  owns columns [c_r, c_{r+1}) of X, iterates them with its own copy of A and
  no per-step communication; the S column blocks are all-gathered once.
* ``sequence_rows``     -- "let the SpMV library take care of the iteration"
   across GPUs: rank r owns the rows [r_r, r_{r+1}) of A
  (nnz-balanced bands); each step computes its band of V_{t+1} = A V_t,
  all-gathers the bands into the full iterate, and accumulates its band's
  projection U_band^T V_band; the L projections are summed over ranks once.

Single applies shard by rows with no exchange (``row_bands``).  Every result
is identical to the 1-GPU result (R20).

``backend`` objects supply the per-rank compute, so the same host logic runs
on the CUDA path (``CudaBackend``) and, in the CPU tests, on any exact
reference implementation.
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------- partitioning ---

def row_bands(row_idx, rows: int, world: int) -> np.ndarray:
    """nnz-balanced contiguous row bands: boundaries b[0]=0 <= ... <= b[world]=rows."""
    counts = np.bincount(np.asarray(row_idx, dtype=np.int64), minlength=rows)[:rows]
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = cum[-1]
    b = [0]
    for r in range(1, world):
        target = total * r / world
        b.append(int(np.searchsorted(cum, target, side="left")))
    b.append(rows)
    b = np.maximum.accumulate(np.clip(np.array(b, dtype=np.int64), 0, rows))
    return b


def column_shards(k: int, world: int) -> np.ndarray:
    """Contiguous column blocks of X: boundaries c[0]=0 <= ... <= c[world]=k."""
    return np.array([(k * r) // world for r in range(world + 1)], dtype=np.int64)


def band_triples(row_idx, col_idx, vals, lo: int, hi: int):
    """The triples of rows [lo, hi), re-based to row 0."""
    ri = np.asarray(row_idx)
    sel = (ri >= lo) & (ri < hi)
    return ((ri[sel] - lo).astype(np.uint32), np.asarray(col_idx)[sel].astype(np.uint32),
            np.asarray(vals)[sel].astype(np.int64))


# -------------------------------------------------------------- backends ---

class CudaBackend:
    """Per-rank compute through the C ABI on the rank's GPU."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = torch.device(device)

    def tensor(self, a):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        return self.torch.from_numpy(a.view(np.int32)).to(self.device)

    def empty(self, shape):
        return self.torch.empty(shape, dtype=self.torch.int32, device=self.device)

    def to_numpy(self, t):
        return t.cpu().numpy().view(np.uint32)

    def create(self, rows, cols, ri, ci, v, m):
        import paper_1004_3719_b200 as ff
        return ff.ffspmv_create(rows, cols, ri, ci, v, m, no_transpose=True)

    def sequence(self, A, X, L, U):
        return A.sequence(X, L, U)

    def apply_block(self, A, X, out):
        import paper_1004_3719_b200 as ff
        return ff.ffspmv_apply_block(A, X.shape[1], 1, X, 0, out)

    def project(self, A, V, U, m):
        """S = U^T V mod m for one band: a length-1 sequence on the band's
        iterate (identity product not needed: S_0 = U^T V)."""
        raise NotImplementedError


def _all_gather_rows(group, band_tensor, counts, torch):
    """All-gather row bands of different heights (padded to the max height)."""
    import torch.distributed as dist
    world = len(counts)
    hmax = int(max(counts))
    k = band_tensor.shape[1]
    pad = torch.zeros((hmax, k), dtype=band_tensor.dtype, device=band_tensor.device)
    pad[: band_tensor.shape[0]] = band_tensor
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([out[r][: counts[r]] for r in range(world)], dim=0)


# ----------------------------------------------------------------- modes ---

def sequence_columns(n, row_idx, col_idx, vals, m, X, L, U, backend, group=None):
    """Column-sharded sequence: returns the full S (L x ku x k), identical on
    every rank.  X, U are host arrays (n x k, n x ku)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    X = np.asarray(X, dtype=np.uint32)
    k = X.shape[1]
    U = X if U is None else np.asarray(U, dtype=np.uint32)
    ku = U.shape[1]
    c = column_shards(k, world)
    A = backend.create(n, n, row_idx, col_idx, vals, m)
    lo, hi = int(c[rank]), int(c[rank + 1])
    if hi > lo:
        S_loc = backend.to_numpy(backend.sequence(A, backend.tensor(X[:, lo:hi]), L,
                                                  backend.tensor(U))).reshape(L, ku, hi - lo)
    else:
        S_loc = np.zeros((L, ku, 0), np.uint32)
    # gather the column blocks (padded to the widest block)
    wmax = int(max(c[1:] - c[:-1]))
    buf = np.zeros((L, ku, wmax), np.uint32)
    buf[:, :, : hi - lo] = S_loc
    t = torch.from_numpy(buf.view(np.int32).copy())
    dev = getattr(backend, "device", torch.device("cpu"))
    t = t.to(dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    S = np.zeros((L, ku, k), np.uint32)
    for r in range(world):
        w = int(c[r + 1] - c[r])
        S[:, :, c[r]:c[r + 1]] = parts[r].cpu().numpy().view(np.uint32)[:, :, :w]
    return S


def sequence_rows(n, row_idx, col_idx, vals, m, X, L, U, backend, group=None, want_vout=False):
    """Row-banded sequence with an all-gather of the iterate every step.
    Returns S (L x ku x k) on every rank (and V_L if asked)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    X = np.asarray(X, dtype=np.uint32)
    k = X.shape[1]
    U = X if U is None else np.asarray(U, dtype=np.uint32)
    ku = U.shape[1]
    b = row_bands(row_idx, n, world)
    counts = [int(b[r + 1] - b[r]) for r in range(world)]
    lo, hi = int(b[rank]), int(b[rank + 1])
    ri, ci, v = band_triples(row_idx, col_idx, vals, lo, hi)
    A_band = backend.create(hi - lo, n, ri, ci, v, m)
    V = backend.tensor(X)                       # full iterate, replicated
    U_band = U[lo:hi].astype(np.uint64)
    S_part = np.zeros((L, ku, k), np.uint64)    # this band's projections (exact, < n * m^2)
    for t in range(L):
        Vb = backend.to_numpy(V)[lo:hi].astype(np.uint64)
        # projection of this band, exact then reduced (object-free: per column)
        S_part[t] = ((U_band.T.astype(object) @ Vb.astype(object)) % m).astype(np.uint64)
        if t + 1 < L or want_vout:
            out = backend.empty((hi - lo, k))
            backend.apply_block(A_band, V, out)
            V = _all_gather_rows(group, out, counts, torch)
    # sum the band projections over ranks (each < m, world * m < 2^63)
    tot = torch.from_numpy(S_part.astype(np.int64))
    dist.all_reduce(tot, group=group)
    S = (tot.numpy() % m).astype(np.uint32)
    if want_vout:
        return S, backend.to_numpy(V)
    return S

"""Multi-GPU drivers: one process per GPU, torch.distributed for
the plumbing (NCCL over NVLink on the GPU box; gloo in the CPU tests).

The partitioning is host logic; every product runs in the C ABI kernels of
the calling rank (``CudaBackend``).  Two modes of the block Wiedemann sequence
(P:457-463):

* ``sequence_columns`` -- the paper's "ship independent set of vector blocks
  of V to different cores ... then gather the results": rank r
  owns columns [c_r, c_{r+1}) of X, iterates them with its own copy of A and
  no per-step communication; the S column blocks are all-gathered once.
* ``sequence_rows``    -- "let the SpMV library take care of the iteration"
   across GPUs: rank r owns the rows [b_r, b_{r+1}) of A
  (nnz-balanced bands); each step computes its band of V_{t+1} = A V_t,
  all-gathers the bands into the full iterate (the per-step exchange over
  NVLink), and projects its band; the L band projections are combined once.

Single applies shard by rows with no exchange (``row_bands``).  Every result
is identical to the 1-GPU result (R20).

The backend supplies the per-rank compute.  ``CudaBackend`` is the product
path; the CPU tests substitute an exact reference backend to check the host
logic (partitioning, gathers, assembly) under gloo with world_size 2.
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
        b.append(int(np.searchsorted(cum, total * r / world, side="left")))
    b.append(rows)
    return np.maximum.accumulate(np.clip(np.array(b, dtype=np.int64), 0, rows))


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

    def project(self, A, V, U, out):
        import paper_1004_3719_b200 as ff
        k, ku = V.shape[1], U.shape[1]
        ws = self.torch.empty(max(1, ff.ffspmv_workspace_size(A, ff.OP_PROJECT, k, ku)),
                              dtype=self.torch.uint8, device=self.device)
        return ff.ffspmv_project(A, k, V, ku, U, out, ws)

    def sum_mod(self, A, parts, out):
        import paper_1004_3719_b200 as ff
        return ff.ffspmv_sum_mod(A, out.numel(), parts.shape[0], parts, out)


def _all_gather_rows(group, band_tensor, counts):
    """All-gather row bands of different heights (padded to the max height)."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    hmax = max(1, int(max(counts)))
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
    wmax = max(1, int(max(c[1:] - c[:-1])))
    dev = getattr(backend, "device", torch.device("cpu"))
    buf = torch.zeros((L, ku, wmax), dtype=torch.int32, device=dev)
    if hi > lo and L:
        S_loc = backend.sequence(A, backend.tensor(X[:, lo:hi]), L, backend.tensor(U))
        buf[:, :, : hi - lo] = S_loc.reshape(L, ku, hi - lo)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
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
    V = backend.tensor(X)                               # full iterate, replicated
    U_band = backend.tensor(U[lo:hi])
    S_band = backend.empty((L, ku, k))                  # this band's projections (residues)
    for t in range(L):
        backend.project(A_band, V[lo:hi], U_band, S_band[t])
        if t + 1 < L or want_vout:
            out = backend.empty((hi - lo, k))
            backend.apply_block(A_band, V, out)
            V = _all_gather_rows(group, out, counts)    # the per-step exchange
    parts = [torch.empty_like(S_band) for _ in range(world)]
    dist.all_gather(parts, S_band, group=group)
    S = backend.empty((L, ku, k))
    backend.sum_mod(A_band, torch.stack(parts), S)      # sum_r S_r mod m on device
    S = backend.to_numpy(S)
    if want_vout:
        return S, backend.to_numpy(V)
    return S


def grid_shape(world: int, k: int, n: int = 0, nnz: int = 0, iterate_bytes: int = 2,
               matrix_bytes_per_nnz: float = 5.4, hbm_gbs: float = 6500.0, nvlink_gbs: float = 900.0):
    """P_r x P_c factorisation of the world for the 2-D mode, chosen by the
    per-step byte model of SURVEY §8e: per GPU the HBM moves matrix / P_r plus
    its column block of the iterate (read in full, band written), and the
    NVLink ingress is (P_r - 1) / P_r of N x k / P_c iterate entries; the step
    time is the larger of the two.  Ties prefer fewer column blocks (a bigger
    block per GPU keeps the SpMM's nonzero reuse).  Without sizes (n = 0) the
    model degenerates to 'most column blocks', P_c <= k."""
    best, best_t = (world, 1), None
    for pc in range(1, world + 1):
        if world % pc or pc > max(1, k):
            continue
        pr = world // pc
        vb = n * (k / pc) * iterate_bytes
        hbm = nnz * matrix_bytes_per_nnz / pr + vb * (1 + 1 / pr)
        nvl = vb * (pr - 1) / pr
        t = max(hbm / hbm_gbs, nvl / nvlink_gbs) if n else -pc
        if best_t is None or t < best_t - 1e-12:
            best, best_t = (pr, pc), t
    return best


_COL_GROUPS = {}


def _column_groups(base, pr, pc):
    """The P_c all-gather groups of a P_r x P_c grid over ranks ``base``,
    created once per (ranks, grid) and reused by later calls (with NCCL each
    group is a communicator; re-creating them per call would leak them)."""
    import torch.distributed as dist
    key = (id(dist.group.WORLD), base, pr, pc)     # a re-initialised world gets new groups
    if key not in _COL_GROUPS:
        _COL_GROUPS[key] = [dist.new_group([base[r * pc + jj] for r in range(pr)]) for jj in range(pc)]
    return _COL_GROUPS[key]


def sequence_2d(n, row_idx, col_idx, vals, m, X, L, U, backend, pr, pc, group=None, want_vout=False,
                on_step=None):
    """2-D sequence on a P_r x P_c grid of ranks (rank = i * P_c + j): rank
    (i, j) owns row band i of A (nnz-balanced) and column block j of X.  Per
    step it computes its band of V_{t+1}[:, block j] and all-gathers the bands
    among the P_r ranks of column block j (the exchange moves (P_r-1)/P_r of
    N x k/P_c instead of N x k); the band projections U[band i]^T V[band i,
    block j] are summed mod m over i once at the end.  P_r = 1 is the column
    mode, P_c = 1 the row mode.  Returns S (L x ku x
    k) on every rank (and V_L if asked).  ``on_step(t)``, if given, is
    called before step t and once more with t = L after the last one (the
    bench brackets its timed steps with device events there)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if pr * pc != world:
        raise ValueError(f"grid {pr} x {pc} does not match world size {world}")
    X = np.asarray(X, dtype=np.uint32)
    k = X.shape[1]
    U = X if U is None else np.asarray(U, dtype=np.uint32)
    ku = U.shape[1]
    i, j = divmod(rank, pc)
    b = row_bands(row_idx, n, pr)
    c = column_shards(k, pc)
    counts = [int(b[r + 1] - b[r]) for r in range(pr)]
    lo, hi = int(b[i]), int(b[i + 1])
    c0, c1 = int(c[j]), int(c[j + 1])
    w = c1 - c0
    # one all-gather group per column block (every rank creates every group,
    # in the same order, as torch.distributed requires)
    base = dist.get_process_group_ranks(group) if group is not None else list(range(world))
    col_groups = _column_groups(tuple(base), pr, pc)
    ri, ci, v = band_triples(row_idx, col_idx, vals, lo, hi)
    A_band = backend.create(hi - lo, n, ri, ci, v, m)
    dev = getattr(backend, "device", torch.device("cpu"))
    wmax = max(1, int(max(c[1:] - c[:-1])))
    S_part = torch.zeros((L, ku, wmax), dtype=torch.int32, device=dev)
    V = None
    if w:
        V = backend.tensor(X[:, c0:c1])                 # column block j, replicated over i
        U_band = backend.tensor(U[lo:hi])
        S_band = backend.empty((L, ku, w))
        for t in range(L):
            if on_step is not None:
                on_step(t)
            backend.project(A_band, V[lo:hi], U_band, S_band[t])
            if t + 1 < L or want_vout:
                out = backend.empty((hi - lo, w))
                backend.apply_block(A_band, V, out)
                V = _all_gather_rows(col_groups[j], out, counts)
        if on_step is not None:
            on_step(L)
        S_part[:, :, :w] = S_band
    parts = [torch.empty_like(S_part) for _ in range(world)]
    dist.all_gather(parts, S_part, group=group)
    S = np.zeros((L, ku, k), np.uint32)
    for jj in range(pc):
        wj = int(c[jj + 1] - c[jj])
        if not wj or not L:
            continue
        stack = torch.stack([parts[r * pc + jj][:, :, :wj].contiguous() for r in range(pr)])
        out = backend.empty((L, ku, wj))
        backend.sum_mod(A_band, stack, out)             # sum over row bands, mod m, on device
        S[:, :, c[jj]:c[jj + 1]] = backend.to_numpy(out)
    if want_vout:
        # V_L: gather the column blocks (row group 0 holds each block complete)
        vb = torch.zeros((n, wmax), dtype=torch.int32, device=dev)
        if w:
            vb[:, :w] = V
        vparts = [torch.empty_like(vb) for _ in range(world)]
        dist.all_gather(vparts, vb, group=group)
        Vout = np.zeros((n, k), np.uint32)
        for jj in range(pc):
            wj = int(c[jj + 1] - c[jj])
            Vout[:, c[jj]:c[jj + 1]] = vparts[jj].cpu().numpy().view(np.uint32)[:, :wj]
        return S, Vout
    return S

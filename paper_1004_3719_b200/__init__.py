"""Thin Python binding of the C ABI in ``include/ffspmv.h`` (libffspmv.so).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  Functions carry the C names; device vectors are
torch CUDA tensors of 4-byte elements (int32 or uint32 bit patterns), passed
by ``data_ptr()`` on the caller's (or torch's current) stream.  There is no
CPU fallback: if the extension is missing, :func:`load` raises.

Paper: Boyer, Dumas & Giorgi, arXiv:1004.3719 (cited "P:line" of PAPER.md).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libffspmv.so")

OK, ERR_INVALID_ARG, ERR_MODULUS, ERR_INDEX, ERR_DIM, ERR_NONSQUARE, ERR_UNSUPPORTED, \
    ERR_NOMEM, ERR_CUDA, ERR_NCCL = range(10)
FMT_AUTO, FMT_SELL, FMT_CSR, FMT_COOS = range(4)
STRATEGY_AUTO, STRATEGY_ROWS, STRATEGY_PANELS, STRATEGY_RUNS = range(4)
OP_APPLY, OP_TRANSPOSE, OP_BLOCK, OP_SEQUENCE, OP_PROJECT = range(5)

# Every symbol include/ffspmv.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "ffspmv_create", "ffspmv_destroy", "ffspmv_get_info", "ffspmv_analyze", "ffspmv_apply",
    "ffspmv_apply_transpose", "ffspmv_apply_block", "ffspmv_apply_host",
    "ffspmv_workspace_size", "ffspmv_sequence", "ffspmv_project", "ffspmv_sum_mod",
    "ffspmv_status_string", "ffspmv_last_error", "ffspmv_version", "ffspmv_kernel_launches",
    "ffspmv_comm_unique_id", "ffspmv_comm_create", "ffspmv_comm_create_local", "ffspmv_comm_destroy",
]


class ffspmv_options(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("no_transpose", ctypes.c_int32),
        ("segregate_pm1", ctypes.c_int32),
        ("force_format", ctypes.c_int32),
        ("band_rows", ctypes.c_uint32),
        ("long_row", ctypes.c_uint32),
        ("force_acc_bits", ctypes.c_int32),
        ("check_inputs", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("panel_rows", ctypes.c_uint32),
        ("panel_cols", ctypes.c_uint32),
        ("panel_xbits", ctypes.c_uint32),
        ("comm", ctypes.c_void_p),
        ("dist_rows", ctypes.c_uint32),
    ]


class ffspmv_info(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("modulus", ctypes.c_uint32),
        ("rows", ctypes.c_uint64),
        ("cols", ctypes.c_uint64),
        ("nnz_input", ctypes.c_uint64),
        ("nnz", ctypes.c_uint64),
        ("nnz_pm1", ctypes.c_uint64),
        ("nnz_valued", ctypes.c_uint64),
        ("value_bytes", ctypes.c_uint32),
        ("iterate_bytes", ctypes.c_uint32),
        ("bands", ctypes.c_uint32),
        ("bands_sell", ctypes.c_uint32),
        ("bands_csr", ctypes.c_uint32),
        ("bands_coos", ctypes.c_uint32),
        ("slices", ctypes.c_uint64),
        ("csr_groups", ctypes.c_uint64),
        ("long_rows", ctypes.c_uint64),
        ("split_rows", ctypes.c_uint64),
        ("padded_slots", ctypes.c_uint64),
        ("acc_slices_u32", ctypes.c_uint32),
        ("acc_slices_u64", ctypes.c_uint32),
        ("acc_slices_u96", ctypes.c_uint32),
        ("acc_bits_max", ctypes.c_uint32),
        ("device_bytes", ctypes.c_uint64),
        ("stream_bytes", ctypes.c_uint64),
        ("alg_bytes_apply", ctypes.c_uint64),
        ("alg_bytes_transpose", ctypes.c_uint64),
        ("has_transpose", ctypes.c_uint32),
        ("create_seconds", ctypes.c_double),
        ("strategy_apply", ctypes.c_uint32),
        ("strategy_transpose", ctypes.c_uint32),
        ("panels", ctypes.c_uint32),
        ("panel_bands", ctypes.c_uint32),
        ("panel_stream_bytes", ctypes.c_uint64),
        ("gather_locality", ctypes.c_double),
        ("panel_xbits", ctypes.c_uint32),
        ("dist_ranks", ctypes.c_uint32),
        ("dist_grid_rows", ctypes.c_uint32),
        ("dist_band_row0", ctypes.c_uint64),
        ("dist_band_rows", ctypes.c_uint64),
    ]


class FFSPMVError(RuntimeError):
    def __init__(self, status, message):
        self.status = status
        super().__init__(f"{status_name(status)}: {message}")


_lib = None


def load(path: str = LIB_PATH):
    """Load libffspmv.so (built by ``python -m paper_1004_3719_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sig = {
        "ffspmv_create": [ctypes.POINTER(P), u64, u64, u64, P, P, P, u32, ctypes.POINTER(ffspmv_options)],
        "ffspmv_destroy": [P],
        "ffspmv_get_info": [P, ctypes.POINTER(ffspmv_info)],
        "ffspmv_analyze": [u64, u64, u64, P, P, P, u32, ctypes.POINTER(ffspmv_options),
                           ctypes.POINTER(ffspmv_info), i32, P, P, P, u64, ctypes.POINTER(u64)],
        "ffspmv_apply": [P, u32, P, u64, u32, P, u64, P],
        "ffspmv_apply_transpose": [P, u32, P, u64, u32, P, u64, P],
        "ffspmv_apply_block": [P, u32, u32, P, u64, u32, P, u64, P],
        "ffspmv_apply_host": [P, i32, u32, P, u32, P, P],
        "ffspmv_workspace_size": [P, i32, u32, u32, ctypes.POINTER(ctypes.c_size_t)],
        "ffspmv_sequence": [P, u32, P, u32, P, u64, P, P, P, ctypes.c_size_t, P],
        "ffspmv_project": [P, u32, P, u32, P, P, P, ctypes.c_size_t, P],
        "ffspmv_sum_mod": [P, u64, u32, P, P, P],
        "ffspmv_comm_unique_id": [P],
        "ffspmv_comm_create": [ctypes.POINTER(P), P, i32, i32],
        "ffspmv_comm_create_local": [P, i32],
        "ffspmv_comm_destroy": [P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.ffspmv_status_string.argtypes = [ctypes.c_int]
    lib.ffspmv_status_string.restype = ctypes.c_char_p
    lib.ffspmv_last_error.argtypes = []
    lib.ffspmv_last_error.restype = ctypes.c_char_p
    lib.ffspmv_version.restype = ctypes.c_int
    lib.ffspmv_kernel_launches.restype = ctypes.c_uint64
    _lib = lib
    return lib


def status_name(s: int) -> str:
    return load().ffspmv_status_string(s).decode()


def ffspmv_last_error() -> str:
    return load().ffspmv_last_error().decode()


def ffspmv_status_string(s: int) -> str:
    return status_name(s)


def ffspmv_version() -> int:
    return load().ffspmv_version()


def ffspmv_kernel_launches() -> int:
    return int(load().ffspmv_kernel_launches())


def _check(rc):
    if rc != OK:
        raise FFSPMVError(rc, ffspmv_last_error())


def make_options(device=-1, no_transpose=False, segregate_pm1=0, force_format=FMT_AUTO,
                 band_rows=0, long_row=0, force_acc_bits=0, check_inputs=False,
                 strategy=STRATEGY_AUTO, panel_rows=0, panel_cols=0, panel_xbits=0, comm=None,
                 dist_rows=0):
    o = ffspmv_options()
    o.struct_size = ctypes.sizeof(ffspmv_options)
    o.device = device
    o.no_transpose = int(bool(no_transpose))
    o.segregate_pm1 = segregate_pm1
    o.force_format = force_format
    o.band_rows = band_rows
    o.long_row = long_row
    o.force_acc_bits = force_acc_bits
    o.check_inputs = int(bool(check_inputs))
    o.strategy = strategy
    o.panel_rows = panel_rows
    o.panel_cols = panel_cols
    o.panel_xbits = panel_xbits
    o.comm = comm.handle.value if isinstance(comm, Comm) else comm
    o.dist_rows = dist_rows
    return o


def _info_dict(info: ffspmv_info) -> dict:
    return {name: getattr(info, name) for name, _ in info._fields_}


def _triples(row_idx, col_idx, vals):
    ri = np.ascontiguousarray(row_idx, dtype=np.uint32)
    ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
    v = np.ascontiguousarray(vals, dtype=np.int64)
    if not (ri.shape == ci.shape == v.shape) or ri.ndim != 1:
        raise ValueError("row_idx, col_idx and vals must be 1-D arrays of equal length")
    return ri, ci, v


class Matrix:
    """Handle of a matrix built on the device (owns the C handle)."""

    def __init__(self, handle: int, rows: int, cols: int, modulus: int):
        self.handle = ctypes.c_void_p(handle)
        self.rows, self.cols, self.modulus = rows, cols, modulus

    def __del__(self):
        if getattr(self, "handle", None) and self.handle.value and _lib is not None:
            _lib.ffspmv_destroy(self.handle)
            self.handle = ctypes.c_void_p(0)

    # convenience wrappers (allocate outputs with torch, then call the C ABI)
    def info(self) -> dict:
        return ffspmv_get_info(self)

    def apply(self, x, y=None, alpha=1, beta=0, stream=None):
        import torch
        if y is None:
            y = torch.empty(self.rows, dtype=x.dtype, device=x.device)
        return ffspmv_apply(self, alpha, x, beta, y, stream)

    def apply_transpose(self, x, y=None, alpha=1, beta=0, stream=None):
        import torch
        if y is None:
            y = torch.empty(self.cols, dtype=x.dtype, device=x.device)
        return ffspmv_apply_transpose(self, alpha, x, beta, y, stream)

    def apply_block(self, X, Y=None, alpha=1, beta=0, stream=None):
        import torch
        if Y is None:
            Y = torch.empty((self.rows, X.shape[1]), dtype=X.dtype, device=X.device)
        return ffspmv_apply_block(self, X.shape[1], alpha, X, beta, Y, stream)

    def sequence(self, X, L, U=None, want_vout=False, stream=None):
        import torch
        k = X.shape[1]
        ku = U.shape[1] if U is not None else k
        S = torch.empty((L, ku, k), dtype=X.dtype, device=X.device)
        V = torch.empty_like(X) if want_vout else None
        ws = torch.empty(max(1, ffspmv_workspace_size(self, OP_SEQUENCE, k, ku)), dtype=torch.uint8,
                         device=X.device)
        ffspmv_sequence(self, k, X, ku, U, L, S, V, ws, stream)
        return (S, V) if want_vout else S


def _h(A):
    return A.handle if isinstance(A, Matrix) else ctypes.c_void_p(A)


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if t.element_size() != 4:
            raise TypeError("vectors must have 4-byte elements (int32 / uint32)")
        if not t.is_cuda:
            raise TypeError("device entry points need CUDA tensors")
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(int(t))


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


# --------------------------------------------------------------- C names ---

def ffspmv_create(rows, cols, row_idx, col_idx, vals, modulus, options=None, **kw) -> Matrix:
    """Build A from COO triples (host arrays) on the current CUDA device."""
    lib = load()
    ri, ci, v = _triples(row_idx, col_idx, vals)
    opts = options if options is not None else make_options(**kw)
    h = ctypes.c_void_p()
    _check(lib.ffspmv_create(ctypes.byref(h), rows, cols, ri.size,
                             ri.ctypes.data_as(ctypes.c_void_p), ci.ctypes.data_as(ctypes.c_void_p),
                             v.ctypes.data_as(ctypes.c_void_p), modulus, ctypes.byref(opts)))
    return Matrix(h.value, rows, cols, modulus)


def ffspmv_destroy(A: Matrix):
    _check(load().ffspmv_destroy(_h(A)))
    if isinstance(A, Matrix):
        A.handle = ctypes.c_void_p(0)


def ffspmv_get_info(A) -> dict:
    info = ffspmv_info()
    _check(load().ffspmv_get_info(_h(A), ctypes.byref(info)))
    return _info_dict(info)


def ffspmv_analyze(rows, cols, row_idx, col_idx, vals, modulus, transpose=False,
                   reconstruct=False, options=None, **kw):
    """Host-only planner; optionally returns the triples rebuilt from the
    packed layout (rows, cols, vals arrays)."""
    lib = load()
    ri, ci, v = _triples(row_idx, col_idx, vals)
    opts = options if options is not None else make_options(**kw)
    info = ffspmv_info()
    rec = None
    args = [None, None, None, 0, None]
    if reconstruct:
        cap = ri.size + 1
        rec = [np.zeros(cap, np.uint32) for _ in range(3)]
        n = ctypes.c_uint64()
        args = [r.ctypes.data_as(ctypes.c_void_p) for r in rec] + [cap, ctypes.byref(n)]
    _check(lib.ffspmv_analyze(rows, cols, ri.size, ri.ctypes.data_as(ctypes.c_void_p),
                              ci.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p),
                              modulus, ctypes.byref(opts), ctypes.byref(info), int(bool(transpose)),
                              *args))
    d = _info_dict(info)
    if reconstruct:
        return d, tuple(r[: n.value] for r in rec)
    return d


def ffspmv_apply(A, alpha, x, beta, y, stream=None):
    """y <- (alpha A x + beta y) mod m on device tensors."""
    _check(load().ffspmv_apply(_h(A), alpha % (1 << 32), _ptr(x), x.numel(), beta % (1 << 32),
                               _ptr(y), y.numel(), _stream(stream)))
    return y


def ffspmv_apply_transpose(A, alpha, x, beta, y, stream=None):
    """y <- (alpha A^T x + beta y) mod m."""
    _check(load().ffspmv_apply_transpose(_h(A), alpha % (1 << 32), _ptr(x), x.numel(),
                                         beta % (1 << 32), _ptr(y), y.numel(), _stream(stream)))
    return y


def ffspmv_apply_block(A, k, alpha, X, beta, Y, stream=None):
    """Y <- (alpha A X + beta Y) mod m; X, Y 2-D with unit inner stride."""
    if X.dim() != 2 or Y.dim() != 2:
        raise ValueError("X and Y must be 2-D")
    for T in (X, Y):
        if T.numel() and T.shape[1] > 1 and T.stride(1) != 1:
            raise ValueError("X and Y must have contiguous rows")
    ldx = max(X.stride(0), k) if X.shape[0] > 1 else k
    ldy = max(Y.stride(0), k) if Y.shape[0] > 1 else k
    _check(load().ffspmv_apply_block(_h(A), k, alpha % (1 << 32), _ptr(X), ldx,
                                     beta % (1 << 32), _ptr(Y), ldy, _stream(stream)))
    return Y


def ffspmv_apply_host(A, op, alpha, x_host, beta, y_host, stream=None):
    """End-to-end apply on host numpy uint32 arrays (synchronous)."""
    x = np.ascontiguousarray(x_host, dtype=np.uint32)
    if not (isinstance(y_host, np.ndarray) and y_host.dtype == np.uint32 and y_host.flags.c_contiguous):
        raise TypeError("y_host must be a C-contiguous uint32 numpy array")
    _check(load().ffspmv_apply_host(_h(A), op, alpha % (1 << 32), x.ctypes.data_as(ctypes.c_void_p),
                                    beta % (1 << 32), y_host.ctypes.data_as(ctypes.c_void_p),
                                    _stream(stream)))
    return y_host


def ffspmv_workspace_size(A, op, k, ku) -> int:
    b = ctypes.c_size_t()
    _check(load().ffspmv_workspace_size(_h(A), op, k, ku, ctypes.byref(b)))
    return b.value


def ffspmv_sequence(A, k, X, ku, U, L, S, V_out, workspace, stream=None):
    """S[t] = U^T A^t X mod m for t < L; V_out <- A^L X."""
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    ws = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else None
    _check(load().ffspmv_sequence(_h(A), k, _ptr(X), ku, _ptr(U), L, _ptr(S), _ptr(V_out), ws,
                                  nbytes, _stream(stream)))
    return S


def ffspmv_project(A, k, V, ku, U, S, workspace, stream=None):
    """S = U^T V mod m over the rows of A (ku x k)."""
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    ws = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else None
    _check(load().ffspmv_project(_h(A), k, _ptr(V), ku, _ptr(U), _ptr(S), ws, nbytes,
                                 _stream(stream)))
    return S


# ------------------------------------------------------------ communicators ---

class Comm:
    """A communicator of the distributed sequence (owns the C handle)."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle = ctypes.c_void_p(handle)
        self.nranks, self.rank = nranks, rank

    def close(self):
        if self.handle.value and _lib is not None:
            _check(_lib.ffspmv_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p(0)


def ffspmv_comm_unique_id() -> bytes:
    """128-byte NCCL unique id (call on one rank, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().ffspmv_comm_unique_id(buf))
    return buf.raw


def ffspmv_comm_create(uid: bytes, nranks: int, rank: int) -> Comm:
    """NCCL communicator (collective over the nranks processes)."""
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load().ffspmv_comm_create(ctypes.byref(h), buf, nranks, rank))
    return Comm(h.value, nranks, rank)


def ffspmv_comm_create_local(nranks: int):
    """In-process group of nranks communicators (ranks = host threads on one
    device) for testing the distributed path on one GPU."""
    arr = (ctypes.c_void_p * nranks)()
    _check(load().ffspmv_comm_create_local(arr, nranks))
    return [Comm(arr[r], nranks, r) for r in range(nranks)]


def ffspmv_comm_destroy(c: Comm):
    c.close()


def comm_from_torch(group=None) -> Comm:
    """NCCL communicator over a torch.distributed process group: rank 0 draws
    the unique id and broadcasts it over the group (argument marshalling only:
    the per-step exchange runs inside ffspmv_sequence)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t[:] = torch.frombuffer(bytearray(ffspmv_comm_unique_id()), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return ffspmv_comm_create(bytes(t.cpu().numpy().tobytes()), world, rank)


def ffspmv_sum_mod(A, count, nparts, parts, out, stream=None):
    """out[i] = sum_p parts[p*count + i] mod m (device tensors)."""
    _check(load().ffspmv_sum_mod(_h(A), count, nparts, _ptr(parts), _ptr(out), _stream(stream)))
    return out

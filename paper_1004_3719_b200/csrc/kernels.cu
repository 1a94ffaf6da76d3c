// Apply (y <- alpha A x + beta y) and block apply (Y <- alpha A X + beta Y)
// kernels for sm_100a.  SURVEY §8 rows a-5, a-6 (same kernel on the packed
// A^T), a-7.
//
// Work decomposition: one warp per work item, items ordered
//   [long rows (longest first)] [SELL slices] [CSR / COO_S groups] [zero rows]
// so the long rows start in the first wave ("unbalanced rows ... will
// produce many idle threads").  The hardware block scheduler balances the
// rest dynamically.
#include <atomic>

#include "device.cuh"

namespace ffspmv {

static std::atomic<uint64_t> g_launches{0};
uint64_t kernel_launch_count() { return g_launches.load(std::memory_order_relaxed); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

constexpr int WARPS = 4;  // warps per CTA of the item kernels

__device__ __forceinline__ SliceHdr load_hdr(const SliceHdr *p) {
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
    SliceHdr h;
    *reinterpret_cast<uint4 *>(&h) = v;
    return h;
}

static inline uint32_t total_items(const DevOp &op) {
    return op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
}

// =========================================================== apply ========

// SELL slice: lane = row; slot j of the lane at off + 32 j + lane, so every
// index / value load of the warp is one coalesced 128 B (64 B, 32 B) line.
template <class Acc, class VT>
__device__ __forceinline__ void apply_slice(const DevOp &op, const DevMod &M, uint32_t s,
                                            const SliceHdr &h, uint32_t lane, uint32_t alpha,
                                            const uint32_t *__restrict__ x, uint32_t beta,
                                            uint32_t *__restrict__ y) {
    uint32_t row = ld_stream(op.perm + s * 32 + lane);
    Acc acc;
    auto g = [x](uint32_t c) { return ld_gather(x + c); };
    walk<true>(acc, op.pcol, h.off_p + lane, 32u, (uint32_t)h.wp, op.vcol,
               reinterpret_cast<const VT *>(op.vval), h.off_v + lane, 32u, (uint32_t)h.wv, M.m, g);
    if (row != PAD_ROW) {
        uint32_t yold = beta ? y[row] : 0u;
        y[row] = epilogue(acc.reduce(M), alpha, beta, yold, M);
    }
}

// Long row (or one chunk of a split row): the warp streams the row's
// contiguous entries (Bell's "vector" approach with V = 32), each lane
// reduces its share, then __shfl_xor sums the residues.
template <class Acc, class VT>
__device__ __forceinline__ void apply_long(const DevOp &op, const DevMod &M, const LongItem &it,
                                           uint32_t lane, uint32_t alpha,
                                           const uint32_t *__restrict__ x, uint32_t beta,
                                           uint32_t *__restrict__ y) {
    Acc acc;
    auto g = [x](uint32_t c) { return ld_gather(x + c); };
    uint32_t np = it.len_p > lane ? (it.len_p - lane + 31) / 32 : 0;
    uint32_t nv = it.len_v > lane ? (it.len_v - lane + 31) / 32 : 0;
    walk<true>(acc, op.pcol, it.off_p + lane, 32u, np, op.vcol,
               reinterpret_cast<const VT *>(op.vval), it.off_v + lane, 32u, nv, M.m, g);
    uint32_t tot = sum_residues(acc.reduce(M), 1, 16, M);
    if (lane != 0) return;
    if (it.split == NO_SPLIT) {
        uint32_t yold = beta ? y[it.row] : 0u;
        y[it.row] = epilogue(tot, alpha, beta, yold, M);
        return;
    }
    // Split row: chunk residues are summed exactly in u64 (< nchunks * m);
    // the last chunk to arrive finalises and resets the scratch cell.
    uint32_t nch = it.nch_reg & 0x0FFFFFFFu;
    atomicAdd(op.split_acc + it.split, (unsigned long long)tot);
    __threadfence();
    uint32_t prev = atomicAdd(op.split_cnt + it.split, 1u);
    if (prev == nch - 1) {
        __threadfence();
        unsigned long long total = atomicExch(op.split_acc + it.split, 0ull);
        atomicExch(op.split_cnt + it.split, 0u);
        uint32_t yold = beta ? y[it.row] : 0u;
        y[it.row] = epilogue(mod64(total, M), alpha, beta, yold, M);
    }
}

// CSR-vector / COO_S group: V = 2^vlog lanes per row, 32/V rows per pass.
template <class Acc, class VT>
__device__ __forceinline__ void apply_group(const DevOp &op, const DevMod &M, const CsrGroup &gr,
                                            uint32_t lane, uint32_t alpha,
                                            const uint32_t *__restrict__ x, uint32_t beta,
                                            uint32_t *__restrict__ y) {
    const uint32_t vlog = gr.vlog, V = 1u << vlog, R = 32u >> vlog;
    const uint32_t sub = lane >> vlog, sl = lane & (V - 1);
    auto g = [x](uint32_t c) { return ld_gather(x + c); };
    for (uint32_t base = 0; base < gr.nrows; base += R) {
        uint32_t i = base + sub;
        bool live = i < gr.nrows;
        Acc acc;
        uint32_t row = 0;
        if (live) {
            uint32_t li = gr.first + i;
            row = op.csr_rows[li];
            uint32_t p0 = op.csr_pptr[li], p1 = op.csr_pptr[li + 1];
            uint32_t v0 = op.csr_vptr[li], v1 = op.csr_vptr[li + 1];
            uint32_t np = (p1 - p0) > sl ? (p1 - p0 - sl + V - 1) >> vlog : 0;
            uint32_t nv = (v1 - v0) > sl ? (v1 - v0 - sl + V - 1) >> vlog : 0;
            walk<true>(acc, op.pcol, p0 + sl, V, np, op.vcol, reinterpret_cast<const VT *>(op.vval),
                       v0 + sl, V, nv, M.m, g);
        }
        uint32_t tot = sum_residues(acc.reduce(M), 1, (int)V / 2, M);
        if (live && sl == 0) {
            uint32_t yold = beta ? y[row] : 0u;
            y[row] = epilogue(tot, alpha, beta, yold, M);
        }
    }
}

__device__ __forceinline__ void zero_rows_apply(const DevOp &op, const DevMod &M, uint32_t w,
                                                uint32_t lane, uint32_t beta, uint32_t *y) {
    uint32_t i = w * 32 + lane;
    if (i >= op.n_zero_rows) return;
    uint32_t row = op.zero_rows[i];
    y[row] = beta ? mod64((uint64_t)beta * y[row], M) : 0u;
}

template <class VT>
__global__ void __launch_bounds__(WARPS * 32)
k_apply(DevOp op, DevMod M, uint32_t alpha, const uint32_t *__restrict__ x, uint32_t beta,
        uint32_t *__restrict__ y) {
    uint32_t w = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (w < op.n_long) {
        const LongItem it = op.longs[w];
        switch (it.nch_reg >> 28) {
            case ACC32: apply_long<Acc32, VT>(op, M, it, lane, alpha, x, beta, y); break;
            case ACC64: apply_long<Acc64, VT>(op, M, it, lane, alpha, x, beta, y); break;
            default: apply_long<Acc96, VT>(op, M, it, lane, alpha, x, beta, y); break;
        }
        return;
    }
    w -= op.n_long;
    if (w < op.n_slices) {
        const SliceHdr h = load_hdr(op.slices + w);
        switch (h.regime) {
            case ACC32: apply_slice<Acc32, VT>(op, M, w, h, lane, alpha, x, beta, y); break;
            case ACC64: apply_slice<Acc64, VT>(op, M, w, h, lane, alpha, x, beta, y); break;
            default: apply_slice<Acc96, VT>(op, M, w, h, lane, alpha, x, beta, y); break;
        }
        return;
    }
    w -= op.n_slices;
    if (w < op.n_groups) {
        const CsrGroup gr = op.groups[w];
        switch (gr.regime) {
            case ACC32: apply_group<Acc32, VT>(op, M, gr, lane, alpha, x, beta, y); break;
            case ACC64: apply_group<Acc64, VT>(op, M, gr, lane, alpha, x, beta, y); break;
            default: apply_group<Acc96, VT>(op, M, gr, lane, alpha, x, beta, y); break;
        }
        return;
    }
    w -= op.n_groups;
    zero_rows_apply(op, M, w, lane, beta, y);
}

int launch_apply(const DevOp &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                 uint32_t beta, uint32_t *y, void *stream) {
    uint32_t items = total_items(op);
    if (items == 0) return 0;
    dim3 grid((items + WARPS - 1) / WARPS), block(WARPS * 32);
    cudaStream_t st = (cudaStream_t)stream;
    switch (M.vbytes) {
        case 1: k_apply<uint8_t><<<grid, block, 0, st>>>(op, M, alpha, x, beta, y); break;
        case 2: k_apply<uint16_t><<<grid, block, 0, st>>>(op, M, alpha, x, beta, y); break;
        default: k_apply<uint32_t><<<grid, block, 0, st>>>(op, M, alpha, x, beta, y); break;
    }
    count_launch();
    return (int)cudaGetLastError();
}

// ====================================================== input check =======
__global__ void k_check_canonical(const uint32_t *__restrict__ v, uint64_t n, uint64_t ld,
                                  uint64_t w, uint32_t m, uint32_t *flag) {
    uint64_t total = n * w;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = i / w, c = i % w;
        if (v[r * ld + c] >= m) atomicOr(flag, 1u);
    }
}

int launch_check_canonical(const uint32_t *v, uint64_t n, uint64_t ld, uint64_t w, uint32_t m,
                           uint32_t *flag_dev, void *stream) {
    if (n == 0 || w == 0) return 0;
    uint64_t total = n * w;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    k_check_canonical<<<blocks, 256, 0, (cudaStream_t)stream>>>(v, n, ld, w, m, flag_dev);
    count_launch();
    return (int)cudaGetLastError();
}

// ============================================ transpose without A^T =======
// y <- alpha A^T x + beta y from the rows layout of A when A^T is not stored
// ("matrices such that A and A^T cannot be simultaneously stored
// ... occurs on GPU's"): every entry a_rc scatters its term into acc[c], a
// u64 per column, with a global atomic add.  The term is reduced below m+1
// (x_r or m - x_r for +-1 entries, a x_r mod m for valued ones), so a column
// sum stays below nnz_col (m + 1) < 2^64: exact and independent of the order
// of the atomics.  k_scatter_finish reduces, applies alpha / beta and clears
// acc for the next call.
template <class VT>
__device__ __forceinline__ void scatter_entry(unsigned long long *acc, uint32_t c, uint32_t xr, bool pm,
                                              uint32_t a, const DevMod &M) {
    if (c == PAD_COL) return;
    uint64_t t;
    if (pm) t = (c & SIGN_BIT) ? (uint64_t)(M.m - xr) : xr;
    else t = mod64((uint64_t)a * xr, M);
    if (t) atomicAdd(acc + (c & COL_MASK), (unsigned long long)t);
}

template <class VT>
__global__ void __launch_bounds__(WARPS * 32)
k_scatter_t(DevOp op, DevMod M, const uint32_t *__restrict__ x, unsigned long long *__restrict__ acc) {
    uint32_t w = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    const VT *vals = reinterpret_cast<const VT *>(op.vval);
    if (w < op.n_long) {
        const LongItem it = op.longs[w];
        const uint32_t xr = __ldg(x + it.row);
        for (uint32_t j = lane; j < it.len_p; j += 32) scatter_entry<VT>(acc, op.pcol[it.off_p + j], xr, true, 0, M);
        for (uint32_t j = lane; j < it.len_v; j += 32)
            scatter_entry<VT>(acc, op.vcol[it.off_v + j], xr, false, vals[it.off_v + j], M);
        return;
    }
    w -= op.n_long;
    if (w < op.n_slices) {
        const SliceHdr h = load_hdr(op.slices + w);
        const uint32_t row = op.perm[w * 32 + lane];
        if (row == PAD_ROW) return;
        const uint32_t xr = __ldg(x + row);
        for (uint32_t j = 0; j < h.wp; ++j) scatter_entry<VT>(acc, op.pcol[h.off_p + j * 32 + lane], xr, true, 0, M);
        for (uint32_t j = 0; j < h.wv; ++j) {
            const uint32_t i = h.off_v + j * 32 + lane;
            scatter_entry<VT>(acc, op.vcol[i], xr, false, vals[i], M);
        }
        return;
    }
    w -= op.n_slices;
    if (w < op.n_groups) {
        const CsrGroup gr = op.groups[w];
        for (uint32_t i = 0; i < gr.nrows; ++i) {
            const uint32_t li = gr.first + i;
            const uint32_t xr = __ldg(x + op.csr_rows[li]);
            for (uint32_t t = op.csr_pptr[li] + lane; t < op.csr_pptr[li + 1]; t += 32)
                scatter_entry<VT>(acc, op.pcol[t], xr, true, 0, M);
            for (uint32_t t = op.csr_vptr[li] + lane; t < op.csr_vptr[li + 1]; t += 32)
                scatter_entry<VT>(acc, op.vcol[t], xr, false, vals[t], M);
        }
    }
    // zero rows scatter nothing
}

__global__ void k_scatter_finish(unsigned long long *__restrict__ acc, uint32_t n, DevMod M, uint32_t alpha,
                                 uint32_t beta, uint32_t *__restrict__ y) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const uint64_t s = acc[c];
        acc[c] = 0;
        y[c] = epilogue(mod64(s, M), alpha, beta, beta ? y[c] : 0u, M);
    }
}

int launch_apply_scatter_t(const DevOp &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                           uint32_t beta, uint32_t *y, unsigned long long *acc, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t items = total_items(op);
    if (items) {
        dim3 grid((items + WARPS - 1) / WARPS), block(WARPS * 32);
        switch (M.vbytes) {
            case 1: k_scatter_t<uint8_t><<<grid, block, 0, st>>>(op, M, x, acc); break;
            case 2: k_scatter_t<uint16_t><<<grid, block, 0, st>>>(op, M, x, acc); break;
            default: k_scatter_t<uint32_t><<<grid, block, 0, st>>>(op, M, x, acc); break;
        }
        count_launch();
    }
    if (op.cols) {
        const uint32_t blocks = std::min<uint32_t>((op.cols + 255) / 256, 148u * 8);
        k_scatter_finish<<<blocks, 256, 0, st>>>(acc, op.cols, M, alpha, beta, y);
        count_launch();
    }
    return (int)cudaGetLastError();
}

}  // namespace ffspmv

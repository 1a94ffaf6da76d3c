// Block apply Y <- alpha A X + beta Y as header templates:
// instantiated for u32 blocks in block.cu and for the narrow sequence
// iterate in seq.cu.
#pragma once

#include "device.cuh"

namespace ffspmv {

void count_launch();
constexpr int BWARPS = 4;  // warps per CTA of the block kernels

__device__ __forceinline__ SliceHdr load_hdr_b(const SliceHdr *p) {
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
    SliceHdr h;
    *reinterpret_cast<uint4 *>(&h) = v;
    return h;
}

static inline uint32_t total_items_b(const DevOp &op) {
    return op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
}

// =========================================================== block ========
// Lanes own vector columns (KP lanes per row, 32/KP rows per warp pass): each
// nonzero is broadcast to the KP lanes of its row and reused for KP columns
// ("we traverse the matrix only once and x and y are read/written
// contiguously").  k > 32 loops over column chunks of 32.

template <class Acc, class VT, int KP, class TX, class TY>
__device__ __forceinline__ void block_slice(const DevOp &op, const DevMod &M, uint32_t s,
                                            const SliceHdr &h, uint32_t lane, uint32_t k,
                                            uint32_t alpha, const TX *__restrict__ X,
                                            uint64_t ldx, uint32_t beta, TY *__restrict__ Y,
                                            uint64_t ldy) {
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    for (uint32_t c0 = 0; c0 < k; c0 += KP) {
        const uint32_t col = c0 + cl;
        const bool colok = col < k;
        auto gat = [X, ldx, col, colok](uint32_t c) {
            return colok ? ld_gather(X + (uint64_t)c * ldx + col) : 0u;
        };
        for (uint32_t rl = g; rl < h.nrows; rl += G) {
            uint32_t row = op.perm[s * 32 + rl];
            Acc acc;
            walk<false>(acc, op.pcol, h.off_p + rl, 32u, (uint32_t)h.wp, op.vcol,
                        reinterpret_cast<const VT *>(op.vval), h.off_v + rl, 32u, (uint32_t)h.wv,
                        M.m, gat);
            if (colok) {
                TY *yp = Y + (uint64_t)row * ldy + col;
                *yp = (TY)epilogue(acc.reduce(M), alpha, beta, beta ? *yp : 0u, M);
            }
        }
    }
}

template <class VT, int KP, class TX, class TY>
__device__ __forceinline__ void block_long(const DevOp &op, const DevMod &M, uint32_t w,
                                           const LongItem &it, uint32_t lane, uint32_t k,
                                           uint32_t alpha, const TX *__restrict__ X,
                                           uint64_t ldx, uint32_t beta, TY *__restrict__ Y,
                                           uint64_t ldy) {
    if (it.chunk != 0) return;  // a split row is handled whole by its first chunk
    const uint32_t nch = it.nch_reg & 0x0FFFFFFFu;
    const LongItem last = op.longs[w + nch - 1];
    const uint32_t lp = last.off_p + last.len_p - it.off_p;
    const uint32_t lv = last.off_v + last.len_v - it.off_v;
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    const uint32_t np = lp > g ? (lp - g + G - 1) / G : 0;
    const uint32_t nv = lv > g ? (lv - g + G - 1) / G : 0;
    for (uint32_t c0 = 0; c0 < k; c0 += KP) {
        const uint32_t col = c0 + cl;
        const bool colok = col < k;
        auto gat = [X, ldx, col, colok](uint32_t c) {
            return colok ? ld_gather(X + (uint64_t)c * ldx + col) : 0u;
        };
        Acc96 acc;  // any row length: always exact
        walk<false>(acc, op.pcol, it.off_p + g, G, np, op.vcol,
                    reinterpret_cast<const VT *>(op.vval), it.off_v + g, G, nv, M.m, gat);
        uint32_t tot = sum_residues(acc.reduce(M), KP, 16, M);
        if (g == 0 && colok) {
            TY *yp = Y + (uint64_t)it.row * ldy + col;
            *yp = (TY)epilogue(tot, alpha, beta, beta ? *yp : 0u, M);
        }
    }
}

template <class Acc, class VT, int KP, class TX, class TY>
__device__ __forceinline__ void block_group(const DevOp &op, const DevMod &M, const CsrGroup &gr,
                                            uint32_t lane, uint32_t k, uint32_t alpha,
                                            const TX *__restrict__ X, uint64_t ldx,
                                            uint32_t beta, TY *__restrict__ Y, uint64_t ldy) {
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    for (uint32_t c0 = 0; c0 < k; c0 += KP) {
        const uint32_t col = c0 + cl;
        const bool colok = col < k;
        auto gat = [X, ldx, col, colok](uint32_t c) {
            return colok ? ld_gather(X + (uint64_t)c * ldx + col) : 0u;
        };
        for (uint32_t i = g; i < gr.nrows; i += G) {
            const uint32_t li = gr.first + i;
            const uint32_t row = op.csr_rows[li];
            const uint32_t p0 = op.csr_pptr[li], p1 = op.csr_pptr[li + 1];
            const uint32_t v0 = op.csr_vptr[li], v1 = op.csr_vptr[li + 1];
            Acc acc;
            walk<false>(acc, op.pcol, p0, 1u, p1 - p0, op.vcol,
                        reinterpret_cast<const VT *>(op.vval), v0, 1u, v1 - v0, M.m, gat);
            if (colok) {
                TY *yp = Y + (uint64_t)row * ldy + col;
                *yp = (TY)epilogue(acc.reduce(M), alpha, beta, beta ? *yp : 0u, M);
            }
        }
    }
}

template <int KP, class TY>
__device__ __forceinline__ void block_zero(const DevOp &op, const DevMod &M, uint32_t w,
                                           uint32_t lane, uint32_t k, uint32_t beta,
                                           TY *__restrict__ Y, uint64_t ldy) {
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    for (uint32_t i = g; i < 32; i += G) {
        uint32_t zi = w * 32 + i;
        if (zi >= op.n_zero_rows) break;
        uint32_t row = op.zero_rows[zi];
        for (uint32_t col = cl; col < k; col += KP) {
            TY *yp = Y + (uint64_t)row * ldy + col;
            *yp = (TY)(beta ? mod64((uint64_t)beta * *yp, M) : 0u);
        }
    }
}

template <class VT, int KP, class TX, class TY>
__global__ void __launch_bounds__(BWARPS * 32)
k_block(DevOp op, DevMod M, uint32_t k, uint32_t alpha, const TX *__restrict__ X,
        uint64_t ldx, uint32_t beta, TY *__restrict__ Y, uint64_t ldy) {
    uint32_t w = blockIdx.x * BWARPS + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (w < op.n_long) {
        const LongItem it = op.longs[w];
        block_long<VT, KP, TX, TY>(op, M, w, it, lane, k, alpha, X, ldx, beta, Y, ldy);
        return;
    }
    w -= op.n_long;
    if (w < op.n_slices) {
        const SliceHdr h = load_hdr_b(op.slices + w);
        switch (h.regime) {
            case ACC32: block_slice<Acc32, VT, KP, TX, TY>(op, M, w, h, lane, k, alpha, X, ldx, beta, Y, ldy); break;
            case ACC64: block_slice<Acc64, VT, KP, TX, TY>(op, M, w, h, lane, k, alpha, X, ldx, beta, Y, ldy); break;
            default: block_slice<Acc96, VT, KP, TX, TY>(op, M, w, h, lane, k, alpha, X, ldx, beta, Y, ldy); break;
        }
        return;
    }
    w -= op.n_slices;
    if (w < op.n_groups) {
        const CsrGroup gr = op.groups[w];
        switch (gr.regime) {
            case ACC32: block_group<Acc32, VT, KP, TX, TY>(op, M, gr, lane, k, alpha, X, ldx, beta, Y, ldy); break;
            case ACC64: block_group<Acc64, VT, KP, TX, TY>(op, M, gr, lane, k, alpha, X, ldx, beta, Y, ldy); break;
            default: block_group<Acc96, VT, KP, TX, TY>(op, M, gr, lane, k, alpha, X, ldx, beta, Y, ldy); break;
        }
        return;
    }
    w -= op.n_groups;
    block_zero<KP, TY>(op, M, w, lane, k, beta, Y, ldy);
}

template <class VT, class TX, class TY>
static void launch_block_vt(dim3 grid, dim3 block, cudaStream_t st, const DevOp &op,
                            const DevMod &M, uint32_t k, uint32_t alpha, const TX *X,
                            uint64_t ldx, uint32_t beta, TY *Y, uint64_t ldy) {
    if (k <= 1) k_block<VT, 1, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
    else if (k <= 2) k_block<VT, 2, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
    else if (k <= 4) k_block<VT, 4, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
    else if (k <= 8) k_block<VT, 8, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
    else if (k <= 16) k_block<VT, 16, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
    else k_block<VT, 32, TX, TY><<<grid, block, 0, st>>>(op, M, k, alpha, X, ldx, beta, Y, ldy);
}

template <class TX, class TY>
int launch_block_t(const DevOp &op, const DevMod &M, uint32_t k, uint32_t alpha, const TX *X,
                   uint64_t ldx, uint32_t beta, TY *Y, uint64_t ldy, void *stream) {
    uint32_t items = total_items_b(op);
    if (items == 0) return 0;
    dim3 grid((items + BWARPS - 1) / BWARPS), block(BWARPS * 32);
    cudaStream_t st = (cudaStream_t)stream;
    switch (M.vbytes) {
        case 1: launch_block_vt<uint8_t, TX, TY>(grid, block, st, op, M, k, alpha, X, ldx, beta, Y, ldy); break;
        case 2: launch_block_vt<uint16_t, TX, TY>(grid, block, st, op, M, k, alpha, X, ldx, beta, Y, ldy); break;
        default: launch_block_vt<uint32_t, TX, TY>(grid, block, st, op, M, k, alpha, X, ldx, beta, Y, ldy); break;
    }
    count_launch();
    return (int)cudaGetLastError();
}


}  // namespace ffspmv

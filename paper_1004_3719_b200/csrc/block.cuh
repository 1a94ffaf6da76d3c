// Block apply Y <- alpha A X + beta Y as header templates,
// shared by ffspmv_apply_block (block.cu, u32 blocks) and the block Wiedemann
// sequence (seq.cu, narrow iterate + fused projection).
//
// Lanes own vector columns: KP = min(32, pow2ceil(k)) lanes share a matrix row
// and each owns one column, G = 32/KP rows are in flight per warp, so every
// nonzero is read once and reused for KP columns ("we traverse the matrix only
// once and x and y are read/written contiguously").  k > 32 loops
// over column chunks of 32.
//
// SELL slices are walked slot-major: the warp loads slot j of all 32 rows with
// one coalesced load, then each lane takes the (col, value) of each of its NR
// rows by __shfl_sync and issues NR independent gathers of X -- NR loads in
// flight per lane instead of a dependent walk per row.  When k % 4 == 0 the
// slices take block_slice_as instead (4 columns per lane, gathers landed in
// shared memory by cp.async, see there).
//
// Results leave through an output policy `Out`:
//   out.put(row, col, colok, residue)   called exactly once per (row, col)
// (BlockOut: alpha/beta epilogue into Y; the sequence adds the projection).
#pragma once

#include "device.cuh"

// 1: the cp.async walks' matrix-stream copies and the block output stores
// carry L2 evict-first hints (0: no hints, A/B measurement)
#ifndef FFSPMV_AS_HINT
#define FFSPMV_AS_HINT 1
#endif

namespace ffspmv {

void count_launch();
constexpr int BWARPS = 4;  // warps per CTA of the non-persistent block kernel

__device__ __forceinline__ SliceHdr load_hdr_b(const SliceHdr *p) {
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
    SliceHdr h;
    *reinterpret_cast<uint4 *>(&h) = v;
    return h;
}

static inline uint32_t total_items_b(const DevOp &op) {
    return op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
}

template <class TY>
struct BlockOut {
    TY *Y;
    uint64_t ldy;
    uint32_t alpha, beta;
    __device__ __forceinline__ void put(uint32_t row, uint32_t col, bool colok, uint32_t r,
                                        const DevMod &M) {
        if (!colok) return;
        TY *p = Y + (uint64_t)row * ldy + col;
        *p = (TY)epilogue(r, alpha, beta, beta ? (uint32_t)*p : 0u, M);
    }
    __device__ __forceinline__ void zero(uint32_t row, uint32_t col, const DevMod &M) {
        TY *p = Y + (uint64_t)row * ldy + col;
        *p = (TY)(beta ? mod64((uint64_t)beta * (uint32_t)*p, M) : 0u);
    }
    // columns col .. col + 3 (all valid when colok: k % 4 == 0); u32 blocks
    // with beta = 0 leave as one 16-byte store, evict-first in L2 (the output
    // is not re-read by this launch, the gathered X is)
    // (HINT = false: plain stores -- measured faster for the two-pass k = 32
    // walk, 258 vs 274 us on c4)
    template <bool HINT>
    __device__ __forceinline__ void put4(uint32_t row, uint32_t col, bool colok, const uint32_t (&r)[4],
                                         const DevMod &M) {
        if (!colok) return;
        TY *p = Y + (uint64_t)row * ldy + col;
        if constexpr (sizeof(TY) == 4 && HINT && FFSPMV_AS_HINT) {
            if (!beta && ((uintptr_t)p & 15) == 0) {
                const uint32_t a0 = epilogue(r[0], alpha, 0u, 0u, M), a1 = epilogue(r[1], alpha, 0u, 0u, M),
                               a2 = epilogue(r[2], alpha, 0u, 0u, M), a3 = epilogue(r[3], alpha, 0u, 0u, M);
                asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;"
                             ::"l"(p), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "l"(POLICY_EVICT_FIRST) : "memory");
                return;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) p[c] = (TY)epilogue(r[c], alpha, beta, beta ? (uint32_t)p[c] : 0u, M);
    }
};

// G = 32/KP rows in flight per warp, NR rows per lane per pass (<= NRMAX,
// bounding the accumulator registers), PASSES passes over the slice.
template <int KP, int NRMAX>
struct SliceShape {
    static constexpr int G = 32 / KP;
    static constexpr int NR = KP < NRMAX ? KP : NRMAX;
    static constexpr int PASSES = 32 / (G * NR);
};

template <class Acc, class VT, int KP, int NRMAX, class TX, class Out>
__device__ __forceinline__ void block_slice(const DevOp &op, const DevMod &M, uint32_t s,
                                            const SliceHdr &h, uint32_t lane, uint32_t k,
                                            const TX *__restrict__ X, uint32_t ldx, Out &out) {
    using S = SliceShape<KP, NRMAX>;
    const uint32_t g = lane / KP, cl = lane % KP;
    const uint32_t m = M.m;
    const uint32_t *pc = op.pcol + h.off_p + lane;
    const uint32_t *vc = op.vcol + h.off_v + lane;
    const VT *vv = reinterpret_cast<const VT *>(op.vval) + h.off_v + lane;
    const uint32_t wp = h.wp, wv = h.wv;
    for (uint32_t c0 = 0; c0 < k; c0 += KP) {
        const uint32_t col = c0 + cl;
        const bool colok = col < k;
#pragma unroll 1
        for (int pass = 0; pass < S::PASSES; ++pass) {
            const uint32_t rbase = pass * S::G * S::NR + g;
            Acc acc[S::NR];
            // +-1 slots: addend x or m - x
            uint32_t cw = wp ? ld_bcast(pc) : PAD_COL;
            for (uint32_t j = 0; j < wp; ++j) {
                const uint32_t cur = cw;
                if (j + 1 < wp) cw = ld_bcast(pc + (j + 1) * 32);
                uint32_t xv[S::NR], cs[S::NR];
#pragma unroll
                for (int i = 0; i < S::NR; ++i) {
                    cs[i] = __shfl_sync(0xFFFFFFFFu, cur, rbase + i * S::G);
                    // 32-bit element index, one IMAD.WIDE for the address
                    const uint32_t idx = (cs[i] & COL_MASK) * ldx + col;
                    xv[i] = (cs[i] != PAD_COL && colok) ? (uint32_t)ld_gather(X + idx) : 0u;
                }
#pragma unroll
                for (int i = 0; i < S::NR; ++i) acc[i].add((cs[i] & SIGN_BIT) ? m - xv[i] : xv[i]);
            }
            // valued slots: addend a * x
            uint32_t vw = wv ? ld_bcast(vc) : PAD_COL;
            uint32_t aw = wv ? ld_bcast(vv) : 0u;
            for (uint32_t j = 0; j < wv; ++j) {
                const uint32_t cur = vw, cura = aw;
                if (j + 1 < wv) { vw = ld_bcast(vc + (j + 1) * 32); aw = ld_bcast(vv + (j + 1) * 32); }
                uint32_t xv[S::NR], as[S::NR];
#pragma unroll
                for (int i = 0; i < S::NR; ++i) {
                    const uint32_t c = __shfl_sync(0xFFFFFFFFu, cur, rbase + i * S::G);
                    as[i] = __shfl_sync(0xFFFFFFFFu, cura, rbase + i * S::G);
                    const uint32_t idx = c * ldx + col;
                    xv[i] = (c != PAD_COL && colok) ? (uint32_t)ld_gather(X + idx) : 0u;
                }
#pragma unroll
                for (int i = 0; i < S::NR; ++i) acc[i].mad(as[i], xv[i]);
            }
#pragma unroll
            for (int i = 0; i < S::NR; ++i) {
                const uint32_t r = rbase + i * S::G;
                if (r < h.nrows) out.put(op.perm[s * 32 + r], col, colok, acc[i].reduce(M), M);
            }
        }
    }
}

// Long row: entries split over the G row groups, each lane a column; the
// group residues are summed with __shfl_xor.  A split row is handled whole
// by its first chunk (always exact in u96).
template <class VT, int KP, class TX, class Out>
__device__ __forceinline__ void block_long(const DevOp &op, const DevMod &M, uint32_t w,
                                           const LongItem &it, uint32_t lane, uint32_t k,
                                           const TX *__restrict__ X, uint32_t ldx, Out &out) {
    if (it.chunk != 0) return;
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
            return colok ? (uint32_t)ld_gather(X + (size_t)(c * ldx + col)) : 0u;
        };
        Acc96 acc;
        walk<false>(acc, op.pcol, it.off_p + g, G, np, op.vcol,
                    reinterpret_cast<const VT *>(op.vval), it.off_v + g, G, nv, M.m, gat);
        uint32_t tot = sum_residues(acc.reduce(M), KP, 16, M);
        if (g == 0) out.put(it.row, col, colok, tot, M);
    }
}

template <class Acc, class VT, int KP, class TX, class Out>
__device__ __forceinline__ void block_group(const DevOp &op, const DevMod &M, const CsrGroup &gr,
                                            uint32_t lane, uint32_t k, const TX *__restrict__ X,
                                            uint32_t ldx, Out &out) {
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    for (uint32_t c0 = 0; c0 < k; c0 += KP) {
        const uint32_t col = c0 + cl;
        const bool colok = col < k;
        auto gat = [X, ldx, col, colok](uint32_t c) {
            return colok ? (uint32_t)ld_gather(X + (size_t)(c * ldx + col)) : 0u;
        };
        for (uint32_t i = g; i < gr.nrows; i += G) {
            const uint32_t li = gr.first + i;
            const uint32_t row = op.csr_rows[li];
            const uint32_t p0 = op.csr_pptr[li], p1 = op.csr_pptr[li + 1];
            const uint32_t v0 = op.csr_vptr[li], v1 = op.csr_vptr[li + 1];
            Acc acc;
            walk<false>(acc, op.pcol, p0, 1u, p1 - p0, op.vcol,
                        reinterpret_cast<const VT *>(op.vval), v0, 1u, v1 - v0, M.m, gat);
            out.put(row, col, colok, acc.reduce(M), M);
        }
    }
}

// Rows with no entries (COO_S bands): the output is beta*Y (or 0), i.e. the
// residue 0 through the policy.
template <int KP, class Out>
__device__ __forceinline__ void block_zero(const DevOp &op, const DevMod &M, uint32_t w,
                                           uint32_t lane, uint32_t k, Out &out) {
    constexpr uint32_t G = 32 / KP;
    const uint32_t g = lane / KP, cl = lane % KP;
    for (uint32_t i = g; i < 32; i += G) {
        uint32_t zi = w * 32 + i;
        if (zi >= op.n_zero_rows) break;
        uint32_t row = op.zero_rows[zi];
        for (uint32_t c0 = 0; c0 < k; c0 += KP) out.put(row, c0 + cl, c0 + cl < k, 0u, M);
    }
}

// One work item (any kind) of the block product.
template <class VT, int KP, int NRMAX, class TX, class Out>
__device__ __forceinline__ void block_item(const DevOp &op, const DevMod &M, uint32_t w,
                                           uint32_t lane, uint32_t k, const TX *__restrict__ X,
                                           uint32_t ldx, Out &out) {
    if (w < op.n_long) {
        const LongItem it = op.longs[w];
        block_long<VT, KP>(op, M, w, it, lane, k, X, ldx, out);
        return;
    }
    w -= op.n_long;
    if (w < op.n_slices) {
        const SliceHdr h = load_hdr_b(op.slices + w);
        switch (h.regime) {
            case ACC32: block_slice<Acc32, VT, KP, NRMAX>(op, M, w, h, lane, k, X, ldx, out); break;
            case ACC64: block_slice<Acc64, VT, KP, NRMAX>(op, M, w, h, lane, k, X, ldx, out); break;
            default: block_slice<Acc96, VT, KP, (NRMAX > 8 ? 8 : NRMAX)>(op, M, w, h, lane, k, X, ldx, out); break;
        }
        return;
    }
    w -= op.n_slices;
    if (w < op.n_groups) {
        const CsrGroup gr = op.groups[w];
        switch (gr.regime) {
            case ACC32: block_group<Acc32, VT, KP>(op, M, gr, lane, k, X, ldx, out); break;
            case ACC64: block_group<Acc64, VT, KP>(op, M, gr, lane, k, X, ldx, out); break;
            default: block_group<Acc96, VT, KP>(op, M, gr, lane, k, X, ldx, out); break;
        }
        return;
    }
    w -= op.n_groups;
    block_zero<KP>(op, M, w, lane, k, out);
}

template <class VT, int KP, class TX, class TY>
__global__ void __launch_bounds__(BWARPS * 32)
k_block(DevOp op, DevMod M, uint32_t k, const TX *__restrict__ X, uint32_t ldx, BlockOut<TY> out) {
    const uint32_t w = blockIdx.x * BWARPS + (threadIdx.x >> 5);
    block_item<VT, KP, 16>(op, M, w, threadIdx.x & 31, k, X, ldx, out);
}

// ---------------------------------------------------- vectorised columns ---
// CPL consecutive columns per lane: one 8 / 16-byte gather of X per (row,
// slot) feeds CPL accumulators, so the per-gather index / address / shuffle /
// predicate work is shared by CPL columns.  Requires k % CPL == 0, ldx % CPL
// == 0 and an aligned X (checked on the host).
template <class TX, int CPL> struct VecT;
template <> struct VecT<uint32_t, 4> { typedef uint4 T; };
template <> struct VecT<uint32_t, 2> { typedef uint2 T; };
template <> struct VecT<uint16_t, 4> { typedef uint2 T; };
template <> struct VecT<uint16_t, 2> { typedef uint32_t T; };
template <> struct VecT<uint8_t, 4> { typedef uint32_t T; };
template <> struct VecT<uint8_t, 2> { typedef uint16_t T; };

template <class TX, int CPL>
__device__ __forceinline__ void ld_vec(const TX *p, uint32_t (&v)[CPL]) {
    typedef typename VecT<TX, CPL>::T V;
    const V w = __ldg(reinterpret_cast<const V *>(p));
    if constexpr (sizeof(TX) == 1) {
        const uint32_t b = (uint32_t)w;
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = (b >> (8 * c)) & 0xFFu;
        return;
    }
    const uint32_t *u = reinterpret_cast<const uint32_t *>(&w);
    if constexpr (sizeof(TX) == 4) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = u[c];
    } else {
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = (u[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
    }
}

// Predicated vector gather (zeros when !pred) without a branch: the masked
// lanes (slice padding, columns >= k) issue no memory request.
template <class TX, int CPL>
__device__ __forceinline__ void ld_vec_pred(const TX *p, bool pred, uint32_t (&v)[CPL]) {
    uint32_t u[4] = {0, 0, 0, 0};
    constexpr int BYTES = CPL * (int)sizeof(TX);
    if constexpr (BYTES == 16) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
                     "@q ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                     : "+r"(u[0]), "+r"(u[1]), "+r"(u[2]), "+r"(u[3]) : "l"(p), "r"((uint32_t)pred));
    } else if constexpr (BYTES == 8) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                     "@q ld.global.nc.v2.u32 {%0, %1}, [%2];\n\t}"
                     : "+r"(u[0]), "+r"(u[1]) : "l"(p), "r"((uint32_t)pred));
    } else if constexpr (BYTES == 4) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.u32 %0, [%1];\n\t}"
                     : "+r"(u[0]) : "l"(p), "r"((uint32_t)pred));
    } else {
        unsigned short hw = 0;
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.u16 %0, [%1];\n\t}"
                     : "+h"(hw) : "l"(p), "r"((uint32_t)pred));
        u[0] = hw;
    }
    if constexpr (sizeof(TX) == 1) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = (u[0] >> (8 * c)) & 0xFFu;
    } else if constexpr (sizeof(TX) == 4) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = u[c];
    } else {
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = (u[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
    }
}

// Asynchronous-copy slice walk (the default vec4 path).  The random X row
// gathers are latency-bound: served from L2 they need ~100+ KB in flight
// per SM (tools/gather_bench3.cu), far more than register-landed loads
// allow next to the NR x CPL accumulators of a lane (a register-landed
// version of this walk kept ~40 KB in flight at 20 warps/SM: 235 us for c4
// k = 16 against 139 us here).  Here the gathers land in a per-warp
// shared-memory ring with cp.async (LDGSTS, zero-filled for padding slots),
// D slots ahead of the accumulation, and the slot index words (and values)
// are copied 2D slots ahead into their own rings, so no load result waits
// in a register: the in-flight bytes are bounded by shared memory (D slots
// x 32 rows x CPL columns per warp) instead of registers.  Step j of a pass:
// wait for the copies of step j - D, accumulate slot j from the rings, then
// issue the gathers of slot j + D (index words from the ring) and the index
// / value copies of slot j + 2D.  Lanes: KPV lanes per row, CPL = 4 columns per lane, G = 32 / KPV row groups, NR
// rows per lane per pass.
template <int D, int NR, class VT>
struct AsRing {
    static constexpr uint32_t data_bytes = D * NR * 32 * 16;
    static constexpr uint32_t bytes = data_bytes + 2 * D * 128 * 2;
};

// index words / values of the matrix stream: read once, evict first from L2
// so the gathered X / V_t rows keep the cache (FFSPMV_AS_HINT = 0: no hint)
// (HINT = false when the walk re-reads the stream: several passes per slice)
template <bool HINT = true>
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src, uint32_t n) {
    if constexpr (FFSPMV_AS_HINT && HINT)
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;"
                     ::"r"(dst), "l"(src), "r"(n), "l"(POLICY_EVICT_FIRST) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_v(uint32_t dst, const void *src, uint32_t n) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
    else if constexpr (BYTES == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}

// N consecutive naturally aligned shared elements of type T (N * sizeof(T)
// <= 16 bytes) with one vector load, widened to u32: a lane's NR index words
// or values in the rings (lanes own consecutive rows, see block_slice_as).
template <class T, int N>
__device__ __forceinline__ void lds_vec(const void *p, uint32_t (&v)[N]) {
    constexpr int B = N * (int)sizeof(T);
    static_assert(B == 1 || B == 2 || B == 4 || B == 8 || B == 16, "vector width");
    uint32_t u[4] = {0, 0, 0, 0};
    if constexpr (B == 16) {
        const uint4 q = *reinterpret_cast<const uint4 *>(p);
        u[0] = q.x; u[1] = q.y; u[2] = q.z; u[3] = q.w;
    } else if constexpr (B == 8) {
        const uint2 q = *reinterpret_cast<const uint2 *>(p);
        u[0] = q.x; u[1] = q.y;
    } else if constexpr (B == 4) {
        u[0] = *reinterpret_cast<const uint32_t *>(p);
    } else if constexpr (B == 2) {
        u[0] = *reinterpret_cast<const uint16_t *>(p);
    } else {
        u[0] = *reinterpret_cast<const uint8_t *>(p);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if constexpr (sizeof(T) == 4) v[i] = u[i];
        else if constexpr (sizeof(T) == 2) v[i] = (u[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
        else v[i] = (u[i >> 2] >> (8 * (i & 3))) & 0xFFu;
    }
}

template <class Acc, class VT, int KPV, int NR, int D, class TX, class Out>
__device__ __forceinline__ void block_slice_as(const DevOp &op, const DevMod &M, uint32_t s,
                                               const SliceHdr &h, uint32_t lane, uint32_t k,
                                               const TX *__restrict__ X, uint32_t ldx, Out &out,
                                               unsigned char *ring, uint32_t fold_every) {
    static_assert((D & (D - 1)) == 0, "ring depth must be a power of two");
    constexpr bool FOLD = std::is_same<Acc, Acc64F>::value;
    constexpr int CPL = 4;
    constexpr int BYTES = CPL * (int)sizeof(TX);
    constexpr uint32_t G = 32 / KPV;
    constexpr int PASSES = 32 / (G * NR);
    using R = AsRing<D, NR, VT>;
    const uint32_t sdata = (uint32_t)__cvta_generic_to_shared(ring) + lane * 16;
    const uint32_t siw = (uint32_t)__cvta_generic_to_shared(ring) + R::data_bytes;
    const uint32_t siv = siw + 2 * D * 128;
    const uint4 *data = reinterpret_cast<const uint4 *>(ring) + lane;
    const uint32_t *iw = reinterpret_cast<const uint32_t *>(ring + R::data_bytes);
    const unsigned char *iv = ring + R::data_bytes + 2 * D * 128;
    const uint32_t g = lane / KPV, cl = lane % KPV;
    const uint32_t m = M.m;
    const uint32_t wp = h.wp, wt = h.wp + h.wv;
    const uint32_t *pcl = op.pcol + h.off_p + lane;
    const uint32_t *vcl = op.vcol + h.off_v + lane - wp * 32;          // index by slot j >= wp
    const unsigned char *vbl = reinterpret_cast<const unsigned char *>(op.vval) +
                               ((uint64_t)h.off_v - wp * 32) * sizeof(VT) + lane * 4;
    const bool vlane = lane < 8 * sizeof(VT);
    for (uint32_t c0 = 0; c0 < k; c0 += KPV * CPL) {
        const uint32_t col = c0 + cl * CPL;
        const bool colok = col < k;
        const TX *Xc = X + col;
#pragma unroll 1
        for (int pass = 0; pass < PASSES; ++pass) {
            // a lane's NR rows of this pass are consecutive (rbase .. rbase +
            // NR - 1), so their index words / values come with one vector load
            const uint32_t rbase = pass * G * NR + g * NR;
            // copies of slot j: its index word / value bytes into idx ring
            // (j mod 2D), its rows into data ring (j mod D)
            auto copy_idx = [&](uint32_t j) {
                const uint32_t q = (j & (2 * D - 1)) * 128;
                constexpr bool once = PASSES == 1;   // the stream is read once per column chunk
                cp_async4<once>(siw + q + lane * 4, j < wp ? pcl + j * 32 : vcl + j * 32, 4);
                if (j >= wp && vlane) cp_async4<once>(siv + q + lane * 4, vbl + (uint64_t)j * 32 * sizeof(VT), 4);
            };
            auto copy_data = [&](uint32_t j) {
                uint32_t w[NR];
                lds_vec<uint32_t, NR>(iw + (j & (2 * D - 1)) * 32 + rbase, w);
                const uint32_t dst = sdata + (j & (D - 1)) * (NR * 512);
#pragma unroll
                for (int i = 0; i < NR; ++i) {
                    const uint32_t c = w[i];
                    const bool ok = c != PAD_COL && colok;
                    cp_async_v<BYTES>(dst + i * 512, Xc + (ok ? (c & COL_MASK) * ldx : 0u), ok ? BYTES : 0);
                }
            };
            Acc acc[NR][CPL];
            // KIND: 0 = +-1 slot, 1 = valued slot, 2 = decided by j < wp (the
            // steady loops are split at wp so their consume has no branch)
            auto consume = [&](uint32_t j, auto kind) {
                constexpr int KIND = decltype(kind)::value;
                const uint4 *d = data + (j & (D - 1)) * (NR * 32);
                const uint32_t q = j & (2 * D - 1);
                uint32_t wa[NR];     // the rows' index words (+-1: sign) or values
                if (KIND == 0 || (KIND == 2 && j < wp)) lds_vec<uint32_t, NR>(iw + q * 32 + rbase, wa);
                else lds_vec<VT, NR>(iv + q * 128 + rbase * sizeof(VT), wa);
#pragma unroll
                for (int i = 0; i < NR; ++i) {
                    const uint4 v = d[i * 32];
                    const uint32_t xv[4] = {v.x, v.y, v.z, v.w};
                    uint32_t xs[CPL];
                    if constexpr (sizeof(TX) == 4) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) xs[c] = xv[c];
                    } else if constexpr (sizeof(TX) == 1) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) xs[c] = (xv[0] >> (8 * c)) & 0xFFu;
                    } else {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) xs[c] = (xv[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                    }
                    if (KIND == 0 || (KIND == 2 && j < wp)) {
                        // -1: (x ^ ~0) + (m + 1) = m - x (mod 2^32)
                        const uint32_t sm = (uint32_t)((int32_t)wa[i] >> 31), sa = sm & (m + 1);
#pragma unroll
                        for (int c = 0; c < CPL; ++c) acc[i][c].add((xs[c] ^ sm) + sa);
                    } else {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) acc[i][c].mad(wa[i], xs[c]);
                    }
                }
            };
            using PM = std::integral_constant<int, 0>;
            using VAL = std::integral_constant<int, 1>;
            using ANY = std::integral_constant<int, 2>;
            auto wait_sync = [&]() {
                asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
                __syncwarp();
            };
            auto commit = []() { asm volatile("cp.async.commit_group;" ::: "memory"); };
            uint32_t since_fold = 0;
            auto maybe_fold = [&]() {
                if constexpr (FOLD) {
                    if (++since_fold == fold_every) {
                        since_fold = 0;
#pragma unroll
                        for (int i = 0; i < NR; ++i)
#pragma unroll
                            for (int c = 0; c < CPL; ++c) acc[i][c].fold(M.r32);
                    }
                }
            };
            // prologue: index words of slots 0 .. 2D-1, gathers of slots 0 .. D-1
            for (uint32_t t = 0; t < 2 * D; ++t) {
                if (t >= (uint32_t)D) {
                    wait_sync();
                    if (t - D < wt) copy_data(t - D);
                }
                if (t < wt) copy_idx(t);
                commit();
            }
            // steady state: consume j, gathers of j + D, index words of j + 2D
            uint32_t j = 0;
            // split at wp for KPV >= 4 (A/B on one box: c4 k = 16 / 32 147 -> 129
            // us, 258 -> 244 us; k = 8 86 -> 96 us, so KPV = 2 keeps one loop)
            constexpr bool SPLIT = KPV >= 4;
            const uint32_t jend = wt > 2 * D ? wt - 2 * D : 0, jpm = SPLIT ? min(wp, jend) : 0u;
#pragma unroll 1
            for (; SPLIT && j < jpm; ++j) {
                wait_sync();
                consume(j, PM());
                maybe_fold();
                __syncwarp();
                copy_idx(j + 2 * D);
                copy_data(j + D);
                commit();
            }
#pragma unroll 1
            for (; j < jend; ++j) {
                wait_sync();
                if constexpr (SPLIT) consume(j, VAL());
                else consume(j, ANY());
                maybe_fold();
                __syncwarp();
                copy_idx(j + 2 * D);
                copy_data(j + D);
                commit();
            }
#pragma unroll 1
            for (; j < wt; ++j) {
                wait_sync();
                consume(j, ANY());
                maybe_fold();
                __syncwarp();
                if (j + D < wt) copy_data(j + D);
                commit();
            }
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const uint32_t r = rbase + i;
                if (r < h.nrows) {
                    const uint32_t row = op.perm[s * 32 + r];
                    uint32_t res[CPL];
#pragma unroll
                    for (int c = 0; c < CPL; ++c) res[c] = acc[i][c].reduce(M);
                    out.template put4<PASSES == 1>(row, col, colok, res, M);
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
        }
    }
}

// D and the occupancy bound: measured on c4 (tools/time_block.py, A/B builds
// of tools/build_variant_flags.sh): D = 2 at 6 CTAs/SM 88.6 / 139 / 270 us
// for k = 8 / 16 / 32 against D = 4 (88.1 / 188 / 285) and D = 2 at 8
// CTAs/SM (90.1 / 166 / 302).
#ifndef FFSPMV_BLOCK_AS_D
#define FFSPMV_BLOCK_AS_D 2     // slots in flight per warp (block_slice_as)
#endif
#ifndef FFSPMV_BLOCK_MINB
#define FFSPMV_BLOCK_MINB 6     // resident 4-warp CTAs per SM the register budget is sized for
#endif

// SELL slices only (warp w = slice w); the other items go to k_block_rest,
// so their register needs do not constrain this kernel's occupancy.  NR:
// rows per lane per pass (NR x 4 accumulators).
template <class Acc, class VT, int KPV, int NR, class TX, class TY>
__global__ void __launch_bounds__(BWARPS * 32, FFSPMV_BLOCK_MINB)
k_block_as(DevOp op, DevMod M, uint32_t k, const TX *__restrict__ X, uint32_t ldx,
           BlockOut<TY> out, uint32_t fold_every) {
    constexpr int D = FFSPMV_BLOCK_AS_D;
    extern __shared__ __align__(16) unsigned char as_smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t s = blockIdx.x * BWARPS + warp;
    if (s >= op.n_slices) return;
    const SliceHdr h = load_hdr_b(op.slices + s);
    block_slice_as<Acc, VT, KPV, NR, D>(op, M, s, h, threadIdx.x & 31, k, X, ldx, out,
                                        as_smem + warp * AsRing<D, NR, VT>::bytes, fold_every);
}

// Every item except the SELL slices: long rows, CSR / COO_S groups, zero rows.
template <class VT, int KP, class TX, class TY>
__global__ void __launch_bounds__(BWARPS * 32)
k_block_rest(DevOp op, DevMod M, uint32_t k, const TX *__restrict__ X, uint32_t ldx,
             BlockOut<TY> out) {
    uint32_t w = blockIdx.x * BWARPS + (threadIdx.x >> 5);
    if (w >= op.n_long) w += op.n_slices;
    block_item<VT, KP, 16>(op, M, w, threadIdx.x & 31, k, X, ldx, out);
}

template <class Acc, class VT, int KPV, int NR, class TX, class TY>
static void launch_as(dim3 grid, dim3 block, cudaStream_t st, const DevOp &op, const DevMod &M,
                      uint32_t k, const TX *X, uint32_t ldx, BlockOut<TY> out, uint32_t fold_every = 0) {
    constexpr int D = FFSPMV_BLOCK_AS_D;
    const int smem = BWARPS * AsRing<D, NR, VT>::bytes;
    auto kern = k_block_as<Acc, VT, KPV, NR, TX, TY>;
    static uint64_t configured = 0;   // per instantiation: devices whose attribute is set
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured >> (dev & 63) & 1)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured |= 1ull << (dev & 63);
    }
    kern<<<grid, block, smem, st>>>(op, M, k, X, ldx, out, fold_every);
}

template <class VT, class TX, class TY>
static void launch_block_vt(dim3 grid, dim3 block, cudaStream_t st, const DevOp &op,
                            const DevMod &M, uint32_t k, const TX *X, uint32_t ldx,
                            BlockOut<TY> out) {
    const bool vec4 = k >= 8 && k % 4 == 0 && ldx % 4 == 0 &&
                      ((uintptr_t)X % (4 * sizeof(TX))) == 0;
    if (vec4) {
        const uint32_t rest = total_items_b(op) - op.n_slices;
        const dim3 gs((op.n_slices + BWARPS - 1) / BWARPS), gr((rest + BWARPS - 1) / BWARPS);
        if (rest) {
            if (k <= 8) k_block_rest<VT, 8, TX, TY><<<gr, block, 0, st>>>(op, M, k, X, ldx, out);
            else if (k <= 16) k_block_rest<VT, 16, TX, TY><<<gr, block, 0, st>>>(op, M, k, X, ldx, out);
            else k_block_rest<VT, 32, TX, TY><<<gr, block, 0, st>>>(op, M, k, X, ldx, out);
            count_launch();
        }
        if (op.n_slices) {
            // rows per lane per pass: 32 / G for k <= 16 (one pass), 4 above
            const uint32_t fe = fold_capacity(M.m, M.r32);
            if (op.acc96 && fe >= 2) {
                if (k <= 8) launch_as<Acc64F, VT, 2, 2>(gs, block, st, op, M, k, X, ldx, out, fe);
                else if (k <= 16) launch_as<Acc64F, VT, 4, 4>(gs, block, st, op, M, k, X, ldx, out, fe);
                else launch_as<Acc64F, VT, 8, 4>(gs, block, st, op, M, k, X, ldx, out, fe);
            } else if (op.acc96) {
                if (k <= 8) launch_as<Acc96, VT, 2, 2>(gs, block, st, op, M, k, X, ldx, out);
                else if (k <= 16) launch_as<Acc96, VT, 4, 4>(gs, block, st, op, M, k, X, ldx, out);
                else launch_as<Acc96, VT, 8, 4>(gs, block, st, op, M, k, X, ldx, out);
            } else {
                if (k <= 8) launch_as<Acc64, VT, 2, 2>(gs, block, st, op, M, k, X, ldx, out);
                else if (k <= 16) launch_as<Acc64, VT, 4, 4>(gs, block, st, op, M, k, X, ldx, out);
                else launch_as<Acc64, VT, 8, 4>(gs, block, st, op, M, k, X, ldx, out);
            }
        }
        return;
    }
    if (k <= 1) k_block<VT, 1, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
    else if (k <= 2) k_block<VT, 2, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
    else if (k <= 4) k_block<VT, 4, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
    else if (k <= 8) k_block<VT, 8, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
    else if (k <= 16) k_block<VT, 16, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
    else k_block<VT, 32, TX, TY><<<grid, block, 0, st>>>(op, M, k, X, ldx, out);
}

template <class TX, class TY>
int launch_block_t(const DevOp &op, const DevMod &M, uint32_t k, uint32_t alpha, const TX *X,
                   uint64_t ldx, uint32_t beta, TY *Y, uint64_t ldy, void *stream) {
    uint32_t items = total_items_b(op);
    if (items == 0) return 0;
    dim3 grid((items + BWARPS - 1) / BWARPS), block(BWARPS * 32);
    cudaStream_t st = (cudaStream_t)stream;
    BlockOut<TY> out{Y, ldy, alpha, beta};
    // X is indexed with 32-bit element offsets (one IMAD.WIDE per gather)
    if ((uint64_t)op.cols * ldx >= (1ull << 32)) return (int)cudaErrorInvalidValue;
    const uint32_t ld32 = (uint32_t)ldx;
    switch (M.vbytes) {
        case 1: launch_block_vt<uint8_t, TX, TY>(grid, block, st, op, M, k, X, ld32, out); break;
        case 2: launch_block_vt<uint16_t, TX, TY>(grid, block, st, op, M, k, X, ld32, out); break;
        default: launch_block_vt<uint32_t, TX, TY>(grid, block, st, op, M, k, X, ld32, out); break;
    }
    count_launch();
    return (int)cudaGetLastError();
}

// Explicit instantiations live in block.cu (u32 -> u32) and block16.cu (u16
// iterates), so seq.cu does not recompile the ~90 block kernels (build time).
#define FFSPMV_BLOCK_LAUNCH(TX, TY)                                                              \
    int launch_block_t<TX, TY>(const DevOp &, const DevMod &, uint32_t, uint32_t, const TX *,  \
                               uint64_t, uint32_t, TY *, uint64_t, void *)
#ifndef FFSPMV_BLOCK_INSTANTIATE
extern template FFSPMV_BLOCK_LAUNCH(uint32_t, uint32_t);
extern template FFSPMV_BLOCK_LAUNCH(uint16_t, uint16_t);
extern template FFSPMV_BLOCK_LAUNCH(uint16_t, uint32_t);
extern template FFSPMV_BLOCK_LAUNCH(uint8_t, uint8_t);
extern template FFSPMV_BLOCK_LAUNCH(uint8_t, uint32_t);
#endif

}  // namespace ffspmv

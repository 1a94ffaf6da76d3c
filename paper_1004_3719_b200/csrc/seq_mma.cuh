// Fused sequence step with a tensor-core projection (SURVEY §8 a-8 + a-9).
//
// One persistent launch per step computes V_{t+1} = A V_t for the SELL
// slices with 4-column vector gathers of the u16 iterate, and the projection
// U^T V_{t+1} of each 32-row slice as a 16 x k x 32 integer contraction on the
// tensor cores: residues < 2^16 are split into u8 limbs (hi, lo) and
//   U^T V = 2^16 Uh^T Vh + 2^8 (Uh^T Vl + Ul^T Vh) + Ul^T Vl
// with mma.sync.m16n8k32 u8 x u8 -> s32 (exact: a slice adds at most
// 32 * 255^2 per element; the s32 accumulators are folded into u64 every 512
// slices).  The projection is a real contraction (k_u * k * N MACs per step,
// more than the SpMM's k * nnz) but too small for tcgen05's M >= 64 tiles
// (M = k_u = 16), hence the warp-level MMA.
//
// U is constant over the sequence, so its limbs are pre-arranged once per call
// in fragment order (U_frag: per slice 2 planes x 32 lanes x 16 bytes), and a
// warp loads its A fragments with two coalesced 16-byte loads per slice.  The
// warp writes the slice's fresh V values into a shared tile transposed by
// column (VT[plane][col][row], bytes), from which the B fragments are read.
//
// Rows outside SELL slices (long rows, CSR / COO_S groups, zero rows) take the
// scalar path and add their projection with shared-memory atomics.
#pragma once

#include "block.cuh"

namespace ffspmv {

constexpr int SMMA_WARPS = 8;
constexpr int SMMA_KMAX = 16;     // iterate columns handled by the fused kernel (k <= 16)
constexpr int SMMA_FOLD = 512;    // slices between s32 -> u64 folds
// byte stride of the hi / lo planes of the transposed limb tile VT[plane][col][row]
// in the k <= 16 half-slice kernels (k_seq_step_h)
constexpr int SEQ_VT_PLANE = SMMA_KMAX * 32;

// NR consecutive rows x 4 columns per lane: KPV = k/4 lanes per row (1, 2,
// 4), G = 32/KPV row groups, group g owns rows NR*g .. NR*g+NR-1, so a lane's
// values of one column pack into NR bytes of the transposed tile.
template <int KPV>
struct SeqShape {
    static constexpr int G = 32 / KPV;   // row groups
    static constexpr int NR = 32 / G;    // rows per lane (= KPV)
    static_assert(NR <= 4, "fused MMA path: k <= 16");
};

__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// U fragment layout for slice s (ku <= 16): plane q (0 = hi, 1 = lo), lane,
// register j: bytes b = 0..3 hold U_q[row r][col a] with
//   a = (lane >> 2) + 8 * (j & 1),  r = (lane & 3) * 4 + 16 * (j >> 1) + b
// (the m16n8k32 A-operand layout, A[a][r] = U[r][a]).
__global__ void k_seq_ufrag(const uint32_t *__restrict__ U, uint32_t ku, const uint32_t *__restrict__ perm,
                            const SliceHdr *__restrict__ slices, uint32_t nslices,
                            uint32_t *__restrict__ ufrag) {
    const uint64_t total = (uint64_t)nslices * 2 * 32 * 4;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = i & 3, lane = (i >> 2) & 31, q = (i >> 7) & 1;
        const uint64_t s = i >> 8;
        const uint32_t a = (lane >> 2) + 8 * (j & 1);
        const uint32_t nrows = slices[s].nrows;
        uint32_t word = 0;
        for (uint32_t b = 0; b < 4; ++b) {
            const uint32_t r = (lane & 3) * 4 + 16 * (j >> 1) + b;
            uint32_t v = 0;
            if (r < nrows && a < ku) {
                const uint32_t row = perm[s * 32 + r];
                const uint32_t u = U[(uint64_t)row * ku + a];
                v = q == 0 ? (u >> 8) & 0xFFu : u & 0xFFu;
            }
            word |= v << (8 * b);
        }
        ufrag[i] = word;
    }
}

// Per-warp u64 projection accumulators live in shared memory,
// p64[(nt*4 + e)*32 + lane] (lane-contiguous: conflict-free), so no
// accumulator state stays in registers across slices: each slice's MMAs start
// from zero and are folded into p64 right away.
constexpr int SMMA_P64 = (SMMA_KMAX / 8) * 4 * 32;   // u64 per warp

// SpMM of one SELL slice (u16 iterate, 4 columns per lane) + its projection.
template <class Acc, class VT, int KPV>
__device__ __forceinline__ void seq_slice_mma(const DevOp &op, const DevMod &M, uint32_t s,
                                              const SliceHdr &h, uint32_t lane, uint32_t k,
                                              const uint16_t *__restrict__ Vin,
                                              uint16_t *__restrict__ Vout,
                                              const uint32_t *__restrict__ ufrag,
                                              uint8_t *vt, unsigned long long *p64) {
    using S = SeqShape<KPV>;
    const uint32_t g = lane / KPV, cl = lane % KPV;
    const uint32_t col = cl * 4;
    const bool colok = col < k;
    const uint32_t m = M.m;
    const uint32_t *pc = op.pcol + h.off_p + lane;
    const uint32_t *vc = op.vcol + h.off_v + lane;
    const VT *vv = reinterpret_cast<const VT *>(op.vval) + h.off_v + lane;
    const uint32_t wp = h.wp, wv = h.wv;
    const uint32_t rbase = g * S::NR;
    Acc acc[S::NR][4];
    uint32_t cw = wp ? ld_bcast(pc) : PAD_COL;
    for (uint32_t j = 0; j < wp; ++j) {
        const uint32_t cur = cw;
        if (j + 1 < wp) cw = ld_bcast(pc + (j + 1) * 32);
        uint32_t xv[S::NR][4], cs[S::NR];
#pragma unroll
        for (int i = 0; i < S::NR; ++i) {
            cs[i] = __shfl_sync(0xFFFFFFFFu, cur, rbase + i);
            ld_vec_pred<uint16_t, 4>(Vin + ((cs[i] & COL_MASK) * k + col), cs[i] != PAD_COL && colok,
                                     xv[i]);
        }
#pragma unroll
        for (int i = 0; i < S::NR; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[i][c].add((cs[i] & SIGN_BIT) ? m - xv[i][c] : xv[i][c]);
    }
    uint32_t vw = wv ? ld_bcast(vc) : PAD_COL;
    uint32_t aw = wv ? ld_bcast(vv) : 0u;
    for (uint32_t j = 0; j < wv; ++j) {
        const uint32_t cur = vw, cura = aw;
        if (j + 1 < wv) { vw = ld_bcast(vc + (j + 1) * 32); aw = ld_bcast(vv + (j + 1) * 32); }
        uint32_t xv[S::NR][4], as[S::NR];
#pragma unroll
        for (int i = 0; i < S::NR; ++i) {
            const uint32_t c = __shfl_sync(0xFFFFFFFFu, cur, rbase + i);
            as[i] = __shfl_sync(0xFFFFFFFFu, cura, rbase + i);
            ld_vec_pred<uint16_t, 4>(Vin + (c * k + col), c != PAD_COL && colok, xv[i]);
        }
#pragma unroll
        for (int i = 0; i < S::NR; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[i][c].mad(as[i], xv[i][c]);
    }
    // residues -> V_{t+1} (8-byte stores) and the transposed limb tile
    uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < S::NR; ++i) {
        const uint32_t r = rbase + i;
        uint32_t v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = acc[i][c].reduce(M);
        if (r < h.nrows && colok) {
            const uint32_t row = op.perm[s * 32 + r];
            uint2 w;
            w.x = v[0] | (v[1] << 16);
            w.y = v[2] | (v[3] << 16);
            *reinterpret_cast<uint2 *>(Vout + (uint64_t)row * k + col) = w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = 0;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            hi[c] |= ((v[c] >> 8) & 0xFFu) << (8 * i);
            lo[c] |= (v[c] & 0xFFu) << (8 * i);
        }
    }
    // VT[plane][col][row]: 32 x 32 bytes per plane; this lane owns rows
    // rbase .. rbase+NR-1 (NR bytes, NR-aligned) of columns col..col+3
    if (colok) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint8_t *ph = vt + (col + c) * 32 + rbase, *pl = ph + 32 * 32;
            if constexpr (S::NR == 4) {
                *reinterpret_cast<uint32_t *>(ph) = hi[c];
                *reinterpret_cast<uint32_t *>(pl) = lo[c];
            } else if constexpr (S::NR == 2) {
                *reinterpret_cast<uint16_t *>(ph) = (uint16_t)hi[c];
                *reinterpret_cast<uint16_t *>(pl) = (uint16_t)lo[c];
            } else {
                *ph = (uint8_t)hi[c];
                *pl = (uint8_t)lo[c];
            }
        }
    }
    __syncwarp();
    // A fragments (U limbs) of this slice: two coalesced 16-byte loads
    const uint4 ah4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256) + lane);
    const uint4 al4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256 + 128) + lane);
    const uint32_t ah[4] = {ah4.x, ah4.y, ah4.z, ah4.w}, al[4] = {al4.x, al4.y, al4.z, al4.w};
    const uint32_t gid = lane >> 2, tig = lane & 3;
    const int ntiles = (int)((k + 7) / 8);
#pragma unroll
    for (int nt = 0; nt < SMMA_KMAX / 8; ++nt) {
        if (nt >= ntiles) break;
        const uint32_t b = nt * 8 + gid;
        uint32_t bh[2], bl[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const uint32_t off = b * 32 + tig * 4 + 16 * jj;
            bh[jj] = *reinterpret_cast<const uint32_t *>(vt + off);
            bl[jj] = *reinterpret_cast<const uint32_t *>(vt + 32 * 32 + off);
        }
        // U^T V = 2^16 Uh^T Vh + 2^8 (Uh^T Vl + Ul^T Vh) + Ul^T Vl; one slice
        // adds at most 32 * 255^2 per element (x2 for the cross term): s32-exact
        int hh[4] = {0, 0, 0, 0}, cr[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
        mma_u8(hh, ah, bh);
        mma_u8(cr, ah, bl);
        mma_u8(cr, al, bh);
        mma_u8(ll, al, bl);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            p64[(nt * 4 + e) * 32 + lane] += ((unsigned long long)(uint32_t)hh[e] << 16) +
                                             ((unsigned long long)(uint32_t)cr[e] << 8) +
                                             (uint32_t)ll[e];
    }
    __syncwarp();
}

// Output policy of the scalar path inside the fused kernel: V_{t+1} and the
// projection through shared-memory u64 atomics (rare rows only).
struct SeqScalarOut {
    uint16_t *V;
    const uint32_t *U;
    uint32_t k, ku;
    unsigned long long *pn;   // shared [ku][k]
    __device__ __forceinline__ void put(uint32_t row, uint32_t col, bool colok, uint32_t r,
                                        const DevMod &) {
        if (!colok) return;
        V[(uint64_t)row * k + col] = (uint16_t)r;
        if (r == 0) return;
        for (uint32_t a = 0; a < ku; ++a)
            atomicAdd(pn + a * k + col, (unsigned long long)U[(uint64_t)row * ku + a] * r);
    }
};

template <class VT, int KPV, int KP>
__global__ void __launch_bounds__(SMMA_WARPS * 32, 2)
k_seq_step_mma(DevOp op, DevMod M, uint32_t k, uint32_t ku, const uint16_t *__restrict__ Vin,
               uint16_t *__restrict__ Vout, const uint32_t *__restrict__ U,
               const uint32_t *__restrict__ ufrag, uint32_t *__restrict__ part_out,
               const uint32_t *__restrict__ part_prev, uint32_t nprev, uint32_t *__restrict__ S_prev) {
    __shared__ __align__(16) uint8_t vts[SMMA_WARPS][2 * 32 * 32];
    __shared__ unsigned long long pn[16 * SMMA_KMAX];
    __shared__ unsigned long long p64s[SMMA_WARPS][SMMA_P64];
    __shared__ uint32_t red[SMMA_WARPS][16][SMMA_KMAX];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * SMMA_WARPS + warp, nw = gridDim.x * SMMA_WARPS;
    const uint32_t pairs = ku * k;
    for (uint32_t i = threadIdx.x; i < 16 * SMMA_KMAX; i += SMMA_WARPS * 32) pn[i] = 0;
    for (uint32_t i = lane; i < SMMA_P64; i += 32) p64s[warp][i] = 0;
    __syncthreads();
    // finalise the previous step's S from its CTA partials
    for (uint32_t p = gw; part_prev && p < pairs; p += nw) {
        uint64_t s = 0;
        for (uint32_t c = lane; c < nprev; c += 32) s += part_prev[(uint64_t)c * pairs + p];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) S_prev[p] = mod64(s, M);
    }
    unsigned long long *p64 = p64s[warp];
    SeqScalarOut sout{Vout, U, k, ku, pn};
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    for (uint32_t w = gw; w < items; w += nw) {
        if (w >= op.n_long && w - op.n_long < op.n_slices) {
            const uint32_t s = w - op.n_long;
            const SliceHdr h = load_hdr_b(op.slices + s);
            switch (h.regime) {
                case ACC32: seq_slice_mma<Acc32, VT, KPV>(op, M, s, h, lane, k, Vin, Vout, ufrag, vts[warp], p64); break;
                default: seq_slice_mma<Acc64, VT, KPV>(op, M, s, h, lane, k, Vin, Vout, ufrag, vts[warp], p64); break;
            }
        } else {
            block_item<VT, KP, 8>(op, M, w, lane, k, Vin, k, sout);
        }
    }
    const int ntiles = (int)((k + 7) / 8);
    // C fragment: element e of n-tile nt is (a = gid + 8*(e>>1), b = nt*8 + tig*2 + (e&1))
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < SMMA_KMAX / 8; ++nt) {
        if (nt >= ntiles) break;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t a = gid + 8 * (e >> 1), b = nt * 8 + tig * 2 + (e & 1);
            red[warp][a][b] = mod64(p64[(nt * 4 + e) * 32 + lane], M);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < pairs; i += SMMA_WARPS * 32) {
        const uint32_t a = i / k, b = i - a * k;
        uint64_t s = mod64(pn[a * k + b], M);
#pragma unroll
        for (int w = 0; w < SMMA_WARPS; ++w) s += red[w][a][b];
        part_out[(uint64_t)blockIdx.x * pairs + i] = mod64(s, M);
    }
}

// ------------------------------------------------ lean half-slice variant --
// k in {8, 16}: LPR = k / 8 lanes per row, each lane owns one row and 8
// iterate columns (one 16-byte gather per nonzero), and a warp walks a 32-row
// slice in LPR passes of 32 / LPR rows.  Per lane: 8 u32 accumulators for the
// +-1 part (a -1 adds m - x: < 2^32 for the <= 512 entries of a slice row)
// and 8 u64 accumulators for the valued part (products < 2^32).  The gathers
// of slot j+1 are issued before slot j is accumulated, and the index words
// are read two slots ahead.  ~60 registers -> 4 CTAs of 8 warps per SM.
__device__ __forceinline__ uint4 gather16(const uint16_t *__restrict__ V, uint32_t word, uint32_t k,
                                          uint32_t c0) {
    uint4 v = make_uint4(0, 0, 0, 0);
    const uint16_t *p = V + (uint64_t)(word & COL_MASK) * k + c0;
    asm volatile("{.reg .pred q; setp.ne.u32 q, %5, %6;\n"
                 "@q ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
                 : "l"(p), "r"(word), "r"(PAD_COL));
    return v;
}

template <class VT, int LPR>
__device__ __forceinline__ void seq_slice_h(const DevOp &op, const DevMod &M, uint32_t s,
                                            const SliceHdr &h, uint32_t lane, uint32_t k,
                                            const uint16_t *__restrict__ Vin,
                                            uint16_t *__restrict__ Vout,
                                            const uint32_t *__restrict__ ufrag, uint8_t *vt,
                                            unsigned long long *p64) {
    constexpr uint32_t RPP = 32 / LPR;
    const uint32_t m = M.m, wp = h.wp, wv = h.wv;
    const uint32_t c0 = (lane % LPR) * 8;
    const uint32_t *pc = op.pcol + h.off_p + lane;
    const uint32_t *vc = op.vcol + h.off_v + lane;
    const VT *vv = reinterpret_cast<const VT *>(op.vval) + h.off_v + lane;
#pragma unroll
    for (uint32_t pass = 0; pass < (uint32_t)LPR; ++pass) {
        const uint32_t rl = pass * RPP + lane / LPR;
        uint32_t a32[8];
        unsigned long long a64[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { a32[i] = 0; a64[i] = 0; }
        // +-1 slots: x, or m - x for a -1 (sign bit of the index word)
        {
            uint32_t w1 = wp > 1 ? ld_bcast(pc + 32) : PAD_COL;
            uint32_t c = __shfl_sync(0xFFFFFFFFu, wp ? ld_bcast(pc) : PAD_COL, rl);
            uint4 x = gather16(Vin, c, k, c0);
            for (uint32_t j = 0; j < wp; ++j) {
                const uint32_t w2 = j + 2 < wp ? ld_bcast(pc + (j + 2) * 32) : PAD_COL;
                const uint32_t cn = __shfl_sync(0xFFFFFFFFu, w1, rl);
                const uint4 xn = gather16(Vin, cn, k, c0);
                // -1: (v ^ ~0) + (m + 1) = m - v  (mod 2^32)
                const uint32_t sm = (c & SIGN_BIT) && c != PAD_COL ? 0xFFFFFFFFu : 0u, sa = sm & (m + 1);
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a32[2 * i] += ((xs[i] & 0xFFFFu) ^ sm) + sa;
                    a32[2 * i + 1] += ((xs[i] >> 16) ^ sm) + sa;
                }
                c = cn;
                x = xn;
                w1 = w2;
            }
        }
        // valued slots
        {
            uint32_t w1 = wv > 1 ? ld_bcast(vc + 32) : PAD_COL;
            uint32_t v1 = wv > 1 ? ld_bcast(vv + 32) : 0u;
            uint32_t c = __shfl_sync(0xFFFFFFFFu, wv ? ld_bcast(vc) : PAD_COL, rl);
            uint32_t a = __shfl_sync(0xFFFFFFFFu, wv ? ld_bcast(vv) : 0u, rl);
            uint4 x = gather16(Vin, c, k, c0);
            for (uint32_t j = 0; j < wv; ++j) {
                const uint32_t w2 = j + 2 < wv ? ld_bcast(vc + (j + 2) * 32) : PAD_COL;
                const uint32_t v2 = j + 2 < wv ? ld_bcast(vv + (j + 2) * 32) : 0u;
                const uint32_t cn = __shfl_sync(0xFFFFFFFFu, w1, rl);
                const uint32_t an = __shfl_sync(0xFFFFFFFFu, v1, rl);
                const uint4 xn = gather16(Vin, cn, k, c0);
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a64[2 * i] += (unsigned long long)a * (xs[i] & 0xFFFFu);
                    a64[2 * i + 1] += (unsigned long long)a * (xs[i] >> 16);
                }
                c = cn;
                a = an;
                x = xn;
                w1 = w2;
                v1 = v2;
            }
        }
        // residues -> V_{t+1} (one 16-byte store) and the transposed limb
        // tile VT[plane][col][row] (bytes) for the projection
        // row sums < 512 (2^32 + 2^16) < 2^48 (slice rows hold <= long_row <=
        // 65535 entries: < 2^48 as well)
        uint32_t r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = mod48(a64[i] + a32[i], M);
        if (rl >= h.nrows) {
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = 0;
        } else if (c0 < k) {
            const uint32_t row = op.perm[s * 32 + rl];
            *reinterpret_cast<uint4 *>(Vout + (uint64_t)row * k + c0) =
                make_uint4(r[0] | r[1] << 16, r[2] | r[3] << 16, r[4] | r[5] << 16, r[6] | r[7] << 16);
        }
        if (c0 < k) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                vt[(c0 + i) * 32 + rl] = (uint8_t)(r[i] >> 8);
                vt[SEQ_VT_PLANE + (c0 + i) * 32 + rl] = (uint8_t)r[i];
            }
        }
    }
    __syncwarp();
    // projection of the slice: U^T V as in seq_slice_mma
    const uint4 ah4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256) + lane);
    const uint4 al4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256 + 128) + lane);
    const uint32_t ah[4] = {ah4.x, ah4.y, ah4.z, ah4.w}, al[4] = {al4.x, al4.y, al4.z, al4.w};
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < LPR; ++nt) {
        const uint32_t b = nt * 8 + gid;
        uint32_t bh[2], bl[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const uint32_t off = b * 32 + tig * 4 + 16 * jj;
            bh[jj] = *reinterpret_cast<const uint32_t *>(vt + off);
            bl[jj] = *reinterpret_cast<const uint32_t *>(vt + SEQ_VT_PLANE + off);
        }
        int hh[4] = {0, 0, 0, 0}, cr[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
        mma_u8(hh, ah, bh);
        mma_u8(cr, ah, bl);
        mma_u8(cr, al, bh);
        mma_u8(ll, al, bl);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            p64[(nt * 4 + e) * 32 + lane] += ((unsigned long long)(uint32_t)hh[e] << 16) +
                                             ((unsigned long long)(uint32_t)cr[e] << 8) +
                                             (uint32_t)ll[e];
    }
    __syncwarp();
}

// cp.async variant of seq_slice_h (the default for k in {8, 16}): the same
// lane map (LPR lanes per row, 8 iterate columns = one 16-byte gather per
// lane and nonzero) but all LPR passes at once (NR = LPR rows per lane) and
// the gathers landed in a per-warp shared-memory ring D slots ahead of the
// accumulation, the slot index words / values 2D slots ahead (as in
// block_slice_as: no in-flight load waits in a register, so the bytes in
// flight are bounded by shared memory, not by the accumulators' registers).
// The residues, V_{t+1} stores and the MMA projection are those of
// seq_slice_h.
#ifndef FFSPMV_SEQ_AS_D
#define FFSPMV_SEQ_AS_D 2
#endif
#ifndef FFSPMV_SEQ_A64
#define FFSPMV_SEQ_A64 0
#endif
template <int LPR>
struct SeqRing {
    static constexpr int D = FFSPMV_SEQ_AS_D;
    static constexpr uint32_t data_bytes = D * LPR * 32 * 16;
    static constexpr uint32_t bytes = data_bytes + 2 * D * 128 * 2;
};

template <class VT, int LPR>
__device__ __forceinline__ void seq_slice_as(const DevOp &op, const DevMod &M, uint32_t s,
                                             const SliceHdr &h, uint32_t lane, uint32_t k,
                                             const uint16_t *__restrict__ Vin,
                                             uint16_t *__restrict__ Vout,
                                             const uint32_t *__restrict__ ufrag, uint8_t *vt,
                                             unsigned long long *p64, unsigned char *ring) {
    constexpr int D = SeqRing<LPR>::D;
    constexpr int NR = LPR;                 // rows per lane (one pass over the slice)
    static_assert((D & (D - 1)) == 0, "ring depth must be a power of two");
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(ring);
    const uint32_t sdata = sbase + lane * 16;
    const uint32_t siw = sbase + SeqRing<LPR>::data_bytes, siv = siw + 2 * D * 128;
    const uint4 *data = reinterpret_cast<const uint4 *>(ring) + lane;
    const uint32_t *iw = reinterpret_cast<const uint32_t *>(ring + SeqRing<LPR>::data_bytes);
    const unsigned char *iv = ring + SeqRing<LPR>::data_bytes + 2 * D * 128;
    const uint32_t m = M.m, wp = h.wp, wt = h.wp + h.wv;
    const uint32_t c0 = (lane % LPR) * 8, g = lane / LPR;
    const bool colok = c0 < k;
    const uint16_t *Vc = Vin + c0;
    const uint32_t *pcl = op.pcol + h.off_p + lane;
    const uint32_t *vcl = op.vcol + h.off_v + lane - wp * 32;
    const unsigned char *vbl = reinterpret_cast<const unsigned char *>(op.vval) +
                               ((uint64_t)h.off_v - wp * 32) * sizeof(VT) + lane * 4;
    const bool vlane = lane < 8 * sizeof(VT);
    // +-1 addends in u32 (a -1 adds m - x: < 2^32 for <= 65535 entries) and
    // valued products in u64; FFSPMV_SEQ_A64 keeps both in the u64 (16 fewer
    // registers for NR = 2, one more instruction per +-1 addend)
#if FFSPMV_SEQ_A64
    constexpr int A32N = 1;
#else
    constexpr int A32N = NR;
#endif
    uint32_t a32[A32N][8];
    unsigned long long a64[NR][8];
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) { a64[i][c] = 0; if (i < A32N) a32[i][c] = 0; }
    // loaded now, used after the slot walk (its latency hides behind it)
    uint32_t prow[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) prow[i] = g * NR + i < h.nrows ? __ldg(op.perm + s * 32 + g * NR + i) : 0u;

    auto copy_idx = [&](uint32_t j) {
        const uint32_t q = (j & (2 * D - 1)) * 128;
        cp_async4(siw + q + lane * 4, j < wp ? pcl + j * 32 : vcl + j * 32, 4);
        if (j >= wp && vlane) cp_async4(siv + q + lane * 4, vbl + (uint64_t)j * 32 * sizeof(VT), 4);
    };
    // a lane's NR rows are consecutive (g NR .. g NR + NR - 1): one vector
    // load of their index words / values per slot
    auto copy_data = [&](uint32_t j) {
        uint32_t w[NR];
        lds_vec<uint32_t, NR>(iw + (j & (2 * D - 1)) * 32 + g * NR, w);
        const uint32_t dst = sdata + (j & (D - 1)) * (NR * 512);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const uint32_t c = w[i];
            const bool ok = c != PAD_COL && colok;
            cp_async_v<16>(dst + i * 512, Vc + (ok ? (c & COL_MASK) * k : 0u), ok ? 16u : 0u);
        }
    };
    // KIND: 0 = +-1 slot, 1 = valued, 2 = decided by j < wp (see block_slice_as)
    auto consume = [&](uint32_t j, auto kind) {
        constexpr int KIND = decltype(kind)::value;
        const uint4 *d = data + (j & (D - 1)) * (NR * 32);
        const uint32_t q = j & (2 * D - 1);
        uint32_t wa[NR];     // the rows' index words (+-1: sign) or values
        if (KIND == 0 || (KIND == 2 && j < wp)) lds_vec<uint32_t, NR>(iw + q * 32 + g * NR, wa);
        else lds_vec<VT, NR>(iv + q * 128 + g * NR * sizeof(VT), wa);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const uint4 v = d[i * 32];
            const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
            if (KIND == 0 || (KIND == 2 && j < wp)) {
                // -1: (x ^ ~0) + (m + 1) = m - x (mod 2^32)
                const uint32_t sm = (uint32_t)((int32_t)wa[i] >> 31), sa = sm & (m + 1);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
#if FFSPMV_SEQ_A64
                    a64[i][2 * c] += ((xs[c] & 0xFFFFu) ^ sm) + sa;
                    a64[i][2 * c + 1] += ((xs[c] >> 16) ^ sm) + sa;
#else
                    a32[i][2 * c] += ((xs[c] & 0xFFFFu) ^ sm) + sa;
                    a32[i][2 * c + 1] += ((xs[c] >> 16) ^ sm) + sa;
#endif
                }
            } else {
                const uint32_t a = wa[i];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    a64[i][2 * c] += (unsigned long long)a * (xs[c] & 0xFFFFu);
                    a64[i][2 * c + 1] += (unsigned long long)a * (xs[c] >> 16);
                }
            }
        }
    };
    auto wait_sync = [&]() {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        __syncwarp();
    };
    auto commit = []() { asm volatile("cp.async.commit_group;" ::: "memory"); };
    for (uint32_t t = 0; t < 2 * D; ++t) {
        if (t >= (uint32_t)D) {
            wait_sync();
            if (t - D < wt) copy_data(t - D);
        }
        if (t < wt) copy_idx(t);
        commit();
    }
    using PM = std::integral_constant<int, 0>;
    using VAL = std::integral_constant<int, 1>;
    using ANY = std::integral_constant<int, 2>;
    uint32_t j = 0;
    // split at wp for k = 16 (c5: 0.225 -> 0.215 ms/step); k = 8 keeps one
    // loop (the 4-column block walk with two lanes per row was slower split)
    constexpr bool SPLIT = LPR >= 2;
    const uint32_t jend = wt > 2 * D ? wt - 2 * D : 0, jpm = SPLIT ? min(wp, jend) : 0u;
#pragma unroll 1
    for (; SPLIT && j < jpm; ++j) {
        wait_sync();
        consume(j, PM());
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
        __syncwarp();
        copy_idx(j + 2 * D);
        copy_data(j + D);
        commit();
    }
#pragma unroll 1
    for (; j < wt; ++j) {
        wait_sync();
        consume(j, ANY());
        __syncwarp();
        if (j + D < wt) copy_data(j + D);
        commit();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    // U fragments of the slice: loaded before the residue arithmetic they wait behind
    const uint4 ah4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256) + lane);
    const uint4 al4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256 + 128) + lane);
    // residues -> V_{t+1} and the transposed limb tile (as seq_slice_h); the
    // lane's NR rows are adjacent in the tile, so NR = 2 writes both rows'
    // bytes of a column with one 16-bit store per plane
    uint32_t r[NR][8];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const uint32_t rl = g * NR + i;
#pragma unroll
        for (int c = 0; c < 8; ++c) r[i][c] = mod48(a64[i][c] + (FFSPMV_SEQ_A64 ? 0u : a32[i < A32N ? i : 0][c]), M);
        if (rl >= h.nrows) {
#pragma unroll
            for (int c = 0; c < 8; ++c) r[i][c] = 0;
        } else if (colok) {
            *reinterpret_cast<uint4 *>(Vout + (uint64_t)prow[i] * k + c0) =
                make_uint4(r[i][0] | r[i][1] << 16, r[i][2] | r[i][3] << 16, r[i][4] | r[i][5] << 16,
                           r[i][6] | r[i][7] << 16);
        }
    }
    if (colok) {
        if constexpr (NR == 2) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t off = (c0 + c) * 32 + g * 2;
                *reinterpret_cast<uint16_t *>(vt + off) = (uint16_t)((r[0][c] >> 8) | (r[1][c] & 0xFF00u));
                *reinterpret_cast<uint16_t *>(vt + SEQ_VT_PLANE + off) = (uint16_t)((r[0][c] & 0xFFu) | (r[1][c] & 0xFFu) << 8);
            }
        } else {
#pragma unroll
            for (int i = 0; i < NR; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    vt[(c0 + c) * 32 + g * NR + i] = (uint8_t)(r[i][c] >> 8);
                    vt[SEQ_VT_PLANE + (c0 + c) * 32 + g * NR + i] = (uint8_t)r[i][c];
                }
        }
    }
    __syncwarp();
    const uint32_t ah[4] = {ah4.x, ah4.y, ah4.z, ah4.w}, al[4] = {al4.x, al4.y, al4.z, al4.w};
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < LPR; ++nt) {
        const uint32_t b = nt * 8 + gid;
        uint32_t bh[2], bl[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const uint32_t off = b * 32 + tig * 4 + 16 * jj;
            bh[jj] = *reinterpret_cast<const uint32_t *>(vt + off);
            bl[jj] = *reinterpret_cast<const uint32_t *>(vt + SEQ_VT_PLANE + off);
        }
        int hh[4] = {0, 0, 0, 0}, cr[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
        mma_u8(hh, ah, bh);
        mma_u8(cr, ah, bl);
        mma_u8(cr, al, bh);
        mma_u8(ll, al, bl);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            p64[(nt * 4 + e) * 32 + lane] += ((unsigned long long)(uint32_t)hh[e] << 16) +
                                             ((unsigned long long)(uint32_t)cr[e] << 8) +
                                             (uint32_t)ll[e];
    }
    __syncwarp();
}

// rows outside SELL slices (long rows, CSR / COO_S groups, zero rows): kept
// out of line so their register needs do not constrain the slice path
// (reads the operator view from a device copy: taking the address of the
// kernel parameter would move it to local memory for the whole kernel)
template <class VT, int KP>
__device__ __noinline__ void seq_item_scalar(const DevOp *__restrict__ opg, const DevMod M, uint32_t w,
                                             uint32_t lane, uint32_t k, const uint16_t *__restrict__ Vin,
                                             SeqScalarOut o) {
    const DevOp op = *opg;
    block_item<VT, KP, 8>(op, M, w, lane, k, Vin, k, o);
}

#ifndef FFSPMV_SEQ_AS
#define FFSPMV_SEQ_AS 1          // 1: seq_slice_as (cp.async ring), 0: seq_slice_h
#endif
#ifndef FFSPMV_SEQ_MINB
#define FFSPMV_SEQ_MINB 3
#endif
template <class VT, int LPR>
__global__ void __launch_bounds__(SMMA_WARPS * 32, FFSPMV_SEQ_MINB)
k_seq_step_h(DevOp op, const DevOp *__restrict__ opdev, DevMod M, uint32_t k, uint32_t ku,
             const uint16_t *__restrict__ Vin,
             uint16_t *__restrict__ Vout, const uint32_t *__restrict__ U,
             const uint32_t *__restrict__ ufrag, uint32_t *__restrict__ part_out,
             const uint32_t *__restrict__ part_prev, uint32_t nprev, uint32_t *__restrict__ S_prev,
             uint32_t *__restrict__ ctr, uint32_t *__restrict__ ctr_next) {
    __shared__ __align__(16) uint8_t vts[SMMA_WARPS][2 * SEQ_VT_PLANE];
    __shared__ unsigned long long pn[16 * SMMA_KMAX];
    __shared__ unsigned long long p64s[SMMA_WARPS][SMMA_P64];
    extern __shared__ __align__(16) unsigned char seq_ring[];
    // the CTA's final reduction tile: aliases each warp's own ring (idle once
    // the warp has no items left) on the cp.async path
    typedef uint32_t RedTile[16][SMMA_KMAX];
    static_assert(sizeof(RedTile) <= SeqRing<1>::bytes, "reduction tile fits a warp's ring");
#if FFSPMV_SEQ_AS
    auto red = [&](uint32_t w) -> RedTile & { return *reinterpret_cast<RedTile *>(seq_ring + w * SeqRing<LPR>::bytes); };
#else
    __shared__ RedTile red_s[SMMA_WARPS];
    auto red = [&](uint32_t w) -> RedTile & { return red_s[w]; };
#endif
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * SMMA_WARPS + warp, nw = gridDim.x * SMMA_WARPS;
    const uint32_t pairs = ku * k;
    for (uint32_t i = threadIdx.x; i < 16 * SMMA_KMAX; i += SMMA_WARPS * 32) pn[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ctr_next = 0;   // the next step's work counter
    for (uint32_t i = lane; i < SMMA_P64; i += 32) p64s[warp][i] = 0;
    __syncthreads();
    for (uint32_t p = gw; part_prev && p < pairs; p += nw) {
        uint64_t sacc = 0;
        for (uint32_t c = lane; c < nprev; c += 32) sacc += part_prev[(uint64_t)c * pairs + p];
        for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xFFFFFFFFu, sacc, o);
        if (lane == 0) S_prev[p] = mod64(sacc, M);
    }
    unsigned long long *p64 = p64s[warp];
    SeqScalarOut sout{Vout, U, k, ku, pn};
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    // items (long rows first, then slices, groups, zero rows) are taken
    // dynamically from a per-step counter: a warp holding a long row or a
    // wide slice takes fewer items (the skewed GL7d rows left the static
    // round-robin split waiting at the final barrier); the next item's
    // atomic is issued before the current item and read after it
    uint32_t w = 0;
    if (lane == 0) w = atomicAdd(ctr, 1u);
    w = __shfl_sync(0xFFFFFFFFu, w, 0);
    while (w < items) {
        uint32_t wn = 0;
        if (lane == 0) wn = atomicAdd(ctr, 1u);
        if (w >= op.n_long && w - op.n_long < op.n_slices) {
            const uint32_t s = w - op.n_long;
            const SliceHdr h = load_hdr_b(op.slices + s);
            if constexpr (FFSPMV_SEQ_AS) {
                seq_slice_as<VT, LPR>(op, M, s, h, lane, k, Vin, Vout, ufrag, vts[warp], p64,
                                      seq_ring + warp * SeqRing<LPR>::bytes);
            } else {
                seq_slice_h<VT, LPR>(op, M, s, h, lane, k, Vin, Vout, ufrag, vts[warp], p64);
            }
        } else {
            seq_item_scalar<VT, 8 * LPR>(opdev, M, w, lane, k, Vin, sout);
        }
        w = __shfl_sync(0xFFFFFFFFu, wn, 0);
    }
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < LPR; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t a = gid + 8 * (e >> 1), b = nt * 8 + tig * 2 + (e & 1);
            red(warp)[a][b] = mod64(p64[(nt * 4 + e) * 32 + lane], M);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < pairs; i += SMMA_WARPS * 32) {
        const uint32_t a = i / k, b = i - a * k;
        uint64_t sacc = mod64(pn[a * k + b], M);
#pragma unroll
        for (int w = 0; w < SMMA_WARPS; ++w) sacc += red(w)[a][b];
        part_out[(uint64_t)blockIdx.x * pairs + i] = mod64(sacc, M);
    }
}

// ------------------------------------------------ byte iterate (m <= 256) --
// k = 16, u8 iterate: one lane per row, its 16 columns gathered with one
// 16-byte load per nonzero (the iterate is half the bytes of the u16 one:
// P:631 "compressed" vectors for small fields).  Every addend is at most
// max(m, (m-1)^2) <= 65025 and a slice row holds at most long_row <= 65535
// entries, so a row's sum stays below 2^32: one u32 accumulator per column.
// The projection needs one u8 x u8 MMA per n-tile (single-limb residues).
__device__ __forceinline__ uint4 gather16b(const uint8_t *__restrict__ V, uint32_t word) {
    uint4 v = make_uint4(0, 0, 0, 0);
    const uint8_t *p = V + (uint64_t)(word & COL_MASK) * 16;
    asm volatile("{.reg .pred q; setp.ne.u32 q, %5, %6;\n"
                 "@q ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
                 : "l"(p), "r"(word), "r"(PAD_COL));
    return v;
}

template <class VT>
__device__ __forceinline__ void seq_slice_b(const DevOp &op, const DevMod &M, uint32_t s,
                                            const SliceHdr &h, uint32_t lane,
                                            const uint8_t *__restrict__ Vin,
                                            uint8_t *__restrict__ Vout,
                                            const uint32_t *__restrict__ ufrag, uint8_t *vt,
                                            unsigned long long *p64) {
    const uint32_t m = M.m, wp = h.wp, wv = h.wv;
    const uint32_t *pc = op.pcol + h.off_p + lane;
    const uint32_t *vc = op.vcol + h.off_v + lane;
    const VT *vv = reinterpret_cast<const VT *>(op.vval) + h.off_v + lane;
    uint32_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    // the output row and the U fragments, loaded now and used after the walk
    const uint32_t prow = lane < h.nrows ? __ldg(op.perm + s * 32 + lane) : 0u;
    const uint4 al4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256 + 128) + lane);
    // +-1 slots: x, or m - x for a -1: (x ^ ~0) + (m + 1) = m - x (mod 2^32)
    {
        uint32_t c = wp ? ld_bcast(pc) : PAD_COL;
        uint32_t w1 = wp > 1 ? ld_bcast(pc + 32) : PAD_COL;
        uint4 x = gather16b(Vin, c);
        for (uint32_t j = 0; j < wp; ++j) {
            const uint32_t w2 = j + 2 < wp ? ld_bcast(pc + (j + 2) * 32) : PAD_COL;
            const uint4 xn = gather16b(Vin, w1);
            const uint32_t sm = (c & SIGN_BIT) && c != PAD_COL ? 0xFFFFFFFFu : 0u, sa = sm & (m + 1);
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += (((xs[i >> 2] >> (8 * (i & 3))) & 0xFFu) ^ sm) + sa;
            c = w1;
            x = xn;
            w1 = w2;
        }
    }
    {
        uint32_t c = wv ? ld_bcast(vc) : PAD_COL, a = wv ? ld_bcast(vv) : 0u;
        uint32_t w1 = wv > 1 ? ld_bcast(vc + 32) : PAD_COL, a1 = wv > 1 ? ld_bcast(vv + 32) : 0u;
        uint4 x = gather16b(Vin, c);
        for (uint32_t j = 0; j < wv; ++j) {
            const uint32_t w2 = j + 2 < wv ? ld_bcast(vc + (j + 2) * 32) : PAD_COL;
            const uint32_t a2 = j + 2 < wv ? ld_bcast(vv + (j + 2) * 32) : 0u;
            const uint4 xn = gather16b(Vin, w1);
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += a * ((xs[i >> 2] >> (8 * (i & 3))) & 0xFFu);
            c = w1;
            a = a1;
            x = xn;
            w1 = w2;
            a1 = a2;
        }
    }
    // residues -> V_{t+1} (one 16-byte store) and the transposed byte tile
    // VT[col][row] for the projection
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = mod32_min(acc[i], M);
    if (lane >= h.nrows) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = 0;
    } else {
        const uint32_t row = prow;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = r[4 * q] | r[4 * q + 1] << 8 | r[4 * q + 2] << 16 | r[4 * q + 3] << 24;
        *reinterpret_cast<uint4 *>(Vout + (uint64_t)row * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) vt[i * 32 + lane] = (uint8_t)r[i];
    __syncwarp();
    // projection: U^T V with single-limb residues (the U fragments' low plane)
    const uint32_t al[4] = {al4.x, al4.y, al4.z, al4.w};
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const uint32_t b = nt * 8 + gid;
        uint32_t bl[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) bl[jj] = *reinterpret_cast<const uint32_t *>(vt + b * 32 + tig * 4 + 16 * jj);
        int ll[4] = {0, 0, 0, 0};   // a slice adds at most 32 * 255^2: s32-exact
        mma_u8(ll, al, bl);
#pragma unroll
        for (int e = 0; e < 4; ++e) p64[(nt * 4 + e) * 32 + lane] += (uint32_t)ll[e];
    }
    __syncwarp();
}

// cp.async variant of seq_slice_b (the default): the lane's 16-byte row
// gathers land in a per-warp shared ring 2 slots ahead, index words / values
// 4 slots ahead (see seq_slice_as).
template <class VT>
__device__ __forceinline__ void seq_slice_b_as(const DevOp &op, const DevMod &M, uint32_t s,
                                               const SliceHdr &h, uint32_t lane,
                                               const uint8_t *__restrict__ Vin,
                                               uint8_t *__restrict__ Vout,
                                               const uint32_t *__restrict__ ufrag, uint8_t *vt,
                                               unsigned long long *p64, unsigned char *ring) {
    constexpr int D = SeqRing<1>::D;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(ring);
    const uint32_t sdata = sbase + lane * 16;
    const uint32_t siw = sbase + SeqRing<1>::data_bytes, siv = siw + 2 * D * 128;
    const uint4 *data = reinterpret_cast<const uint4 *>(ring) + lane;
    const uint32_t *iw = reinterpret_cast<const uint32_t *>(ring + SeqRing<1>::data_bytes);
    const unsigned char *iv = ring + SeqRing<1>::data_bytes + 2 * D * 128;
    const uint32_t m = M.m, wp = h.wp, wt = h.wp + h.wv;
    const uint32_t *pcl = op.pcol + h.off_p + lane;
    const uint32_t *vcl = op.vcol + h.off_v + lane - wp * 32;
    const unsigned char *vbl = reinterpret_cast<const unsigned char *>(op.vval) +
                               ((uint64_t)h.off_v - wp * 32) * sizeof(VT) + lane * 4;
    const bool vlane = lane < 8 * sizeof(VT);
    uint32_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    auto copy_idx = [&](uint32_t j) {
        const uint32_t q = (j & (2 * D - 1)) * 128;
        cp_async4(siw + q + lane * 4, j < wp ? pcl + j * 32 : vcl + j * 32, 4);
        if (j >= wp && vlane) cp_async4(siv + q + lane * 4, vbl + (uint64_t)j * 32 * sizeof(VT), 4);
    };
    auto copy_data = [&](uint32_t j) {
        const uint32_t c = iw[(j & (2 * D - 1)) * 32 + lane];
        const bool ok = c != PAD_COL;
        cp_async_v<16>(sdata + (j & (D - 1)) * 512, Vin + (ok ? (uint64_t)(c & COL_MASK) * 16 : 0u), ok ? 16u : 0u);
    };
    auto consume = [&](uint32_t j) {
        const uint4 v = data[(j & (D - 1)) * 32];
        const uint32_t q = j & (2 * D - 1);
        const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
        if (j < wp) {
            const uint32_t sm = (uint32_t)((int32_t)iw[q * 32 + lane] >> 31), sa = sm & (m + 1);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += (((xs[i >> 2] >> (8 * (i & 3))) & 0xFFu) ^ sm) + sa;
        } else {
            const uint32_t a = reinterpret_cast<const VT *>(iv + q * 128)[lane];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += a * ((xs[i >> 2] >> (8 * (i & 3))) & 0xFFu);
        }
    };
    auto wait_sync = [&]() {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        __syncwarp();
    };
    auto commit = []() { asm volatile("cp.async.commit_group;" ::: "memory"); };
    for (uint32_t t = 0; t < 2 * D; ++t) {
        if (t >= (uint32_t)D) {
            wait_sync();
            if (t - D < wt) copy_data(t - D);
        }
        if (t < wt) copy_idx(t);
        commit();
    }
    uint32_t j = 0;
#pragma unroll 1
    for (; j + 2 * D < wt; ++j) {
        wait_sync();
        consume(j);
        __syncwarp();
        copy_idx(j + 2 * D);
        copy_data(j + D);
        commit();
    }
#pragma unroll 1
    for (; j < wt; ++j) {
        wait_sync();
        consume(j);
        __syncwarp();
        if (j + D < wt) copy_data(j + D);
        commit();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = mod32_min(acc[i], M);
    if (lane >= h.nrows) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = 0;
    } else {
        const uint32_t row = op.perm[s * 32 + lane];
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = r[4 * q] | r[4 * q + 1] << 8 | r[4 * q + 2] << 16 | r[4 * q + 3] << 24;
        *reinterpret_cast<uint4 *>(Vout + (uint64_t)row * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) vt[i * 32 + lane] = (uint8_t)r[i];
    __syncwarp();
    const uint4 al4 = __ldg(reinterpret_cast<const uint4 *>(ufrag + (uint64_t)s * 256 + 128) + lane);
    const uint32_t al[4] = {al4.x, al4.y, al4.z, al4.w};
    const uint32_t gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const uint32_t b = nt * 8 + gid;
        uint32_t bl[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) bl[jj] = *reinterpret_cast<const uint32_t *>(vt + b * 32 + tig * 4 + 16 * jj);
        int ll[4] = {0, 0, 0, 0};
        mma_u8(ll, al, bl);
#pragma unroll
        for (int e = 0; e < 4; ++e) p64[(nt * 4 + e) * 32 + lane] += (uint32_t)ll[e];
    }
    __syncwarp();
}

// the scalar path of the byte kernel (rows outside SELL slices)
struct SeqScalarOutB {
    uint8_t *V;
    const uint32_t *U;
    uint32_t k, ku;
    unsigned long long *pn;
    __device__ __forceinline__ void put(uint32_t row, uint32_t col, bool colok, uint32_t r,
                                        const DevMod &) {
        if (!colok) return;
        V[(uint64_t)row * k + col] = (uint8_t)r;
        if (r == 0) return;
        for (uint32_t a = 0; a < ku; ++a)
            atomicAdd(pn + a * k + col, (unsigned long long)U[(uint64_t)row * ku + a] * r);
    }
};

template <class VT, int KP>
__device__ __noinline__ void seq_item_scalar_b(const DevOp *__restrict__ opg, const DevMod M, uint32_t w,
                                               uint32_t lane, uint32_t k, const uint8_t *__restrict__ Vin,
                                               SeqScalarOutB o) {
    const DevOp op = *opg;
    block_item<VT, KP, 8>(op, M, w, lane, k, Vin, k, o);
}

#ifndef FFSPMV_SEQB_MINB
#define FFSPMV_SEQB_MINB 3
#endif
// The byte kernel keeps its register-landed gathers: measured on the square
// GL7d m = 3 sequence (tools/time_seq.py --config c3sq, dynamic item
// scheduling in both): 0.356 ms/step against 0.385 with the cp.async ring
// (one 16-byte gather per lane and slot: the ring's per-slot bookkeeping is
// not amortised, and the 30 MB byte iterate stays L2-resident).
#ifndef FFSPMV_SEQB_AS
#define FFSPMV_SEQB_AS 0
#endif
template <class VT>
__global__ void __launch_bounds__(SMMA_WARPS * 32, FFSPMV_SEQB_MINB)
k_seq_step_b(DevOp op, const DevOp *__restrict__ opdev, DevMod M, uint32_t k, uint32_t ku,
             const uint8_t *__restrict__ Vin, uint8_t *__restrict__ Vout, const uint32_t *__restrict__ U,
             const uint32_t *__restrict__ ufrag, uint32_t *__restrict__ part_out,
             const uint32_t *__restrict__ part_prev, uint32_t nprev, uint32_t *__restrict__ S_prev,
             uint32_t *__restrict__ ctr, uint32_t *__restrict__ ctr_next) {
    __shared__ __align__(16) uint8_t vts[SMMA_WARPS][32 * 32];
    __shared__ unsigned long long pn[16 * SMMA_KMAX];
    __shared__ unsigned long long p64s[SMMA_WARPS][SMMA_P64];
    // the CTA's final reduction tile of warp w aliases w's own p64 block
    // (its values are read into registers first): 8 KB less static shared
    typedef uint32_t RedTile[16][SMMA_KMAX];
    static_assert(sizeof(RedTile) <= sizeof(p64s[0]), "reduction tile fits a warp's p64 block");
    auto red = [&](uint32_t w) -> RedTile & { return *reinterpret_cast<RedTile *>(&p64s[w][0]); };
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * SMMA_WARPS + warp, nw = gridDim.x * SMMA_WARPS;
    const uint32_t pairs = ku * k;
    for (uint32_t i = threadIdx.x; i < 16 * SMMA_KMAX; i += SMMA_WARPS * 32) pn[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ctr_next = 0;   // the next step's work counter
    for (uint32_t i = lane; i < SMMA_P64; i += 32) p64s[warp][i] = 0;
    __syncthreads();
    for (uint32_t p = gw; part_prev && p < pairs; p += nw) {
        uint64_t sacc = 0;
        for (uint32_t c = lane; c < nprev; c += 32) sacc += part_prev[(uint64_t)c * pairs + p];
        for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xFFFFFFFFu, sacc, o);
        if (lane == 0) S_prev[p] = mod64(sacc, M);
    }
    unsigned long long *p64 = p64s[warp];
    SeqScalarOutB sout{Vout, U, k, ku, pn};
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    // items (long rows first, then slices, groups, zero rows) are taken
    // dynamically from a per-step counter: a warp holding a long row or a
    // wide slice takes fewer items (the skewed GL7d rows left the static
    // round-robin split waiting at the final barrier); the next item's
    // atomic is issued before the current item and read after it
    uint32_t w = 0;
    if (lane == 0) w = atomicAdd(ctr, 1u);
    w = __shfl_sync(0xFFFFFFFFu, w, 0);
    while (w < items) {
        uint32_t wn = 0;
        if (lane == 0) wn = atomicAdd(ctr, 1u);
        if (w >= op.n_long && w - op.n_long < op.n_slices) {
            const uint32_t s = w - op.n_long;
            const SliceHdr h = load_hdr_b(op.slices + s);
            if constexpr (FFSPMV_SEQB_AS) {
                extern __shared__ __align__(16) unsigned char seq_ring_b[];
                seq_slice_b_as<VT>(op, M, s, h, lane, Vin, Vout, ufrag, vts[warp], p64,
                                   seq_ring_b + warp * SeqRing<1>::bytes);
            } else {
                seq_slice_b<VT>(op, M, s, h, lane, Vin, Vout, ufrag, vts[warp], p64);
            }
        } else {
            seq_item_scalar_b<VT, 16>(opdev, M, w, lane, k, Vin, sout);
        }
        w = __shfl_sync(0xFFFFFFFFu, wn, 0);
    }
    const uint32_t gid = lane >> 2, tig = lane & 3;
    uint32_t pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) pr[nt][e] = mod64(p64[(nt * 4 + e) * 32 + lane], M);
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t a = gid + 8 * (e >> 1), b = nt * 8 + tig * 2 + (e & 1);
            red(warp)[a][b] = pr[nt][e];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < pairs; i += SMMA_WARPS * 32) {
        const uint32_t a = i / k, b = i - a * k;
        uint64_t sacc = mod64(pn[a * k + b], M);
#pragma unroll
        for (int w = 0; w < SMMA_WARPS; ++w) sacc += red(w)[a][b];
        part_out[(uint64_t)blockIdx.x * pairs + i] = mod64(sacc, M);
    }
}

}  // namespace ffspmv

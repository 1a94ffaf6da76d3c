// x-staged apply for k = 1 (north star "x tiles staged
// in shared memory").
//
// Measured on B200 (tools/gather_bench*.cu): a random 4-byte gather of x from
// L2 sustains ~240 G/s chip-wide, while a random gather from shared memory
// sustains ~1.6-2.0 T/s and a random shared u32 atomicAdd ~2.0 T/s.  For
// matrices whose columns have no locality (the synthetic SIMC / GL7d-shaped
// configs) the row layout is therefore bound by L2 gathers at ~25% of HBM
// bandwidth; this operator instead stages a panel of x in shared memory and
// accumulates the rows of a band in shared memory, so every nonzero costs one
// coalesced stream read, one shared gather and one shared atomic.
//
//   k_panel         persistent, one 1024-thread CTA per SM, walks its tile
//                   range (panel-major): stage x panel (192 KB), accumulate
//                   band rows, write one u32 per band row into partial[p][row]
//                   (the raw sum when m <= 2^16 -- it is < 2^32 -- else the
//                   residue of the two u32 halves)
//   k_panel_reduce  y[r] = alpha * sum_p partial[p][r] + beta * y[r]  (mod m)
#include "device.cuh"

namespace ffspmv {

void count_launch();

namespace {

constexpr int PANEL_THREADS = 1024;
constexpr int PANEL_GT = 512;      // threads per group (two groups per CTA)

// Shared memory: x panel (W * sizeof(IT)) | accumulators of the two thread
// groups (2 x (R + 1) u32, doubled when SPLIT) | tile-header cache (HC
// headers, 16-byte aligned).
template <bool SPLIT>
__host__ __device__ constexpr uint32_t panel_hc() { return SPLIT ? 16u : 64u; }
// u32 words per group accumulator block, a multiple of 4 (16-byte vectors)
template <bool SPLIT>
__host__ __device__ __forceinline__ uint32_t acc_stride(const PanelGeom &g) {
    return ((SPLIT ? 2 : 1) * (g.R + 1) + 3) / 4 * 4;
}
template <class IT, bool SPLIT>
__host__ __device__ __forceinline__ size_t hc_offset(const PanelGeom &g) {
    return ((size_t)g.W * sizeof(IT) + 2 * (size_t)acc_stride<SPLIT>(g) * 4 + 15) / 16 * 16;
}

// Shared-memory accesses through 32-bit shared addresses (no generic-address
// conversion in the hot loop).  `off` is a byte offset.
template <class IT>
__device__ __forceinline__ uint32_t lds_x(uint32_t base, uint32_t off) {
    uint32_t v;
    if constexpr (sizeof(IT) == 1) {
        unsigned short h;
        asm volatile("ld.shared.u8 %0, [%1];" : "=h"(h) : "r"(base + off));
        v = h;
    } else if constexpr (sizeof(IT) == 2) {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(base + off));
        v = h;
    } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + off));
    }
    return v;
}

// acc[row] += v (two u32 halves at acc and acc + hi_off when SPLIT: each half
// of a residue <= m < 2^32 is < 2^16, and a tile row has at most W < 2^16
// addends)
template <bool SPLIT>
__device__ __forceinline__ void acc_add_s(uint32_t acc_s, uint32_t hi_off, uint32_t row, uint32_t v) {
    if constexpr (SPLIT) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v & 0xFFFFu));
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + hi_off + 4 * row), "r"(v >> 16));
    } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v));
    }
}

// Stream quads: read once -> no L1 allocation, evict-first in L2.  Out of
// range (pred false) -> `dflt` in every lane, which the kernel treats as a
// padding word.
__device__ __forceinline__ uint4 ld_quad(const uint4 *p, bool pred, uint32_t dflt) {
    uint4 v = make_uint4(dflt, dflt, dflt, dflt);
    asm volatile(
        "{.reg .pred q; setp.ne.u32 q, %5, 0;\n"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"((uint32_t)pred), "l"(POLICY_EVICT_FIRST));
    return v;
}
// Raw values of one valued quad (4 x IT packed into .x / .x,.y / .x..w),
// 0 when pred is false; unpacked with vals().
template <class IT>
__device__ __forceinline__ uint4 ld_vraw(const void *base, uint64_t vq, bool pred) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if constexpr (sizeof(IT) == 1) {
        asm volatile("{.reg .pred q; setp.ne.u32 q, %2, 0;\n"
                     "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %3;}"
                     : "+r"(v.x) : "l"(reinterpret_cast<const uint32_t *>(base) + vq), "r"((uint32_t)pred),
                       "l"(POLICY_EVICT_FIRST));
    } else if constexpr (sizeof(IT) == 2) {
        asm volatile("{.reg .pred q; setp.ne.u32 q, %3, 0;\n"
                     "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %4;}"
                     : "+r"(v.x), "+r"(v.y) : "l"(reinterpret_cast<const uint2 *>(base) + vq), "r"((uint32_t)pred),
                       "l"(POLICY_EVICT_FIRST));
    } else {
        v = ld_quad(reinterpret_cast<const uint4 *>(base) + vq, pred, 0u);
    }
    return v;
}
template <class IT>
__device__ __forceinline__ void vals(const uint4 &v, uint32_t (&a)[4]) {
    if constexpr (sizeof(IT) == 1) {
        a[0] = v.x & 0xFFu; a[1] = (v.x >> 8) & 0xFFu; a[2] = (v.x >> 16) & 0xFFu; a[3] = v.x >> 24;
    } else if constexpr (sizeof(IT) == 2) {
        a[0] = v.x & 0xFFFFu; a[1] = v.x >> 16; a[2] = v.y & 0xFFFFu; a[3] = v.y >> 16;
    } else {
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
    }
}

// Bulk L2 prefetch of a tile's quads and value quads (16-byte granules).
__device__ __forceinline__ void prefetch_l2(const void *p, uint64_t bytes) {
    const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15, e = ((uintptr_t)p + bytes + 15) & ~(uintptr_t)15;
    for (uintptr_t q = a; q < e; q += 1u << 20) {
        const uint32_t n = (uint32_t)min((uintptr_t)(1u << 20), e - q);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(n) : "memory");
    }
}
template <class IT>
__device__ __forceinline__ void prefetch_tile(const DevPanel &op, const PanelTile &T) {
    const uint32_t nq = T.nqp + T.nqm + T.nqv;
    if (nq) prefetch_l2(reinterpret_cast<const uint4 *>(op.pent) + T.q0, 16ull * nq);
    if (T.nqv) prefetch_l2(reinterpret_cast<const unsigned char *>(op.vval) + 4ull * sizeof(IT) * T.vq0,
                           4ull * sizeof(IT) * T.nqv);
}

// x panel -> shared memory, converted to the narrow staged type.  Eight
// 16-byte loads per thread are issued before any store; four residues pack
// into one 4-byte (u8) or 8-byte (u16) shared store.
template <class IT>
__device__ __forceinline__ void stage_x(IT *sx, const uint32_t *__restrict__ x, uint64_t c0,
                                        uint32_t wn) {
    const uint32_t *src = x + c0;
    uint32_t done = 0;
    if (((uintptr_t)src & 15) == 0) {
        constexpr int U = 8;
        const uint32_t nvec = wn / 4;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        for (uint32_t base = threadIdx.x; base < nvec; base += U * PANEL_THREADS) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = base + u * PANEL_THREADS;
                v[u] = i < nvec ? __ldg(s4 + i) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = base + u * PANEL_THREADS;
                if (i < nvec) {
                    if constexpr (sizeof(IT) == 1) {
                        reinterpret_cast<uint32_t *>(sx)[i] =
                            __byte_perm(__byte_perm(v[u].x, v[u].y, 0x0040), __byte_perm(v[u].z, v[u].w, 0x0040), 0x5410);
                    } else if constexpr (sizeof(IT) == 2) {
                        reinterpret_cast<uint2 *>(sx)[i] =
                            make_uint2(__byte_perm(v[u].x, v[u].y, 0x5410), __byte_perm(v[u].z, v[u].w, 0x5410));
                    } else {
                        reinterpret_cast<uint4 *>(sx)[i] = v[u];
                    }
                }
            }
        }
        done = nvec * 4;
    }
    for (uint32_t i = done + threadIdx.x; i < wn; i += PANEL_THREADS) sx[i] = (IT)__ldg(src + i);
}

// a * b + c (mod 2^32) kept as one IMAD (the compiler otherwise rewrites
// q * (0 - m) + x as a negation plus a multiply-add)
__device__ __forceinline__ uint32_t mad32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// (a * x) mod m of a valued entry.  LAZY: the Barrett remainder before its
// correction, in [0, 2m) (mod32's argument; the builder checked that a tile
// row's sum of such terms stays < 2^32).
template <bool SPLIT, bool LAZY>
__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t xv, const DevMod &M) {
    if constexpr (SPLIT) return mod64((uint64_t)a * xv, M);
    else if constexpr (LAZY) {
        const uint32_t p = a * xv;
        return mad32(__umulhi(p, M.mu32), 0u - M.m, p);
    } else return mod32(a * xv, M);
}

// Processing of one quad of the tile; kind 0 / 1 / 2 = +1 / -1 / valued.
template <class IT, bool SPLIT, bool LAZY>
__device__ __forceinline__ void do_quad(uint32_t kind, const uint4 &w, const uint4 &raw,
                                        uint32_t sx_s, uint32_t acc_s, uint32_t hi_off, uint32_t rs,
                                        uint32_t rmask, const DevMod &M) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    if (kind == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc_add_s<SPLIT>(acc_s, hi_off, ws[u] & rmask, lds_x<IT>(sx_s, ws[u] >> rs));
    } else if (kind == 1) {
        // m - x <= m (x = 0 adds m: a multiple of m, harmless)
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc_add_s<SPLIT>(acc_s, hi_off, ws[u] & rmask, M.m - lds_x<IT>(sx_s, ws[u] >> rs));
    } else {
        uint32_t a[4];
        vals<IT>(raw, a);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc_add_s<SPLIT>(acc_s, hi_off, ws[u] & rmask,
                             mulmod<SPLIT, LAZY>(a[u], lds_x<IT>(sx_s, ws[u] >> rs), M));
    }
}

// x mod m for x < 2^32, m <= 2^16 (mod32_min with the multiply-add kept whole)
__device__ __forceinline__ uint32_t min32r(uint32_t x, const DevMod &M) {
    const uint32_t r = mad32(__umulhi(x, M.mu32), 0u - M.m, x);
    return min(r, r - M.m);
}

template <class IT, bool SPLIT, bool LAZY>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
k_panel(DevPanel op, DevMod M, const uint32_t *__restrict__ xin, IT *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    const PanelGeom g = op.g;
    IT *sx = reinterpret_cast<IT *>(smem);
    const uint32_t tid = threadIdx.x, grp = tid / PANEL_GT, gt = tid % PANEL_GT;
    // each thread group has its own band accumulators (R + 1 u32, twice when
    // SPLIT: the high halves follow the low ones)
    constexpr uint32_t AW = SPLIT ? 2 : 1;
    uint32_t *acc = reinterpret_cast<uint32_t *>(smem + (size_t)g.W * sizeof(IT)) + grp * acc_stride<SPLIT>(g);
    const uint32_t sx_s = (uint32_t)__cvta_generic_to_shared(sx);
    const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc);
    const uint32_t hi_off = 4 * (g.R + 1);
    const uint32_t rs = g.rs, rmask = (1u << g.rs) - 1, dummy = g.R;
    const uint32_t t0 = op.cta_t0[blockIdx.x], t1 = op.cta_t0[blockIdx.x + 1];
    const uint4 *pq = reinterpret_cast<const uint4 *>(op.pent);
    constexpr uint32_t HC = panel_hc<SPLIT>();
    for (uint32_t i = gt; i < AW * (g.R + 1); i += PANEL_GT) acc[i] = 0;
    auto bar_group = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(PANEL_GT) : "memory"); };
    // Software pipeline over a group's tiles: the first QR quads per thread
    // of its next tile (the whole tile when it has <= QR * PANEL_GT quads)
    // are loaded into registers before the current tile's write-out, so the
    // stream latency hides behind it.
    constexpr int QR = SPLIT ? 2 : 4;
    uint4 rw[QR], ra[QR];
    auto load_regs = [&](const PanelTile &T) {
        const uint32_t nq = T.nqp + T.nqm + T.nqv, ev = T.nqp + T.nqm;
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            const uint32_t q = gt + i * PANEL_GT;
            if (q < nq) {
                rw[i] = ld_quad(pq + T.q0 + q, true, dummy);
                ra[i] = ld_vraw<IT>(op.vval, (uint64_t)T.vq0 + (q - ev), q >= ev);
            }
        }
    };
    PanelTile *hc = reinterpret_cast<PanelTile *>(smem + hc_offset<IT, SPLIT>(g));
    // Segments: runs of the CTA's tiles with one x panel and at most HC
    // tiles.  A segment stages its panel and headers with the whole CTA; then
    // group 0 takes its even tiles and group 1 its odd tiles, each group
    // synchronising only its own 16 warps, so one group's write-out overlaps
    // the other's accumulation.
    for (uint32_t s0 = t0; s0 < t1;) {
        __syncthreads();                       // previous segment done with x and hc
        const uint32_t cnt = min(HC, t1 - s0);
        for (uint32_t i = tid; i < 2 * cnt; i += PANEL_THREADS)
            reinterpret_cast<uint4 *>(hc)[i] = __ldg(reinterpret_cast<const uint4 *>(op.tiles + s0) + i);
        const uint32_t p = __ldg(&op.tiles[s0].p);
        {
            const uint64_t c0 = (uint64_t)p * g.W;
            const uint32_t wn = (uint32_t)min((uint64_t)g.W, (uint64_t)op.cols - c0);
            stage_x<IT>(sx, xin, c0, wn);
        }
        __syncthreads();
        uint32_t n = 1;
        while (n < cnt && hc[n].p == p) ++n;
        if (grp < n) load_regs(hc[grp]);
        if (gt == 0 && grp + 2 < n) prefetch_tile<IT>(op, hc[grp + 2]);
        for (uint32_t j = grp; j < n; j += 2) {
            const PanelTile &T = hc[j];
            // the group's tile after next -> L2, so its register loads hit L2
            if (gt == 0 && j + 4 < n) prefetch_tile<IT>(op, hc[j + 4]);
            const uint32_t e1 = T.nqp, e2 = T.nqp + T.nqm, nq = e2 + T.nqv;
#pragma unroll
            for (int i = 0; i < QR; ++i) {
                const uint32_t q = gt + i * PANEL_GT;
                if (q < nq)
                    do_quad<IT, SPLIT, LAZY>(q < e1 ? 0u : q < e2 ? 1u : 2u, rw[i], ra[i], sx_s, acc_s,
                                             hi_off, rs, rmask, M);
            }
            // quads beyond the register ring: two per thread per round
            for (uint32_t q = gt + QR * PANEL_GT; q < nq; q += 2 * PANEL_GT) {
                const uint32_t qb = q + PANEL_GT;
                const uint4 w0 = ld_quad(pq + T.q0 + q, true, dummy);
                const uint4 w1 = ld_quad(pq + T.q0 + qb, qb < nq, dummy);
                const uint4 a0 = ld_vraw<IT>(op.vval, (uint64_t)T.vq0 + (q - e2), q >= e2);
                const uint4 a1 = ld_vraw<IT>(op.vval, (uint64_t)T.vq0 + (qb - e2), qb >= e2 && qb < nq);
                do_quad<IT, SPLIT, LAZY>(q < e1 ? 0u : q < e2 ? 1u : 2u, w0, a0, sx_s, acc_s, hi_off, rs, rmask, M);
                if (qb < nq)
                    do_quad<IT, SPLIT, LAZY>(qb < e1 ? 0u : qb < e2 ? 1u : 2u, w1, a1, sx_s, acc_s, hi_off, rs,
                                             rmask, M);
            }
            const uint32_t b = T.b, rn = T.rn;
            bar_group();                       // the tile's sums are complete
            if (j + 2 < n) load_regs(hc[j + 2]);
            // one residue per band row -> partial[p][row] (same narrow type
            // as the staged x); re-zero the accumulators.  Four rows per
            // thread per step: one conflict-free 16-byte shared load (lanes
            // read consecutive vectors) and one 4 * sizeof(IT)-byte store.
            // Without SPLIT the row sum is < 2^32 (checked by the builder)
            // and reduces with the 32-bit Barrett; SPLIT: the residue of lo +
            // hi * 2^16.  Rows rn .. round4(rn) hold zeros and land in the
            // padding of the last band.
            IT *out = partial + (uint64_t)p * g.rows_pad + (uint64_t)b * g.R;
            const uint32_t nv = (rn + 3) / 4;
            for (uint32_t v = gt; v < nv; v += PANEL_GT) {
                const uint4 s4 = reinterpret_cast<const uint4 *>(acc)[v];
                reinterpret_cast<uint4 *>(acc)[v] = make_uint4(0, 0, 0, 0);
                uint32_t res[4];
                if constexpr (SPLIT) {
                    const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t r = 4 * v + i;
                        res[i] = mod64((uint64_t)sv[i] + ((uint64_t)acc[g.R + 1 + r] << 16), M);
                        acc[g.R + 1 + r] = 0;
                    }
                    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(
                                     reinterpret_cast<uint4 *>(out) + v),
                                 "r"(res[0]), "r"(res[1]), "r"(res[2]), "r"(res[3]), "l"(POLICY_EVICT_LAST));
                } else {
                    res[0] = min32r(s4.x, M);
                    res[1] = min32r(s4.y, M);
                    res[2] = min32r(s4.z, M);
                    res[3] = min32r(s4.w, M);
                    if constexpr (sizeof(IT) == 1) {
                        asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(
                                         reinterpret_cast<uint32_t *>(out) + v),
                                     "r"(__byte_perm(__byte_perm(res[0], res[1], 0x0040),
                                                     __byte_perm(res[2], res[3], 0x0040), 0x5410)),
                                     "l"(POLICY_EVICT_LAST));
                    } else {
                        asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(
                                         reinterpret_cast<uint2 *>(out) + v),
                                     "r"(__byte_perm(res[0], res[1], 0x5410)), "r"(__byte_perm(res[2], res[3], 0x5410)),
                                     "l"(POLICY_EVICT_LAST));
                    }
                }
            }
            bar_group();                       // zeroing done before the next tile adds
        }
        s0 += n;
    }
}

// y[r] = alpha * sum_p partial[p][r] + beta * y[r]; VEC = 16 / sizeof(IT)
// consecutive rows per thread so each panel's partials load as one 16-byte
// vector (the partial row stride is a multiple of 16).
template <class IT>
__global__ void k_panel_reduce(const IT *__restrict__ partial, uint32_t P, uint32_t rows,
                               uint32_t rows_pad, DevMod M, uint32_t alpha, uint32_t beta,
                               uint32_t *__restrict__ y, bool y_aligned) {
    constexpr int VEC = 16 / sizeof(IT);
    const uint32_t nvec = (rows + VEC - 1) / VEC;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x) {
        uint64_t s[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) s[i] = 0;
        // P residues < 2^32: exact in u64; eight panels' loads in flight
        // (the partials are L2-resident: latency, not bandwidth, bounds this)
        constexpr uint32_t CH = 8;
        for (uint32_t p = 0; p < P; p += CH) {
            uint4 e4[CH];
#pragma unroll
            for (uint32_t j = 0; j < CH; ++j)
                e4[j] = p + j < P ? __ldcs(reinterpret_cast<const uint4 *>(partial + (uint64_t)(p + j) * rows_pad) + v)
                                  : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (uint32_t j = 0; j < CH; ++j) {
                const IT *e = reinterpret_cast<const IT *>(&e4[j]);
#pragma unroll
                for (int i = 0; i < VEC; ++i) s[i] += e[i];
            }
        }
        const uint32_t r0 = v * VEC;
        if (y_aligned && r0 + VEC <= rows) {
#pragma unroll
            for (int i = 0; i < VEC; i += 4) {
                uint4 yo = beta ? *reinterpret_cast<const uint4 *>(y + r0 + i) : make_uint4(0, 0, 0, 0);
                yo.x = epilogue(mod64(s[i], M), alpha, beta, yo.x, M);
                yo.y = epilogue(mod64(s[i + 1], M), alpha, beta, yo.y, M);
                yo.z = epilogue(mod64(s[i + 2], M), alpha, beta, yo.z, M);
                yo.w = epilogue(mod64(s[i + 3], M), alpha, beta, yo.w, M);
                *reinterpret_cast<uint4 *>(y + r0 + i) = yo;
            }
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                const uint32_t r = r0 + i;
                if (r < rows) {
                    const uint32_t yold = beta ? y[r] : 0u;
                    y[r] = epilogue(mod64(s[i], M), alpha, beta, yold, M);
                }
            }
        }
    }
}

// one static per kernel instantiation: the dynamic-smem opt-in is per function
template <class IT, bool SPLIT, bool LAZY>
void run_panel(const DevPanel &op, const DevMod &M, const uint32_t *x, IT *partial, size_t smem,
               cudaStream_t st) {
    static size_t configured[64] = {};     // per device
    int dev = 0;
    cudaGetDevice(&dev);
    size_t &c = configured[dev & 63];
    if (c < smem) {
        cudaFuncSetAttribute(k_panel<IT, SPLIT, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c = smem;
    }
    k_panel<IT, SPLIT, LAZY><<<op.g.nctas, PANEL_THREADS, smem, st>>>(op, M, x, partial);
}

template <class IT, bool SPLIT>
int launch_t(const DevPanel &op, const DevMod &M, uint32_t alpha, const uint32_t *x, uint32_t beta,
             uint32_t *y, cudaStream_t st) {
    const PanelGeom &g = op.g;
    IT *partial = reinterpret_cast<IT *>(op.partial);
    if (g.P > 0 && g.B > 0) {
        const size_t smem = hc_offset<IT, SPLIT>(g) + panel_hc<SPLIT>() * sizeof(PanelTile);
        if (SPLIT || !g.lazy) run_panel<IT, SPLIT, false>(op, M, x, partial, smem, st);
        else run_panel<IT, SPLIT, !SPLIT>(op, M, x, partial, smem, st);
        count_launch();
        int e = (int)cudaGetLastError();
        if (e) return e;
    }
    if (op.rows) {
        constexpr int VEC = 16 / sizeof(IT);
        const uint32_t work = (op.rows + VEC - 1) / VEC;
        const uint32_t blocks = std::max<uint32_t>(1, std::min<uint32_t>((work + 255) / 256, g.nctas * 8));
        const bool y_aligned = ((uintptr_t)y & 15) == 0;
        k_panel_reduce<IT><<<blocks, 256, 0, st>>>(partial, g.P, op.rows, g.rows_pad, M, alpha, beta, y,
                                                   y_aligned);
        count_launch();
    }
    return (int)cudaGetLastError();
}

}  // namespace

int launch_panel_apply(const DevPanel &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                       uint32_t beta, uint32_t *y, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (op.g.xbytes) {
        case 1: return launch_t<uint8_t, false>(op, M, alpha, x, beta, y, st);
        case 2: return launch_t<uint16_t, false>(op, M, alpha, x, beta, y, st);
        default: return launch_t<uint32_t, true>(op, M, alpha, x, beta, y, st);
    }
}

}  // namespace ffspmv

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
constexpr int PBP = 4;  // +-1 entries per thread per round (all loads issued first)
constexpr int PBV = 8;  // valued entries per thread per round
constexpr uint32_t PANEL_NONE = 0xFFFFFFFFu;  // no entry (a packed word never has row >= R)

// Shared-memory accesses through 32-bit shared addresses (no generic-address
// conversion in the hot loop).
template <class IT>
__device__ __forceinline__ uint32_t lds_x(uint32_t base, uint32_t i) {
    uint32_t v;
    if constexpr (sizeof(IT) == 1) {
        unsigned short h;
        asm volatile("ld.shared.u8 %0, [%1];" : "=h"(h) : "r"(base + i));
        v = h;
    } else if constexpr (sizeof(IT) == 2) {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(base + 2 * i));
        v = h;
    } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4 * i));
    }
    return v;
}

// acc[row] += v (two u32 halves at acc and acc + R when SPLIT: each half of
// a residue < 2^32 is < 2^16, and a tile row has at most W < 2^16 addends)
template <bool SPLIT>
__device__ __forceinline__ void acc_add_s(uint32_t acc_s, uint32_t hi_off, uint32_t row, uint32_t v) {
    if constexpr (SPLIT) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v & 0xFFFFu));
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + hi_off + 4 * row), "r"(v >> 16));
    } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v));
    }
}

// partial stores stay in L2 for the reduction pass
__device__ __forceinline__ void st_keep4(uint32_t *p, uint4 v) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(POLICY_EVICT_LAST));
}
__device__ __forceinline__ void st_keep(uint32_t *p, uint32_t v) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v),
                 "l"(POLICY_EVICT_LAST));
}

// x panel -> shared memory, converted to the narrow staged type.  Eight
// 16-byte loads per thread are issued before any store.
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
                    sx[4 * i] = (IT)v[u].x;
                    sx[4 * i + 1] = (IT)v[u].y;
                    sx[4 * i + 2] = (IT)v[u].z;
                    sx[4 * i + 3] = (IT)v[u].w;
                }
            }
        }
        done = nvec * 4;
    }
    for (uint32_t i = done + threadIdx.x; i < wn; i += PANEL_THREADS) sx[i] = (IT)__ldg(src + i);
}

// (a * x) mod m of a valued entry, in 32-bit arithmetic when m <= 2^16
template <bool SPLIT>
__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t xv, const DevMod &M) {
    if constexpr (SPLIT) return mod64((uint64_t)a * xv, M);
    else return mod32(a * xv, M);
}

template <class IT, bool SPLIT, class VT>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
k_panel(DevPanel op, DevMod M, const uint32_t *__restrict__ xin, IT *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    const PanelGeom g = op.g;
    IT *sx = reinterpret_cast<IT *>(smem);
    uint32_t *acc = reinterpret_cast<uint32_t *>(smem + (size_t)g.W * sizeof(IT));
    const uint32_t sx_s = (uint32_t)__cvta_generic_to_shared(sx);
    const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc);
    const uint32_t hi_off = 4 * g.R;                 // SPLIT: high halves at acc + R
    const uint32_t colmask = (1u << g.cb) - 1, signbit = 1u << g.cb, rshift = g.cb + 1;
    const uint32_t t0 = op.cta_t0[blockIdx.x], t1 = op.cta_t0[blockIdx.x + 1];
    const VT *vval = reinterpret_cast<const VT *>(op.vval);
    for (uint32_t i = threadIdx.x; i < g.R * (SPLIT ? 2 : 1); i += PANEL_THREADS) acc[i] = 0;
    uint32_t cur_p = 0xFFFFFFFFu;
    // Round 0 of both streams of the next tile is loaded before the current
    // tile's write-out, so that write-out hides the next tile's first memory
    // round trip.
    uint32_t w[PBP], x[PBV], a[PBV];
    uint32_t te0 = 0, tn = 0, tv0 = 0, tnv = 0;
    auto prefetch = [&](uint32_t tt) {
        te0 = op.tp[tt];
        tn = op.tp[tt + 1] - te0;
        tv0 = op.tv[tt];
        tnv = op.tv[tt + 1] - tv0;
        const uint32_t np = tn - tnv;
        const uint32_t *pw = op.pent + te0, *vw = op.pent + te0 + np;
        const VT *va = vval + tv0;
#pragma unroll
        for (int u = 0; u < PBP; ++u) {
            const uint32_t e = u * PANEL_THREADS + threadIdx.x;
            w[u] = e < np ? ld_stream(pw + e) : PANEL_NONE;
        }
#pragma unroll
        for (int u = 0; u < PBV; ++u) {
            const uint32_t e = u * PANEL_THREADS + threadIdx.x;
            x[u] = e < tnv ? ld_stream(vw + e) : PANEL_NONE;
            a[u] = e < tnv ? ld_stream(va + e) : 0u;
        }
    };
    if (t0 < t1) prefetch(t0);
    for (uint32_t t = t0; t < t1; ++t) {
        const uint32_t p = t / g.B, b = t - p * g.B;
        if (p != cur_p) {
            const uint64_t c0 = (uint64_t)p * g.W;
            const uint32_t wn = (uint32_t)min((uint64_t)g.W, (uint64_t)op.cols - c0);
            stage_x<IT>(sx, xin, c0, wn);
            cur_p = p;
        }
        __syncthreads();
        // The +-1 part [0, np) and the valued part [np, n) of the tile run as
        // two specialised loops; every round issues all its loads before the
        // first shared op.
        {
            const uint32_t np = tn - tnv, nv = tnv;
            const uint32_t *pw = op.pent + te0, *vw = op.pent + te0 + np;
            const VT *va = vval + tv0;
            const uint32_t m = M.m;
            for (uint32_t base = threadIdx.x; base < np; base += PBP * PANEL_THREADS) {
                if (base != threadIdx.x) {
#pragma unroll
                    for (int u = 0; u < PBP; ++u) {
                        const uint32_t e = base + u * PANEL_THREADS;
                        w[u] = e < np ? ld_stream(pw + e) : PANEL_NONE;
                    }
                }
#pragma unroll
                for (int u = 0; u < PBP; ++u) {
                    if (w[u] != PANEL_NONE) {
                        const uint32_t xv = lds_x<IT>(sx_s, w[u] & colmask);
                        const uint32_t ad = (w[u] & signbit) ? (xv ? m - xv : 0u) : xv;
                        acc_add_s<SPLIT>(acc_s, hi_off, w[u] >> rshift, ad);
                    }
                }
            }
            for (uint32_t base = threadIdx.x; base < nv;) {
#pragma unroll
                for (int u = 0; u < PBV; ++u) {
                    if (x[u] != PANEL_NONE) {
                        const uint32_t xv = lds_x<IT>(sx_s, x[u] & colmask);
                        acc_add_s<SPLIT>(acc_s, hi_off, x[u] >> rshift, mulmod<SPLIT>(a[u], xv, M));
                    }
                }
                base += PBV * PANEL_THREADS;
                if (base >= nv) break;
#pragma unroll
                for (int u = 0; u < PBV; ++u) {
                    const uint32_t e = base + u * PANEL_THREADS;
                    x[u] = e < nv ? ld_stream(vw + e) : PANEL_NONE;
                    a[u] = e < nv ? ld_stream(va + e) : 0u;
                }
            }
        }
        __syncthreads();
        if (t + 1 < t1) prefetch(t + 1);
        // one residue per band row -> partial[p][row] (same narrow type as the
        // staged x); re-zero the accumulators.  m <= 2^16: the row sum is
        // < W * m < 2^32 and reduces with the 32-bit Barrett; SPLIT: the
        // residue of lo + hi * 2^16.
        const uint64_t r0 = (uint64_t)b * g.R;
        const uint32_t rn = (uint32_t)min((uint64_t)g.R, (uint64_t)op.rows - r0);
        IT *out = partial + (uint64_t)p * op.rows + r0;
        uint32_t r = 0;
        if (!SPLIT && ((uintptr_t)out % (4 * sizeof(IT))) == 0) {
            const uint32_t nq = rn / 4;
            for (uint32_t q = threadIdx.x; q < nq; q += PANEL_THREADS) {
                const uint4 s4 = reinterpret_cast<const uint4 *>(acc)[q];
                reinterpret_cast<uint4 *>(acc)[q] = make_uint4(0, 0, 0, 0);
                const uint32_t v0 = mod32(s4.x, M), v1 = mod32(s4.y, M), v2 = mod32(s4.z, M),
                               v3 = mod32(s4.w, M);
                if constexpr (sizeof(IT) == 2) {
                    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(out + 4 * q),
                                 "r"(v0 | (v1 << 16)), "r"(v2 | (v3 << 16)), "l"(POLICY_EVICT_LAST));
                } else {
                    st_keep(reinterpret_cast<uint32_t *>(out + 4 * q), v0 | (v1 << 8) | (v2 << 16) | (v3 << 24));
                }
            }
            r = nq * 4;
        }
        for (r += threadIdx.x; r < rn; r += PANEL_THREADS) {
            uint32_t res;
            if constexpr (SPLIT) {
                res = mod64((uint64_t)acc[r] + ((uint64_t)acc[g.R + r] << 16), M);
                acc[g.R + r] = 0;
            } else {
                res = mod32(acc[r], M);
            }
            acc[r] = 0;
            out[r] = (IT)res;
        }
        // the next tile's __syncthreads orders these writes before reuse
    }
}

// y[r] = alpha * sum_p partial[p][r] + beta * y[r]; VEC = 16 / sizeof(IT)
// consecutive rows per thread so each panel's partials load as one 16-byte
// vector (VEC = 1 when rows is not a multiple of it).
template <class IT, int VEC>
__global__ void k_panel_reduce(const IT *__restrict__ partial, uint32_t P, uint32_t rows,
                               DevMod M, uint32_t alpha, uint32_t beta, uint32_t *__restrict__ y) {
    const uint32_t nvec = rows / VEC;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x) {
        uint64_t s[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) s[i] = 0;
        for (uint32_t p = 0; p < P; ++p) {   // P residues < 2^32: exact in u64
            const IT *src = partial + (uint64_t)p * rows + (uint64_t)v * VEC;
            if constexpr (VEC * sizeof(IT) == 16) {
                const uint4 e4 = *reinterpret_cast<const uint4 *>(src);
                const IT *e = reinterpret_cast<const IT *>(&e4);
#pragma unroll
                for (int i = 0; i < VEC; ++i) s[i] += e[i];
            } else {
#pragma unroll
                for (int i = 0; i < VEC; ++i) s[i] += src[i];
            }
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            const uint32_t r = v * VEC + i;
            const uint32_t yold = beta ? y[r] : 0u;
            y[r] = epilogue(mod64(s[i], M), alpha, beta, yold, M);
        }
    }
}

template <class IT, bool SPLIT>
int launch_t(const DevPanel &op, const DevMod &M, uint32_t alpha, const uint32_t *x, uint32_t beta,
             uint32_t *y, cudaStream_t st) {
    const PanelGeom &g = op.g;
    IT *partial = reinterpret_cast<IT *>(op.partial);
    if (g.P > 0 && g.B > 0) {
        size_t smem = (size_t)g.W * sizeof(IT) + (size_t)g.R * 4 * (SPLIT ? 2 : 1);
        auto run = [&](auto kern) {
            static size_t configured = 0;   // per instantiation
            if (configured < smem) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                configured = smem;
            }
            kern<<<g.nctas, PANEL_THREADS, smem, st>>>(op, M, x, partial);
        };
        switch (M.vbytes) {
            case 1: run(k_panel<IT, SPLIT, uint8_t>); break;
            case 2: run(k_panel<IT, SPLIT, uint16_t>); break;
            default: run(k_panel<IT, SPLIT, uint32_t>); break;
        }
        count_launch();
        int e = (int)cudaGetLastError();
        if (e) return e;
    }
    if (op.rows) {
        // each panel's row block is 16-byte aligned only if rows % VEC == 0
        constexpr int VEC = 16 / sizeof(IT);
        const bool vec_ok = (op.rows % VEC) == 0;
        const uint32_t work = vec_ok ? op.rows / VEC : op.rows;
        const uint32_t blocks = std::max<uint32_t>(1, std::min<uint32_t>((work + 255) / 256, g.nctas * 8));
        if (vec_ok)
            k_panel_reduce<IT, VEC><<<blocks, 256, 0, st>>>(partial, g.P, op.rows, M, alpha, beta, y);
        else
            k_panel_reduce<IT, 1><<<blocks, 256, 0, st>>>(partial, g.P, op.rows, M, alpha, beta, y);
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

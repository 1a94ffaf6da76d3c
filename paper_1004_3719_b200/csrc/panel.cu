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
//                   range (panel-major): stage x panel, accumulate band rows,
//                   write one residue per band row into partial[p][row]
//   k_panel_reduce  y[r] = alpha * sum_p partial[p][r] + beta * y[r]  (mod m)
#include "device.cuh"

namespace ffspmv {

void count_launch();

namespace {

constexpr int PANEL_THREADS = 1024;
constexpr int PBP = 4;  // +-1 entries per thread per round (all loads issued first)
constexpr int PBV = 8;  // valued entries per thread per round

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

template <bool SPLIT>
__device__ __forceinline__ void acc_add_s(uint32_t acc_s, uint32_t row, uint32_t v);
constexpr uint32_t PANEL_NONE = 0xFFFFFFFFu;  // no entry (bit 31 of a packed word is 0)

template <bool SPLIT>
__device__ __forceinline__ void acc_add(uint32_t *acc, uint32_t row, uint32_t v);

template <class IT, int WV>
__device__ __forceinline__ void st_keep_vec(IT *p, const uint32_t (&v)[WV]);
constexpr uint32_t ACC_STRIDE = 16384;  // accumulator slots incl. the 64 per-lane dummies

// partial stores stay in L2 for the reduction pass
__device__ __forceinline__ void st_keep(uint8_t *p, uint32_t v) {
    asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(p), "h"((unsigned short)v),
                 "l"(POLICY_EVICT_LAST));
}
__device__ __forceinline__ void st_keep(uint16_t *p, uint32_t v) {
    asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(p), "h"((unsigned short)v),
                 "l"(POLICY_EVICT_LAST));
}
__device__ __forceinline__ void st_keep(uint32_t *p, uint32_t v) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v),
                 "l"(POLICY_EVICT_LAST));
}

template <bool SPLIT>
__device__ __forceinline__ void acc_add(uint32_t *acc, uint32_t row, uint32_t v) {
    if constexpr (SPLIT) {
        atomicAdd(acc + row, v & 0xFFFFu);
        atomicAdd(acc + ACC_STRIDE + row, v >> 16);
    } else {
        atomicAdd(acc + row, v);
    }
}

template <bool SPLIT>
__device__ __forceinline__ void acc_add_s(uint32_t acc_s, uint32_t row, uint32_t v) {
    if constexpr (SPLIT) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v & 0xFFFFu));
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * (ACC_STRIDE + row)), "r"(v >> 16));
    } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(acc_s + 4 * row), "r"(v));
    }
}

// WV consecutive narrow partials in one 4- or 8-byte store (L2 evict_last)
template <class IT, int WV>
__device__ __forceinline__ void st_keep_vec(IT *p, const uint32_t (&v)[WV]) {
    if constexpr (sizeof(IT) == 2 && WV == 4) {
        const uint32_t lo = v[0] | (v[1] << 16), hi = v[2] | (v[3] << 16);
        asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(lo),
                     "r"(hi), "l"(POLICY_EVICT_LAST));
    } else if constexpr (sizeof(IT) == 1 && WV == 4) {
        const uint32_t w = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
        asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(w),
                     "l"(POLICY_EVICT_LAST));
    } else {
#pragma unroll
        for (int i = 0; i < WV; ++i) p[i] = (IT)v[i];
    }
}

// x panel -> shared memory, converted to the narrow staged type.
// Eight 16-byte loads per thread are issued before any store, so a 64k
// column panel costs two memory round trips instead of 64.
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

// Addend of one packed entry, < m.  +-1 entries: x or m - x (0 stays 0);
// valued entries: (a * x) mod m, in 32-bit arithmetic when m <= 2^16.
template <bool SPLIT>
__device__ __forceinline__ uint32_t addend(bool valued, uint32_t w, uint32_t a, uint32_t xv,
                                           const DevMod &M) {
    if (valued) {
        if constexpr (SPLIT) return mod64((uint64_t)a * xv, M);
        else return mod32(a * xv, M);
    }
    return (w & PANEL_SIGN) ? (xv ? M.m - xv : 0u) : xv;
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
    const uint32_t t0 = op.cta_t0[blockIdx.x], t1 = op.cta_t0[blockIdx.x + 1];
    const VT *vval = reinterpret_cast<const VT *>(op.vval);
    for (uint32_t i = threadIdx.x; i < ACC_STRIDE * (SPLIT ? 2 : 1); i += PANEL_THREADS) acc[i] = 0;
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
            const uint32_t e0 = te0, n = tn;
            const uint32_t v0 = tv0, nv = tnv, np = n - nv;
            const uint32_t *pw = op.pent + e0, *vw = op.pent + e0 + np;
            const VT *va = vval + v0;
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
                        const uint32_t xv = lds_x<IT>(sx_s, w[u] & 0xFFFFu);
                        const uint32_t ad = (w[u] & PANEL_SIGN) ? (xv ? m - xv : 0u) : xv;
                        acc_add_s<SPLIT>(acc_s, w[u] >> PANEL_ROW_SHIFT, ad);
                    }
                }
            }
            for (uint32_t base = threadIdx.x;; ) {
#pragma unroll
                for (int u = 0; u < PBV; ++u) {
                    if (x[u] != PANEL_NONE) {
                        const uint32_t xv = lds_x<IT>(sx_s, x[u] & 0xFFFFu);
                        acc_add_s<SPLIT>(acc_s, x[u] >> PANEL_ROW_SHIFT,
                                         addend<SPLIT>(true, 0, a[u], xv, M));
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
        // one residue per band row -> partial[p][row]; re-zero the accumulators
        const uint64_t r0 = (uint64_t)b * g.R;
        const uint32_t rn = (uint32_t)min((uint64_t)g.R, (uint64_t)op.rows - r0);
        IT *out = partial + (uint64_t)p * op.rows + r0;
        constexpr int WV = 16 / sizeof(IT) < 4 ? 16 / sizeof(IT) : 4;   // rows per vector store
        const bool vec = !SPLIT && ((uintptr_t)out % (WV * sizeof(IT))) == 0;
        uint32_t r = 0;
        if (vec) {
            const uint32_t nq = rn / WV;
            for (uint32_t q = threadIdx.x; q < nq; q += PANEL_THREADS) {
                uint32_t v[WV];
                if constexpr (WV == 4) {
                    const uint4 s4 = reinterpret_cast<const uint4 *>(acc)[q];
                    reinterpret_cast<uint4 *>(acc)[q] = make_uint4(0, 0, 0, 0);
                    v[0] = s4.x; v[1] = s4.y; v[2] = s4.z; v[3] = s4.w;
                } else {
#pragma unroll
                    for (int i = 0; i < WV; ++i) { v[i] = acc[q * WV + i]; acc[q * WV + i] = 0; }
                }
#pragma unroll
                for (int i = 0; i < WV; ++i) v[i] = mod32(v[i], M);
                st_keep_vec<IT, WV>(out + q * WV, v);
            }
            r = nq * WV;
        }
        for (r += threadIdx.x; r < rn; r += PANEL_THREADS) {
            uint32_t res;
            if constexpr (SPLIT) {
                // lo, hi < 2^30 (<= W = 2^14 addends each): exact in u64
                res = mod64((uint64_t)acc[r] + ((uint64_t)acc[ACC_STRIDE + r] << 16), M);
                acc[ACC_STRIDE + r] = 0;
            } else {
                res = mod32(acc[r], M);   // < W * m <= 2^32 for m <= 2^16
            }
            acc[r] = 0;
            st_keep(out + r, res);
        }
        // the next tile's __syncthreads orders these writes before reuse
    }
}

// y[r] = alpha * sum_p partial[p][r] + beta * y[r]; VEC consecutive rows per
// thread so each panel's partials load as one vector.
template <class IT, int VEC>
__global__ void k_panel_reduce(const IT *__restrict__ partial, uint32_t P, uint32_t rows,
                               DevMod M, uint32_t alpha, uint32_t beta, uint32_t *__restrict__ y) {
    const uint32_t nvec = rows / VEC;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x) {
        uint64_t s[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) s[i] = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const IT *src = partial + (uint64_t)p * rows + (uint64_t)v * VEC;
            IT e[VEC];
            if constexpr (VEC * sizeof(IT) == 16) {
                *reinterpret_cast<uint4 *>(e) = *reinterpret_cast<const uint4 *>(src);
            } else if constexpr (VEC * sizeof(IT) == 8) {
                *reinterpret_cast<uint2 *>(e) = *reinterpret_cast<const uint2 *>(src);
            } else {
#pragma unroll
                for (int i = 0; i < VEC; ++i) e[i] = src[i];
            }
#pragma unroll
            for (int i = 0; i < VEC; ++i) s[i] += e[i];
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            const uint32_t r = v * VEC + i;
            const uint32_t yold = beta ? y[r] : 0u;
            y[r] = epilogue(mod64(s[i], M), alpha, beta, yold, M);
        }
    }
    // ragged tail (rows % VEC), handled by the first threads
    const uint32_t r = nvec * VEC + blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows && blockIdx.x * blockDim.x + threadIdx.x < VEC) {
        uint64_t s = 0;
        for (uint32_t p = 0; p < P; ++p) s += partial[(uint64_t)p * rows + r];
        const uint32_t yold = beta ? y[r] : 0u;
        y[r] = epilogue(mod64(s, M), alpha, beta, yold, M);
    }
}

template <class IT, bool SPLIT>
int launch_t(const DevPanel &op, const DevMod &M, uint32_t alpha, const uint32_t *x, uint32_t beta,
             uint32_t *y, cudaStream_t st) {
    const PanelGeom &g = op.g;
    IT *partial = reinterpret_cast<IT *>(op.partial);
    if (g.P > 0 && g.B > 0) {
        size_t smem = (size_t)g.W * sizeof(IT) + (size_t)ACC_STRIDE * 4 * (SPLIT ? 2 : 1);
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
        // the partial rows are 16-byte aligned per panel only if rows % VEC == 0
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

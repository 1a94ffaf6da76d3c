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
constexpr int PB = 8;                       // entries per stream per thread per round
constexpr uint32_t PANEL_NONE = 0xFFFFFFFFu;  // no entry (bit 31 is never set in a packed word)

template <class IT>
__device__ __forceinline__ void st_partial(IT *p, uint32_t v) {
    *p = (IT)v;
}

// x panel -> shared memory, converted to the narrow staged type.
template <class IT>
__device__ __forceinline__ void stage_x(IT *sx, const uint32_t *__restrict__ x, uint64_t c0,
                                        uint32_t wn) {
    for (uint32_t i = threadIdx.x; i < wn; i += PANEL_THREADS) sx[i] = (IT)__ldg(x + c0 + i);
}

template <bool SPLIT>
__device__ __forceinline__ void acc_add(uint32_t *acc, uint32_t R, uint32_t row, uint32_t v) {
    if constexpr (SPLIT) {
        atomicAdd(acc + row, v & 0xFFFFu);
        atomicAdd(acc + R + row, v >> 16);
    } else {
        atomicAdd(acc + row, v);
    }
}

template <class IT, bool SPLIT, class VT>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
k_panel(DevPanel op, DevMod M, const uint32_t *__restrict__ x, IT *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    const PanelGeom g = op.g;
    IT *sx = reinterpret_cast<IT *>(smem);
    uint32_t *acc = reinterpret_cast<uint32_t *>(smem + (size_t)g.W * sizeof(IT));
    const uint32_t m = M.m;
    const uint32_t t0 = op.cta_t0[blockIdx.x], t1 = op.cta_t0[blockIdx.x + 1];
    const VT *vval = reinterpret_cast<const VT *>(op.vval);
    for (uint32_t i = threadIdx.x; i < g.R * (SPLIT ? 2 : 1); i += PANEL_THREADS) acc[i] = 0;
    uint32_t cur_p = 0xFFFFFFFFu;
    for (uint32_t t = t0; t < t1; ++t) {
        const uint32_t p = t / g.B, b = t - p * g.B;
        if (p != cur_p) {
            const uint64_t c0 = (uint64_t)p * g.W;
            const uint32_t wn = (uint32_t)min((uint64_t)g.W, (uint64_t)op.cols - c0);
            stage_x<IT>(sx, x, c0, wn);
            cur_p = p;
        }
        __syncthreads();
        // One round issues every load of up to PB +-1 and PB valued entries per
        // thread before the first shared-memory op, so a tile costs about one
        // memory round trip (+-1 addend: x or m - x; valued: (a*x) mod m).
        {
            const uint32_t p0 = op.tp[t], np = op.tp[t + 1] - p0;
            const uint32_t v0 = op.tv[t], nv = op.tv[t + 1] - v0;
            const uint32_t nmax = max(np, nv);
            for (uint32_t base = threadIdx.x; base < nmax; base += PB * PANEL_THREADS) {
                uint32_t w[PB], vw[PB], va[PB];
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    const uint32_t e = base + u * PANEL_THREADS;
                    w[u] = e < np ? ld_stream(op.pent + p0 + e) : PANEL_NONE;
                    vw[u] = e < nv ? ld_stream(op.vent + v0 + e) : PANEL_NONE;
                    va[u] = e < nv ? ld_stream(vval + v0 + e) : 0u;
                }
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    if (w[u] != PANEL_NONE) {
                        const uint32_t xv = sx[w[u] & 0xFFFFu];
                        const uint32_t a = (w[u] & PANEL_SIGN) ? (xv ? m - xv : 0u) : xv;
                        acc_add<SPLIT>(acc, g.R, w[u] >> PANEL_ROW_SHIFT, a);
                    }
                    if (vw[u] != PANEL_NONE) {
                        const uint32_t xv = sx[vw[u] & 0xFFFFu];
                        acc_add<SPLIT>(acc, g.R, vw[u] >> PANEL_ROW_SHIFT,
                                       mod64((uint64_t)va[u] * xv, M));
                    }
                }
            }
        }
        __syncthreads();
        // one residue per band row -> partial[p][row]; re-zero the accumulators
        const uint64_t r0 = (uint64_t)b * g.R;
        const uint32_t rn = (uint32_t)min((uint64_t)g.R, (uint64_t)op.rows - r0);
        IT *out = partial + (uint64_t)p * op.rows + r0;
        for (uint32_t r = threadIdx.x; r < rn; r += PANEL_THREADS) {
            uint64_t s = acc[r];
            acc[r] = 0;
            if constexpr (SPLIT) {
                s += (uint64_t)acc[g.R + r] << 16;
                acc[g.R + r] = 0;
            }
            st_partial(out + r, mod64(s, M));
        }
        // the next tile's __syncthreads orders these writes before reuse
    }
}

template <class IT>
__global__ void k_panel_reduce(const IT *__restrict__ partial, uint32_t P, uint32_t rows,
                               DevMod M, uint32_t alpha, uint32_t beta, uint32_t *__restrict__ y) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        uint64_t s = 0;  // P residues < m: < 2^64 for any P < 2^32
        uint32_t p = 0;
        for (; p + 4 <= P; p += 4) {
            uint32_t v0 = partial[(uint64_t)p * rows + r], v1 = partial[(uint64_t)(p + 1) * rows + r];
            uint32_t v2 = partial[(uint64_t)(p + 2) * rows + r], v3 = partial[(uint64_t)(p + 3) * rows + r];
            s += (uint64_t)v0 + v1 + v2 + v3;
        }
        for (; p < P; ++p) s += partial[(uint64_t)p * rows + r];
        uint32_t yold = beta ? y[r] : 0u;
        y[r] = epilogue(mod64(s, M), alpha, beta, yold, M);
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
        uint32_t blocks = std::min<uint32_t>((op.rows + 255) / 256, g.nctas * 8);
        k_panel_reduce<IT><<<blocks, 256, 0, st>>>(partial, g.P, op.rows, M, alpha, beta, y);
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
        default:
            if (op.g.split) return launch_t<uint32_t, true>(op, M, alpha, x, beta, y, st);
            return launch_t<uint32_t, false>(op, M, alpha, x, beta, y, st);
    }
}

}  // namespace ffspmv

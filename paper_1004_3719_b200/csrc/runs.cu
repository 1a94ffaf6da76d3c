// RUNS apply for k = 1 (north star "x tiles staged in
// shared memory via TMA"): y <- alpha A x + beta y on the tiled operator of
// runs_build.cpp (internal.hpp "runs").
//
//   k_runs_pack  x (u32) -> packed panels xp[p] (xbits per residue, zero
//                beyond cols); triggers the dependent launch at once
//   k_runs       persistent, one 1024-thread CTA per SM; its contiguous
//                range of units (panel p x R-row band, panel-major) is cut
//                into segments of one panel, each staged with cp.async.bulk
//                (mbarrier transaction count) into shared memory; inside a
//                segment every warp takes whole units (a shared counter) and
//                owns private band accumulators, so no CTA barrier separates
//                units; each lane walks RUN_E consecutive entries of a chunk
//                (sorted by row), sums each run of one row in a register and
//                adds it to the warp's accumulators (red.shared) when the row
//                changes; the unit writes one residue per band row into
//                partial[p]
//   k_runs_reduce  y = alpha sum_p partial[p] + beta y (Fig. 2, P:210-222,
//                "foreach submatrix Ai in A do spmv(y, Ai, x); reduce(y, m)"),
//                the programmatic dependent of k_runs
#include <type_traits>

#include "device.cuh"

namespace ffspmv {

void count_launch();

namespace {

constexpr int RT = RUN_WARPS * 32;   // threads per CTA

// ------------------------------------------------------------ pack x ------
// Thread i packs 4 consecutive residues of one panel (one 16-byte load of x
// when aligned) into 4 * XB bits: one byte (XB = 2), two (4), four (8), eight
// (16), sixteen (32).  Panels are multiples of 64 columns, so a group never
// straddles two; elements past cols are zero.
template <int XB>
__global__ void k_runs_pack(const uint32_t *__restrict__ x, uint32_t cols, uint32_t W, uint32_t P,
                            uint32_t panel_bytes, unsigned char *__restrict__ xp) {
    asm volatile("griddepcontrol.launch_dependents;");
    // grid: (groups of 256 x 4 elements, panels); 32-bit indices (W < 2^31)
    const uint32_t per_panel = W / 4;
    const bool aligned = ((uintptr_t)x & 15) == 0;
    for (uint32_t p = blockIdx.y; p < P; p += gridDim.y)
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < per_panel; q += gridDim.x * blockDim.x) {
        const uint64_t c0 = (uint64_t)p * W + 4 * q;     // first column
        uint4 v;
        if (aligned && c0 + 4 <= cols) {
            v = __ldg(reinterpret_cast<const uint4 *>(x + c0));
        } else {
            v.x = c0 < cols ? __ldg(x + c0) : 0u;
            v.y = c0 + 1 < cols ? __ldg(x + c0 + 1) : 0u;
            v.z = c0 + 2 < cols ? __ldg(x + c0 + 2) : 0u;
            v.w = c0 + 3 < cols ? __ldg(x + c0 + 3) : 0u;
        }
        unsigned char *dst = xp + (uint64_t)p * panel_bytes + (uint64_t)q * (XB / 2);   // 4 * XB bits
        if constexpr (XB == 2) {
            *dst = (unsigned char)(v.x | v.y << 2 | v.z << 4 | v.w << 6);
        } else if constexpr (XB == 4) {
            *reinterpret_cast<uint16_t *>(dst) = (uint16_t)(v.x | v.y << 4 | v.z << 8 | v.w << 12);
        } else if constexpr (XB == 8) {
            *reinterpret_cast<uint32_t *>(dst) = v.x | v.y << 8 | v.z << 16 | v.w << 24;
        } else if constexpr (XB == 16) {
            *reinterpret_cast<uint2 *>(dst) = make_uint2(v.x | v.y << 16, v.z | v.w << 16);
        } else {
            *reinterpret_cast<uint4 *>(dst) = v;
        }
    }
}

// y[r] = alpha * sum_p partial[p][r] + beta * y[r] (mod m), RPT = 16 /
// sizeof(PT) rows per thread (one 16-byte load per panel; the partial row
// stride is a multiple of 16).  Launched as the programmatic dependent of
// k_runs: it waits for the whole grid's partials.
template <class PT>
__global__ void k_runs_reduce(const PT *__restrict__ partial, uint32_t P, uint32_t rows,
                              uint32_t rows_pad, DevMod M, uint32_t alpha, uint32_t beta,
                              uint32_t *__restrict__ y) {
    constexpr int RPT = 16 / sizeof(PT);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t nv = (rows + RPT - 1) / RPT;
    const bool y_aligned = ((uintptr_t)y & 15) == 0;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        uint64_t s[RPT];   // P residues < 2^32 each: exact in u64
#pragma unroll
        for (int i = 0; i < RPT; ++i) s[i] = 0;
        for (uint32_t q = 0; q < P; ++q) {
            const uint4 w = __ldcs(reinterpret_cast<const uint4 *>(partial + (uint64_t)q * rows_pad) + v);
            const PT *e = reinterpret_cast<const PT *>(&w);
#pragma unroll
            for (int i = 0; i < RPT; ++i) s[i] += e[i];
        }
        const uint32_t r0 = RPT * v;
        uint32_t r[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            // m <= 2^16 (u8 / u16 partials): P < 2^16 residues sum below 2^32
            if (sizeof(PT) < 4 && P < 65536u) r[i] = mod32_min((uint32_t)s[i], M);
            else r[i] = mod64(s[i], M);
        }
        if (y_aligned && r0 + RPT <= rows) {
#pragma unroll
            for (int i = 0; i < RPT; i += 4) {
                uint4 yo = beta ? *reinterpret_cast<const uint4 *>(y + r0 + i) : make_uint4(0, 0, 0, 0);
                yo.x = epilogue(r[i], alpha, beta, yo.x, M);
                yo.y = epilogue(r[i + 1], alpha, beta, yo.y, M);
                yo.z = epilogue(r[i + 2], alpha, beta, yo.z, M);
                yo.w = epilogue(r[i + 3], alpha, beta, yo.w, M);
                *reinterpret_cast<uint4 *>(y + r0 + i) = yo;
            }
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                if (r0 + i < rows) y[r0 + i] = epilogue(r[i], alpha, beta, beta ? y[r0 + i] : 0u, M);
        }
    }
}

// ------------------------------------------------------- shared helpers ---
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// stream loads: read once, no L1 allocation, evict-first in L2
__device__ __forceinline__ uint4 ld_stream4(const void *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}
__device__ __forceinline__ uint2 ld_stream2(const void *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint64_t bytes) {
    const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15, e = ((uintptr_t)p + bytes + 15) & ~(uintptr_t)15;
    for (uintptr_t q = a; q < e; q += 1u << 20) {
        const uint32_t n = (uint32_t)min((uintptr_t)(1u << 20), e - q);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(n) : "memory");
    }
}

// One lane's share of a chunk: RUN_E entry words (RUN_E / 4 coalesced
// 16-byte loads per warp, 512 contiguous bytes each) and, for a valued chunk,
// RUN_E values (lane-contiguous, RUN_E * VB bytes).
constexpr int RUN_Q = RUN_E / 4;                      // word quads per lane
struct ChunkRegs {
    uint4 w[RUN_Q], v[(RUN_E * 4 + 15) / 16];
};

template <int VB>
__device__ __forceinline__ void load_chunk(const uint32_t *wb, const unsigned char *vb, ChunkRegs &c) {
#pragma unroll
    for (int q = 0; q < RUN_Q; ++q) c.w[q] = ld_stream4(wb + 128 * q);
    if (vb) {
        if constexpr (RUN_E * VB >= 16) {
#pragma unroll
            for (int q = 0; q < RUN_E * VB / 16; ++q) c.v[q] = ld_stream4(vb + 16 * q);
        } else {
            const uint2 t = ld_stream2(vb);   // RUN_E * VB == 8
            c.v[0] = make_uint4(t.x, t.y, 0, 0);
        }
    }
}

template <int VB>
__device__ __forceinline__ uint32_t value_at(const ChunkRegs &c, int j) {
    const uint4 &q = c.v[(j * VB) / 16];
    const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
    if constexpr (VB == 1) return (ws[(j >> 2) & 3] >> (8 * (j & 3))) & 0xFFu;
    else if constexpr (VB == 2) return (ws[(j >> 1) & 3] >> (16 * (j & 1))) & 0xFFFFu;
    else return ws[j & 3];
}

// a * b + c (mod 2^32) as one IMAD
__device__ __forceinline__ uint32_t mad32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Add a finished run to the warp's band accumulator at shared address `ra`:
// narrow (m <= 2^16), the raw u32 sum (the builder bounded every band row's
// unit sum below 2^32); wide, the run's residue split into 16-bit halves
// added to the low / high arrays `hi` bytes apart, so neither half can
// overflow (fewer than 2^16 runs per band row and unit).
template <bool WIDE>
__device__ __forceinline__ void flush_run(uint32_t ra, uint64_t run, uint32_t hi, const DevMod &M) {
    if constexpr (WIDE) {
        const uint32_t r = mod64(run, M);
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ra), "r"(r & 0xFFFFu) : "memory");
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ra + hi), "r"(r >> 16) : "memory");
    } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ra), "r"((uint32_t)run) : "memory");
    }
}

// One chunk of section KIND (0: +1, 1: -1, 2: valued): the RUN_E entries of
// this lane, consecutive in (row, col) order.  accb: the warp's accumulator
// block (shared address, aligned to its size, so the row offset ORs in);
// rm4 = (2^rs - 1) << 2; xs = 5 + rs.
template <int KIND, int XB, bool WIDE, int VB>
__device__ __forceinline__ void do_chunk(const ChunkRegs &c, uint32_t sx, uint32_t accb,
                                         uint32_t rm4, uint32_t xs, uint32_t hi, const DevMod &M) {
    typedef typename std::conditional<WIDE, uint64_t, uint32_t>::type RunT;
    constexpr uint32_t XMASK = XB == 32 ? 0xFFFFFFFFu : (1u << XB) - 1;
    const uint32_t m = M.m;
    // all RUN_E gathers first (independent shared loads in flight), then the
    // run bookkeeping with its conditional flushes
    uint32_t wv[RUN_E], xv[RUN_E];
#pragma unroll
    for (int j = 0; j < (int)RUN_E; ++j) {
        const uint4 &q = c.w[j >> 2];
        wv[j] = (j & 3) == 0 ? q.x : (j & 3) == 1 ? q.y : (j & 3) == 2 ? q.z : q.w;
        const uint32_t word = lds32(sx + (wv[j] >> xs));
        if constexpr (XB == 32) xv[j] = word;
        else xv[j] = __funnelshift_r(word, 0u, wv[j]) & XMASK;   // bit offset = w mod 32
    }
    uint32_t prev = ((wv[0] >> 3) & rm4) | accb;
    RunT run = 0;
#pragma unroll
    for (int j = 0; j < (int)RUN_E; ++j) {
        const uint32_t ra = ((wv[j] >> 3) & rm4) | accb;     // row * 4 | block
        if (j > 0 && ra != prev) {
            flush_run<WIDE>(prev, run, hi, M);
            run = 0;
        }
        prev = ra;
        if constexpr (KIND == 0) {
            run += xv[j];
        } else if constexpr (KIND == 1) {
            run += (RunT)(m - xv[j]);
        } else {
            const uint32_t a = value_at<VB>(c, j);
            if constexpr (WIDE) {
                run += mod64((uint64_t)a * xv[j], M);
            } else {
                // lazy Barrett remainder of a * x < 2^32: in [0, 2m)
                const uint32_t p = a * xv[j];
                run += mad32(__umulhi(p, M.mu32), 0u - m, p);
            }
        }
    }
    flush_run<WIDE>(prev, run, hi, M);
}

template <int XB, bool WIDE, int VB>
__device__ __forceinline__ void do_chunk_kind(uint32_t kind, const ChunkRegs &c, uint32_t sx,
                                              uint32_t accb, uint32_t rm4, uint32_t xs, uint32_t hi,
                                              const DevMod &M) {
    if (kind == 0) do_chunk<0, XB, WIDE, VB>(c, sx, accb, rm4, xs, hi, M);
    else if (kind == 1) do_chunk<1, XB, WIDE, VB>(c, sx, accb, rm4, xs, hi, M);
    else do_chunk<2, XB, WIDE, VB>(c, sx, accb, rm4, xs, hi, M);
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}"
        ::"r"(mbar), "r"(phase) : "memory");
}

template <class PT>
__device__ __forceinline__ void store_partial4(PT *p, const uint32_t (&r)[4]) {
    if constexpr (sizeof(PT) == 1) {
        *reinterpret_cast<uint32_t *>(p) = r[0] | r[1] << 8 | r[2] << 16 | r[3] << 24;
    } else if constexpr (sizeof(PT) == 2) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(r[0] | r[1] << 16, r[2] | r[3] << 16);
    } else {
        *reinterpret_cast<uint4 *>(p) = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// shared layout of k_runs (bytes from the dynamic base): x panel + 16 zero
// bytes | slack so the accumulator blocks align to their size | RUN_WARPS
// blocks of AW * 2^rs u32 | mbarrier | unit counter
__host__ __device__ __forceinline__ uint32_t runs_block_bytes(const RunsGeom &g) {
    return (g.wide ? 2u : 1u) * (4u << g.rs);
}
__host__ __device__ __forceinline__ uint32_t runs_smem_bytes(const RunsGeom &g) {
    return g.panel_bytes + 16 + runs_block_bytes(g) + RUN_WARPS * runs_block_bytes(g) + 16;
}

template <int XB, bool WIDE, int VB, class PT>
__global__ void __launch_bounds__(RT, 1)
k_runs(DevRuns op, DevMod M, uint32_t alpha, uint32_t beta, uint32_t *__restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    const RunsGeom g = op.g;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t bb = runs_block_bytes(g);
    const uint32_t sx_s = smem_u32(smem);
    // accumulator blocks aligned to their size: the row offset ORs in
    const uint32_t acc0 = (sx_s + g.panel_bytes + 16 + bb - 1) / bb * bb;
    const uint32_t accb = acc0 + warp * bb;
    uint32_t *acc = reinterpret_cast<uint32_t *>(smem + (accb - sx_s));
    const uint32_t mbar_s = acc0 + RUN_WARPS * bb, next_s = mbar_s + 8;
    const uint32_t rm4 = ((1u << g.rs) - 1) << 2, xs = 5 + g.rs, hi = 4u << g.rs;
    const uint32_t u0 = op.cta_t0[blockIdx.x], u1 = op.cta_t0[blockIdx.x + 1];
    // prologue (overlaps the pack kernel): zero the accumulators and the
    // padding word, init the mbarrier, L2-prefetch the first units
    for (uint32_t i = lane; i < bb / 4; i += 32) acc[i] = 0;
    if (tid < 4) reinterpret_cast<uint32_t *>(smem + g.panel_bytes)[tid] = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (u0 + warp < u1 && lane == 0) {
        const RunsTile T = op.tiles[u0 + warp];
        prefetch_l2(op.words + (uint64_t)T.c0 * RUN_CHUNK, 4ull * RUN_CHUNK * (T.npc + T.nmc + T.nvc));
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");   // packed x complete
    asm volatile("griddepcontrol.launch_dependents;");    // let the reduction queue up
    uint32_t phase = 0, staged = 0xFFFFFFFFu;
    const char *xp = reinterpret_cast<const char *>(op.xpack);
    const bool direct = g.P == 1;
    const unsigned char *vbase = reinterpret_cast<const unsigned char *>(op.vval);
    // segments: runs of the CTA's units with one x panel (units are
    // panel-major: panel p owns units [p B, (p + 1) B)); inside a segment
    // each warp takes whole units from a shared counter
    for (uint32_t s0 = u0; s0 < u1;) {
        const uint32_t p = s0 / g.B;
        const uint32_t s1 = min(u1, (p + 1) * g.B);
        __syncthreads();                      // previous segment done with x and the counter
        if (tid == 0) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(next_s), "r"(s0 + RUN_WARPS) : "memory");
            if (p != staged) {
                // generic-proxy reads of the old panel are ordered before the
                // async-proxy writes by the barrier above + this proxy fence
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(mbar_s), "r"(g.panel_bytes) : "memory");
                const char *src = xp + (uint64_t)p * g.panel_bytes;
                for (uint32_t off = 0; off < g.panel_bytes; off += 32768u) {
                    const uint32_t n = min(32768u, g.panel_bytes - off);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        ::"r"(sx_s + off), "l"(src + off), "r"(n), "r"(mbar_s) : "memory");
                }
            }
        }
        if (p != staged) {
            mbar_wait(mbar_s, phase);
            phase ^= 1;
            staged = p;
        }
        __syncthreads();
        auto grab = [&]() -> uint32_t {
            uint32_t u = 0;
            if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(u) : "r"(next_s) : "memory");
            return __shfl_sync(0xFFFFFFFFu, u, 0);
        };
        if (s0 + warp < s1) {
            // this warp's units: s0 + warp first, then from the counter.  The
            // next unit's header is read when the current one starts and its
            // first chunk is loaded before the current unit's write-out; the
            // chunks of a unit ping-pong between two register buffers.
            uint32_t u = s0 + warp;
            RunsTile T = op.tiles[u];
            uint32_t un = grab();
            RunsTile Tn = T;
            if (un < s1) {
                Tn = op.tiles[un];
                if (lane == 0)
                    prefetch_l2(op.words + (uint64_t)Tn.c0 * RUN_CHUNK, 4ull * RUN_CHUNK * (Tn.npc + Tn.nmc + Tn.nvc));
            }
            ChunkRegs A, B;
            auto load = [&](const RunsTile &U, uint32_t ch, ChunkRegs &R) {
                const uint32_t ve = U.npc + U.nmc;
                load_chunk<VB>(op.words + (uint64_t)(U.c0 + ch) * RUN_CHUNK + 4 * lane,
                               ch >= ve ? vbase + ((uint64_t)(U.vc0 + ch - ve) * RUN_CHUNK + RUN_E * lane) * VB
                                        : nullptr, R);
            };
            load(T, 0, A);
            while (true) {
                const uint32_t e1 = T.npc, e2 = T.npc + T.nmc, nch = e2 + T.nvc;
                auto kind = [&](uint32_t ch) { return ch < e1 ? 0u : ch < e2 ? 1u : 2u; };
                for (uint32_t ch = 0; ch < nch; ch += 2) {
                    if (ch + 1 < nch) load(T, ch + 1, B);
                    do_chunk_kind<XB, WIDE, VB>(kind(ch), A, sx_s, accb, rm4, xs, hi, M);
                    if (ch + 1 >= nch) break;
                    if (ch + 2 < nch) load(T, ch + 2, A);
                    do_chunk_kind<XB, WIDE, VB>(kind(ch + 1), B, sx_s, accb, rm4, xs, hi, M);
                }
                const bool more = un < s1;
                if (more) load(Tn, 0, A);     // overlaps the write-out
                // unit u complete: one residue per band row -> partial[p] (or
                // y when P == 1); re-zero the accumulators
                __syncwarp();
                const uint32_t rn = T.rn, nv = (rn + 3) / 4;
                const uint64_t row0 = (uint64_t)(u - p * g.B) * g.R;
                PT *part = reinterpret_cast<PT *>(op.partial) + (uint64_t)p * g.rows_pad + row0;
                for (uint32_t v = lane; v < nv; v += 32) {
                    uint32_t res[4];
                    const uint4 s4 = reinterpret_cast<const uint4 *>(acc)[v];
                    reinterpret_cast<uint4 *>(acc)[v] = make_uint4(0, 0, 0, 0);
                    if constexpr (WIDE) {
                        const uint4 h4 = reinterpret_cast<const uint4 *>(acc + (hi / 4))[v];
                        reinterpret_cast<uint4 *>(acc + (hi / 4))[v] = make_uint4(0, 0, 0, 0);
                        res[0] = mod64((uint64_t)s4.x + ((uint64_t)h4.x << 16), M);
                        res[1] = mod64((uint64_t)s4.y + ((uint64_t)h4.y << 16), M);
                        res[2] = mod64((uint64_t)s4.z + ((uint64_t)h4.z << 16), M);
                        res[3] = mod64((uint64_t)s4.w + ((uint64_t)h4.w << 16), M);
                    } else {
                        res[0] = mod64(s4.x, M);
                        res[1] = mod64(s4.y, M);
                        res[2] = mod64(s4.z, M);
                        res[3] = mod64(s4.w, M);
                    }
                    if (direct) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint64_t r = row0 + 4 * v + i;
                            if (4 * v + i < rn) y[r] = epilogue(res[i], alpha, beta, beta ? y[r] : 0u, M);
                        }
                    } else {
                        store_partial4<PT>(part + 4 * v, res);
                    }
                }
                __syncwarp();
                if (!more) break;
                u = un;
                T = Tn;
                un = grab();
                if (un < s1) {
                    Tn = op.tiles[un];
                    if (lane == 0) {
                        prefetch_l2(op.words + (uint64_t)Tn.c0 * RUN_CHUNK, 4ull * RUN_CHUNK * (Tn.npc + Tn.nmc + Tn.nvc));
                        if (Tn.nvc)
                            prefetch_l2(vbase + (uint64_t)Tn.vc0 * RUN_CHUNK * VB, (uint64_t)RUN_CHUNK * VB * Tn.nvc);
                    }
                }
            }
        }
        s0 = s1;
    }
}

template <int XB, bool WIDE, int VB, class PT>
int launch_t(const DevRuns &op, const DevMod &M, uint32_t alpha, const uint32_t *x, uint32_t beta,
             uint32_t *y, cudaStream_t st) {
    const RunsGeom &g = op.g;
    // pack x into the panels (4 residues per thread)
    const uint32_t bx = std::max<uint32_t>(1, std::min<uint32_t>((g.W / 4 + 255) / 256,
                                                                 (148u * 32 + g.P - 1) / g.P));
    k_runs_pack<XB><<<dim3(bx, std::min<uint32_t>(g.P, 65535u)), 256, 0, st>>>(x, op.cols, g.W, g.P, g.panel_bytes,
                                                   reinterpret_cast<unsigned char *>(op.xpack));
    count_launch();
    int e = (int)cudaGetLastError();
    if (e) return e;
    const size_t smem = runs_smem_bytes(g);
    static size_t configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    size_t &c = configured[dev & 63];
    auto kern = k_runs<XB, WIDE, VB, PT>;
    if (c < smem) {
        if ((e = (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
            return e;
        c = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.nctas);
    cfg.blockDim = dim3(RT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = (int)cudaLaunchKernelEx(&cfg, kern, op, M, alpha, beta, y);
    count_launch();
    if (e || g.P == 1) return e ? e : (int)cudaGetLastError();
    // y <- the panels' partials, as the programmatic dependent of k_runs
    // (measured: a fused tail -- arrival counters per band, the CTA
    // completing a band reduces it -- was slower, 87 vs 73 us on c3: the
    // bands' last arrivals bunch on a few CTAs)
    const uint32_t nv = (op.rows + 16 / sizeof(PT) - 1) / (16 / sizeof(PT));
    cfg.gridDim = dim3(std::max<uint32_t>(1, std::min<uint32_t>((nv + 255) / 256, g.nctas * 8)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    e = (int)cudaLaunchKernelEx(&cfg, k_runs_reduce<PT>, reinterpret_cast<const PT *>(op.partial), g.P,
                                op.rows, g.rows_pad, M, alpha, beta, y);
    count_launch();
    return e ? e : (int)cudaGetLastError();
}

}  // namespace

int launch_runs_apply(const DevRuns &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                      uint32_t beta, uint32_t *y, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (op.rows == 0) return 0;
    // stored values and partials: u8 (m <= 256), u16 (m <= 2^16), u32
    if (op.g.wide) return launch_t<32, true, 4, uint32_t>(op, M, alpha, x, beta, y, st);
    if (M.m > 256u) {
        if (op.g.xbits == 32) return launch_t<32, false, 2, uint16_t>(op, M, alpha, x, beta, y, st);
        return launch_t<16, false, 2, uint16_t>(op, M, alpha, x, beta, y, st);
    }
    switch (op.g.xbits) {
        case 2: return launch_t<2, false, 1, uint8_t>(op, M, alpha, x, beta, y, st);
        case 4: return launch_t<4, false, 1, uint8_t>(op, M, alpha, x, beta, y, st);
        case 8: return launch_t<8, false, 1, uint8_t>(op, M, alpha, x, beta, y, st);
        case 16: return launch_t<16, false, 1, uint8_t>(op, M, alpha, x, beta, y, st);
        default: return launch_t<32, false, 1, uint8_t>(op, M, alpha, x, beta, y, st);
    }
}

}  // namespace ffspmv

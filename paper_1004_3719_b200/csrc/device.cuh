// Device helpers: exact integer accumulators (delayed modular reduction,
// P:129-147), Barrett reduction, cache-hinted loads, and the per-row entry
// walkers shared by the apply, block and sequence kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "internal.hpp"

namespace ffspmv {

// L2 cache policies (createpolicy encodings; same values CUTLASS uses).
constexpr uint64_t POLICY_EVICT_FIRST = 0x12F0000000000000ull;
constexpr uint64_t POLICY_EVICT_LAST = 0x14F0000000000000ull;

// ---------------------------------------------------------------- loads ---
// Matrix stream of the lane-per-row kernels: read once, never reused by this
// SM -> do not allocate in L1, evict first from L2 so x stays resident.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
        : "=r"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint16_t *p) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
        : "=h"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint8_t *p) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
        : "=h"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v & 0xFFu;
}
// Matrix stream of the broadcast (block / sequence) kernels: several rows of
// a slice share one 128 B line, so let L1 keep it; still evict-first in L2.
__device__ __forceinline__ uint32_t ld_bcast(const uint32_t *p) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}
__device__ __forceinline__ uint32_t ld_bcast(const uint16_t *p) {
    unsigned short v;
    asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v;
}
__device__ __forceinline__ uint32_t ld_bcast(const uint8_t *p) {
    unsigned short v;
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(POLICY_EVICT_FIRST));
    return v & 0xFFu;
}
// Gathers of x / X / V: reused across the whole launch -> normal caching.
__device__ __forceinline__ uint32_t ld_gather(const uint32_t *p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_gather(const uint16_t *p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_gather(const uint8_t *p) { return __ldg(p); }

// ------------------------------------------------------------ reduction ---
// Barrett: mu = floor(2^64/m) gives q in {floor(x/m) - 1, floor(x/m)}, so a
// single conditional subtraction finishes (DESIGN.md §"Barrett").
__device__ __forceinline__ uint32_t mod64(uint64_t x, const DevMod &M) {
    uint64_t q = __umul64hi(x, M.mu);
    uint64_t r = x - q * (uint64_t)M.m;
    return (uint32_t)(r >= M.m ? r - M.m : r);
}
// 32-bit Barrett for x < 2^32 and m <= 2^16 (mu32 = floor(2^32/m)): the same
// one-correction argument; r < 2m <= 2^17 cannot overflow.
__device__ __forceinline__ uint32_t mod32(uint32_t x, const DevMod &M) {
    uint32_t r = x - __umulhi(x, M.mu32) * M.m;
    return r >= M.m ? r - M.m : r;
}
// x mod m for x < 2^32, m <= 2^16: Barrett remainder r in [0, 2m), then
// min(r, r - m) as unsigned (r - m wraps to a huge value when r < m).
__device__ __forceinline__ uint32_t mod32_min(uint32_t x, const DevMod &M) {
    const uint32_t r = __umulhi(x, M.mu32) * (0u - M.m) + x;
    return min(r, r - M.m);
}
// s mod m for s < 2^48, m <= 2^16: s = h 2^32 + l with h < 2^16, so
// h (2^32 mod m) < 2^32; both halves reduce with mod32_min.
__device__ __forceinline__ uint32_t mod48(uint64_t s, const DevMod &M) {
    const uint32_t u = mod32_min((uint32_t)s, M) + mod32_min((uint32_t)(s >> 32) * M.r32, M);
    return min(u, u - M.m);
}
// (hi * 2^64 + lo) mod m, hi < 2^32: hi mod m < m, (hi mod m)*(2^64 mod m) +
// (lo mod m) < m^2 + m < 2^64.
__device__ __forceinline__ uint32_t mod96(uint32_t hi, uint64_t lo, const DevMod &M) {
    uint64_t rh = mod64((uint64_t)hi, M);
    return mod64(rh * M.r64 + mod64(lo, M), M);
}

// ---------------------------------------------------------- accumulators ---
// +-1 addends are x or m - x (<= m); valued addends a*x <= (m-1)^2.  The
// builder picks the narrowest carrier whose capacity covers the worst row.
struct Acc32 {
    uint32_t s;
    __device__ __forceinline__ Acc32() : s(0) {}
    __device__ __forceinline__ void add(uint32_t v) { s += v; }
    __device__ __forceinline__ void mad(uint32_t a, uint32_t x) { s += a * x; }
    __device__ __forceinline__ uint32_t reduce(const DevMod &M) const { return mod64(s, M); }
};
struct Acc64 {
    uint64_t s;
    __device__ __forceinline__ Acc64() : s(0) {}
    __device__ __forceinline__ void add(uint32_t v) { s += v; }
    __device__ __forceinline__ void mad(uint32_t a, uint32_t x) { s += (uint64_t)a * x; }
    __device__ __forceinline__ uint32_t reduce(const DevMod &M) const { return mod64(s, M); }
};
// u96 = lo (u64 register pair) + h * 2^64: a MAD lowers to one
// IMAD.WIDE.U32 with carry-out plus an IADD3.X that can merge two carries.
struct Acc96 {
    uint64_t lo;
    uint32_t h;
    __device__ __forceinline__ Acc96() : lo(0), h(0) {}
    __device__ __forceinline__ void add(uint32_t v) {
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+l"(lo), "+r"(h) : "l"((uint64_t)v));
    }
    __device__ __forceinline__ void mad(uint32_t a, uint32_t x) {
        asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, %3;\n\tadd.cc.u64 %0, %0, p;\n\taddc.u32 %1, %1, 0;\n\t}"
            : "+l"(lo), "+r"(h) : "r"(a), "r"(x));
    }
    __device__ __forceinline__ uint32_t reduce(const DevMod &M) const { return mod96(h, lo, M); }
};

// u64 carrier folded every `fold_every` addends (block_slice_as): after a
// fold s = hi (2^32 mod m) + lo < 2^32 (r32 + 1), and the host picks
// fold_every so that many addends of at most (m-1)^2 cannot overflow 2^64
// (fold_capacity).  One IMAD.WIDE per product instead of u96 carry chains;
// used when 2^32 mod m is small (e.g. m = 2^31 - 1: r32 = 2, 3 products).
struct Acc64F {
    static constexpr bool kFold = true;
    uint64_t s;
    __device__ __forceinline__ Acc64F() : s(0) {}
    __device__ __forceinline__ void add(uint32_t v) { s += v; }
    __device__ __forceinline__ void mad(uint32_t a, uint32_t x) { s += (uint64_t)a * x; }
    __device__ __forceinline__ void fold(uint32_t r32) {
        s = (uint64_t)(uint32_t)(s >> 32) * r32 + (uint32_t)s;
    }
    __device__ __forceinline__ uint32_t reduce(const DevMod &M) const { return mod64(s, M); }
};

// Addends of at most max((m-1)^2, m) an Acc64F can take between folds.
static inline uint32_t fold_capacity(uint32_t m, uint32_t r32) {
    const unsigned __int128 top = ((unsigned __int128)1 << 64) - 1;
    const unsigned __int128 base = ((unsigned __int128)(r32 + 1ull)) << 32;
    const unsigned __int128 add = std::max<unsigned __int128>((unsigned __int128)(m - 1ull) * (m - 1ull), m);
    if (base >= top) return 0;
    const unsigned __int128 f = (top - base) / add;
    return f > (1u << 30) ? (1u << 30) : (uint32_t)f;
}


// y' = (alpha*r + beta*y) mod m; alpha, beta already reduced mod m; beta == 0
// means y is not read by the caller.
__device__ __forceinline__ uint32_t epilogue(uint32_t r, uint32_t alpha, uint32_t beta,
                                             uint32_t yold, const DevMod &M) {
    uint32_t ar = alpha == 1u ? r : mod64((uint64_t)alpha * r, M);
    if (beta == 0u) return ar;
    uint32_t by = beta == 1u ? yold : mod64((uint64_t)beta * yold, M);
    uint64_t s = (uint64_t)ar + by;
    return (uint32_t)(s >= M.m ? s - M.m : s);
}

// Sum of residues across the lanes of a sub-warp (offsets lo..16 step *2).
__device__ __forceinline__ uint32_t sum_residues(uint32_t r, int first_off, int last_off,
                                                 const DevMod &M) {
    uint64_t s = r;
    for (int o = first_off; o <= last_off; o <<= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    return mod64(s, M);   // at most 32 residues: < 2^37
}

template <bool STREAM, class T>
__device__ __forceinline__ uint32_t ldm(const T *p) {
    if constexpr (STREAM) return ld_stream(p);
    else return ld_bcast(p);
}

// ------------------------------------------------------- entry walkers -----
// One +-1 slot: addend x or m - x; PAD_COL (sign bit clear) contributes 0.
template <class Acc, class GatherFn>
__device__ __forceinline__ void add_pm(Acc &acc, uint32_t c, uint32_t m, GatherFn g) {
    uint32_t xv = (c != PAD_COL) ? g(c & COL_MASK) : 0u;
    acc.add((c & SIGN_BIT) ? m - xv : xv);
}
template <class Acc, class GatherFn>
__device__ __forceinline__ void add_val(Acc &acc, uint32_t c, uint32_t a, GatherFn g) {
    uint32_t xv = (c != PAD_COL) ? g(c) : 0u;
    acc.mad(a, xv);
}

// Walk `count` +-1 slots at base, base+stride, ... and `vcount` valued slots,
// loading the matrix with LD (stream or broadcast policy), unrolled by 4 so
// four index loads are in flight before their gathers.
template <bool STREAM, class Acc, class VT, class GatherFn>
__device__ __forceinline__ void walk(Acc &acc, const uint32_t *pcol, uint32_t pbase, uint32_t pstride,
                                     uint32_t pcount, const uint32_t *vcol, const VT *vval,
                                     uint32_t vbase, uint32_t vstride, uint32_t vcount, uint32_t m,
                                     GatherFn g) {
    uint32_t j = 0;
    for (; j + 4 <= pcount; j += 4) {
        uint32_t c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = ldm<STREAM>(pcol + pbase + (j + u) * pstride);
#pragma unroll
        for (int u = 0; u < 4; ++u) add_pm(acc, c[u], m, g);
    }
    for (; j < pcount; ++j) add_pm(acc, ldm<STREAM>(pcol + pbase + j * pstride), m, g);
    j = 0;
    for (; j + 4 <= vcount; j += 4) {
        uint32_t c[4], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            c[u] = ldm<STREAM>(vcol + vbase + (j + u) * vstride);
            a[u] = ldm<STREAM>(vval + vbase + (j + u) * vstride);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) add_val(acc, c[u], a[u], g);
    }
    for (; j < vcount; ++j) {
        uint32_t i = vbase + j * vstride;
        add_val(acc, ldm<STREAM>(vcol + i), ldm<STREAM>(vval + i), g);
    }
}

}  // namespace ffspmv

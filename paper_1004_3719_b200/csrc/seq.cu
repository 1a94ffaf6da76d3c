// Block Wiedemann sequence S_t = U^T A^t X (P:438 step 1,
// device-resident iteration P:379-419).
//
// The iterate V_t stays on the device in ping-pong buffers, stored in the
// narrowest type holding a residue (u16 for m <= 65536, else u32), which
// halves the gather bytes of the dominant SpMM at m = 65521.  Per step:
//   project   partial[cta][a][b] = sum_{rows of cta} U[r][a] V_t[r][b] mod m
//   finalize  S[t][a][b] = sum_cta partial[cta][a][b] mod m
//   spmm      V_{t+1} = A V_t   (the block kernel of block.cuh, beta = 0)
#include <algorithm>
#include <cstdlib>

#include "block.cuh"
#include "l2window.hpp"
#include "seq_mma.cuh"

namespace ffspmv {

namespace {

constexpr int PROJ_THREADS = 256;
constexpr int PROJ_PPT = 4;  // output pairs per thread per pass

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

uint32_t proj_ctas(uint64_t n) {
    uint64_t c = std::min<uint64_t>((uint64_t)num_sms() * 4, (n + 63) / 64);   // 4 CTAs/SM of k_project_t
    return (uint32_t)std::max<uint64_t>(1, c);
}

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

template <class IT>
__global__ void k_seq_prep(const uint32_t *__restrict__ X, const uint32_t *__restrict__ U,
                           uint64_t nk, uint64_t nku, IT *__restrict__ V0, IT *__restrict__ Uc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk + nku;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < nk) V0[i] = (IT)X[i];
        else Uc[i - nk] = (IT)U[i - nk];
    }
}

template <class IT>
__global__ void k_seq_widen(const IT *__restrict__ V, uint64_t n, uint32_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = V[i];
}

// Exact projection partials.  CTA c owns a contiguous row range; U and V rows
// are staged through shared memory TR rows at a time; each thread owns up to
// PROJ_PPT (a, b) output pairs and accumulates sum_r U[r][a] V[r][b] exactly
// (u64 when rows_per_cta * (m-1)^2 < 2^64, else u96), then reduces mod m.
template <class IT, class Acc>
__global__ void __launch_bounds__(PROJ_THREADS)
k_project(const IT *__restrict__ V, const IT *__restrict__ Uc, uint64_t n, uint32_t k,
          uint32_t ku, uint32_t ldu, uint32_t tr, DevMod M, uint32_t *__restrict__ partial) {
    extern __shared__ uint32_t sm[];
    uint32_t *su = sm;               // tr x ku
    uint32_t *sv = sm + tr * ku;     // tr x k
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t r0 = blockIdx.x * per, r1 = (r0 + per < n) ? r0 + per : n;
    const uint32_t pairs = ku * k;
    for (uint32_t p0 = 0; p0 < pairs; p0 += PROJ_THREADS * PROJ_PPT) {
        Acc acc[PROJ_PPT];
        uint32_t pa[PROJ_PPT], pb[PROJ_PPT];
#pragma unroll
        for (int j = 0; j < PROJ_PPT; ++j) {
            uint32_t p = p0 + threadIdx.x + j * PROJ_THREADS;
            pa[j] = p < pairs ? p / k : 0;
            pb[j] = p < pairs ? p % k : 0;
        }
        for (uint64_t rb = r0; rb < r1; rb += tr) {
            const uint32_t nr = (uint32_t)((r1 - rb < tr) ? r1 - rb : tr);
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < nr * ku; i += PROJ_THREADS)
                su[i] = Uc[(rb + i / ku) * ldu + i % ku];
            for (uint32_t i = threadIdx.x; i < nr * k; i += PROJ_THREADS) sv[i] = V[rb * k + i];
            __syncthreads();
            for (uint32_t r = 0; r < nr; ++r) {
#pragma unroll
                for (int j = 0; j < PROJ_PPT; ++j) acc[j].mad(su[r * ku + pa[j]], sv[r * k + pb[j]]);
            }
        }
#pragma unroll
        for (int j = 0; j < PROJ_PPT; ++j) {
            uint32_t p = p0 + threadIdx.x + j * PROJ_THREADS;
            if (p < pairs) partial[(uint64_t)blockIdx.x * pairs + p] = acc[j].reduce(M);
        }
    }
}

// Register-tiled projection for k, ku <= 64 (the common case): thread
// (g, ta, tb) owns the 4 x 4 block of pairs a in [4ta, 4ta+4), b in [4tb, 4tb+4)
// for the rows r = g (mod G) of each staged tile, so a row costs two 16-byte
// shared loads per 16 exact MACs (instead of two 4-byte loads per MAC); the G
// row groups' residues are summed (< G m < 2^64) at the end.  Same partial
// layout and exactness argument as k_project.
constexpr uint32_t PROJ_TR = 64;

template <class IT, class Acc>
__global__ void __launch_bounds__(PROJ_THREADS)
k_project_t(const IT *__restrict__ V, const IT *__restrict__ Uc, uint64_t n, uint32_t k,
            uint32_t ku, uint32_t ldu, uint32_t tr, bool vec, DevMod M, uint32_t *__restrict__ partial) {
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t K4 = (k + 3) & ~3u, KU4 = (ku + 3) & ~3u;
    uint32_t *su = sm;                         // tr x KU4 (zero padded)
    uint32_t *sv = sm + tr * KU4;              // tr x K4
    const uint32_t ntb = K4 / 4, nt = (KU4 / 4) * ntb;
    const uint32_t G = PROJ_THREADS / nt;      // row groups, >= 1 (k, ku <= 64)
    const uint32_t tid = threadIdx.x, g = tid / nt, tt = tid - g * nt;
    const uint32_t ta = tt / ntb, tb = tt - ta * ntb;
    const bool active = g < G;
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t r0 = min(n, (uint64_t)blockIdx.x * per), r1 = min(n, r0 + per);
    Acc acc[16];
    for (uint64_t rb = r0; rb < r1; rb += tr) {
        const uint32_t nr = (uint32_t)min((uint64_t)tr, r1 - rb);
        __syncthreads();
        if (vec) {
            // u32, k and ku multiples of 4, U unpadded: both tiles are
            // contiguous runs of 16-byte vectors (zero beyond nr rows)
            const uint4 *u4 = reinterpret_cast<const uint4 *>(Uc + rb * ldu);
            const uint4 *v4 = reinterpret_cast<const uint4 *>(V + rb * k);
            const uint32_t nu = nr * KU4 / 4, nv = nr * K4 / 4;
            for (uint32_t i = tid; i < tr * KU4 / 4; i += PROJ_THREADS)
                reinterpret_cast<uint4 *>(su)[i] = i < nu ? __ldcs(u4 + i) : make_uint4(0, 0, 0, 0);
            for (uint32_t i = tid; i < tr * K4 / 4; i += PROJ_THREADS)
                reinterpret_cast<uint4 *>(sv)[i] = i < nv ? __ldcs(v4 + i) : make_uint4(0, 0, 0, 0);
        } else {
            for (uint32_t i = tid; i < tr * KU4; i += PROJ_THREADS) {
                const uint32_t r = i / KU4, c = i - r * KU4;
                su[i] = (r < nr && c < ku) ? (uint32_t)Uc[(rb + r) * ldu + c] : 0u;
            }
            for (uint32_t i = tid; i < tr * K4; i += PROJ_THREADS) {
                const uint32_t r = i / K4, c = i - r * K4;
                sv[i] = (r < nr && c < k) ? (uint32_t)V[(rb + r) * k + c] : 0u;
            }
        }
        __syncthreads();
        if (active) {
            for (uint32_t r = g; r < nr; r += G) {
                const uint4 u = *reinterpret_cast<const uint4 *>(su + r * KU4 + 4 * ta);
                const uint4 v = *reinterpret_cast<const uint4 *>(sv + r * K4 + 4 * tb);
                const uint32_t ua[4] = {u.x, u.y, u.z, u.w}, vb[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i * 4 + j].mad(ua[i], vb[j]);
            }
        }
    }
    __syncthreads();
    uint32_t *red = sm;                        // (G * nt) x 16 residues
    if (active) {
#pragma unroll
        for (int q = 0; q < 16; ++q) red[tid * 16 + q] = acc[q].reduce(M);
    }
    __syncthreads();
    const uint32_t pairs = ku * k;
    for (uint32_t p = tid; p < pairs; p += PROJ_THREADS) {
        const uint32_t a = p / k, b = p - a * k;
        const uint32_t t2 = (a >> 2) * ntb + (b >> 2), q = (a & 3) * 4 + (b & 3);
        uint64_t sacc = 0;
        for (uint32_t gg = 0; gg < G; ++gg) sacc += red[(gg * nt + t2) * 16 + q];
        partial[(uint64_t)blockIdx.x * pairs + p] = mod64(sacc, M);
    }
}

// S_t[p] = sum_c partial[c][p] mod m: one warp per output pair.
__global__ void k_seq_finalize(const uint32_t *__restrict__ partial, uint32_t nctas,
                               uint32_t pairs, DevMod M, uint32_t *__restrict__ S) {
    const uint32_t p = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (p >= pairs) return;
    uint64_t s = 0;   // < nctas * m < 2^64
    for (uint32_t c = lane; c < nctas; c += 32) s += partial[(uint64_t)c * pairs + p];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0) S[p] = mod64(s, M);
}

// ------------------------------------------------------------- fused step ---
// V_{t+1} = A V_t with the projection U^T V_{t+1} fused into the SpMM
// epilogue (SURVEY §8 a-8 + a-9): each lane owns one column of the iterate and
// accumulates P[a] += U[row][a] * V_{t+1}[row][col] for the rows it computes,
// exactly (u64 when every partial sum < 2^64, else u96).  U is staged in a
// padded internal copy (KUP columns, 16-byte rows) so its rows load as uint4.
// Persistent grid; the warps also finalise the previous step's S from its
// CTA partials, so one launch per step.
constexpr int SEQ_WARPS = 8;

template <class IT, int KUP, class PAcc>
struct SeqOut {
    IT *V;
    const IT *U;
    uint32_t k;
    PAcc P[KUP];
    __device__ __forceinline__ void put(uint32_t row, uint32_t col, bool colok, uint32_t r,
                                        const DevMod &M) {
        if (!colok) return;
        V[(uint64_t)row * k + col] = (IT)r;
        constexpr int PER = 16 / sizeof(IT);
        const uint4 *u4 = reinterpret_cast<const uint4 *>(U + (uint64_t)row * KUP);
#pragma unroll
        for (int q = 0; q < KUP / PER; ++q) {
            const uint4 w = __ldg(u4 + q);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                uint32_t ua;
                if constexpr (sizeof(IT) == 1) ua = (ws[e >> 2] >> (8 * (e & 3))) & 0xFFu;
                else if constexpr (sizeof(IT) == 2) ua = (ws[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                else ua = ws[e];
                P[q * PER + e].mad(ua, r);
            }
        }
    }
};

__device__ __forceinline__ void finalize_pairs(const uint32_t *__restrict__ part, uint32_t nctas,
                                               uint32_t pairs, uint32_t gw, uint32_t nw,
                                               uint32_t lane, const DevMod &M,
                                               uint32_t *__restrict__ S) {
    for (uint32_t p = gw; p < pairs; p += nw) {
        uint64_t s = 0;
        for (uint32_t c = lane; c < nctas; c += 32) s += part[(uint64_t)c * pairs + p];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) S[p] = mod64(s, M);
    }
}

template <class VT, int KP, class IT, int KUP, class PAcc>
__global__ void __launch_bounds__(SEQ_WARPS * 32)
k_seq_step(DevOp op, DevMod M, uint32_t k, uint32_t ku, const IT *__restrict__ Vin,
           IT *__restrict__ Vout, const IT *__restrict__ Uc, uint32_t *__restrict__ part_out,
           const uint32_t *__restrict__ part_prev, uint32_t nprev, uint32_t *__restrict__ S_prev) {
    __shared__ uint32_t red[SEQ_WARPS][KUP][KP];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * SEQ_WARPS + warp, nw = gridDim.x * SEQ_WARPS;
    const uint32_t pairs = ku * k;
    if (part_prev) finalize_pairs(part_prev, nprev, pairs, gw, nw, lane, M, S_prev);
    SeqOut<IT, KUP, PAcc> out{Vout, Uc, k};
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    for (uint32_t w = gw; w < items; w += nw) block_item<VT, KP, 8>(op, M, w, lane, k, Vin, k, out);
    // lanes g*KP + cl hold partials of column cl: sum the groups, then the warps
#pragma unroll
    for (int a = 0; a < KUP; ++a) {
        uint32_t r = sum_residues(out.P[a].reduce(M), KP, 16, M);
        if (lane < KP) red[warp][a][lane] = r;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < pairs; i += SEQ_WARPS * 32) {
        const uint32_t a = i / k, c = i - a * k;
        uint64_t s = 0;
#pragma unroll
        for (int w = 0; w < SEQ_WARPS; ++w) s += red[w][a][c];
        part_out[(uint64_t)blockIdx.x * pairs + i] = mod64(s, M);
    }
}

template <class IT, int KUP>
__global__ void k_seq_prep_pad(const uint32_t *__restrict__ X, const uint32_t *__restrict__ U,
                               uint64_t n, uint32_t k, uint32_t ku, IT *__restrict__ V0,
                               IT *__restrict__ Uc) {
    const uint64_t nk = n * k, nu = n * KUP;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk + nu;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < nk) {
            V0[i] = (IT)X[i];
        } else {
            const uint64_t j = i - nk, r = j / KUP;
            const uint32_t a = (uint32_t)(j - r * KUP);
            Uc[j] = a < ku ? (IT)U[r * ku + a] : (IT)0;
        }
    }
}

template <class IT>
struct SeqLayout {
    IT *V[2];
    IT *Uc;          // n x ku (unfused path) or n x KUP padded (fused path)
    uint32_t *partial[2];
    uint32_t *ufrag; // tensor-core path: per slice 256 u32 of U limbs in fragment order
    DevOp *opdev;    // device copy of the operator view (out-of-line scalar path)
    uint32_t *ctr;   // two work counters of the fused steps (step t uses ctr[t & 1])
    size_t bytes;
};

inline uint32_t kup_for(uint32_t ku) { return ku <= 16 ? 16 : 32; }
inline bool fused_ok(uint32_t k, uint32_t ku) { return k <= 32 && ku <= 32; }
// tensor-core projection: u16 iterate (2 limbs), 4 | k <= 16, ku <= 16
inline bool mma_ok(uint32_t m, uint32_t k, uint32_t ku) {
    return m <= 65536u && k % 4 == 0 && k >= 4 && k <= 16 && ku <= 16;
}
// byte-iterate kernel with the tensor-core projection: m <= 256, k = 16
inline bool mma_b_ok(uint32_t m, uint32_t k, uint32_t ku) { return m <= 256u && k == 16 && ku <= 16; }
// the fused tensor-core step for iterate type IT
template <class IT>
inline bool mma_for(uint32_t m, uint32_t k, uint32_t ku) {
    if constexpr (sizeof(IT) == 1) return mma_b_ok(m, k, ku);
    else if constexpr (sizeof(IT) == 2) return mma_ok(m, k, ku);
    else return false;
}
constexpr uint32_t MAX_STEP_CTAS_PER_SM = 8;

template <class IT>
SeqLayout<IT> layout(void *ws, const DevOp &op, uint32_t m, uint32_t k, uint32_t ku, uint32_t nctas) {
    SeqLayout<IT> L{};
    const uint64_t n = op.rows;
    char *p = (char *)ws;
    size_t off = 0;
    const bool mma = mma_for<IT>(m, k, ku);
    const uint32_t ucols = mma ? 0 : fused_ok(k, ku) ? kup_for(ku) : ku;
    // fused steps ping-pong two partial buffers of up to maxc CTA rows (the
    // step kernels' grid, or the projection's for S_0); the unfused path
    // only uses partial[0] with the projection's nctas rows
    const bool fused = mma || fused_ok(k, ku);
    const uint32_t maxc = fused ? std::max<uint32_t>(nctas, (uint32_t)num_sms() * MAX_STEP_CTAS_PER_SM)
                                : nctas;
    size_t vb = align256(n * (size_t)k * sizeof(IT));
    size_t ub = align256(n * (size_t)ucols * sizeof(IT));
    size_t pb = align256((size_t)maxc * ku * k * sizeof(uint32_t));
    size_t fb = mma ? align256((size_t)op.n_slices * 256 * sizeof(uint32_t)) : 0;
    L.V[0] = (IT *)(p + off); off += vb;
    L.V[1] = (IT *)(p + off); off += vb;
    L.Uc = (IT *)(p + off); off += ub;
    L.partial[0] = (uint32_t *)(p + off); off += pb;
    L.partial[1] = (uint32_t *)(p + off); off += fused ? pb : 0;
    L.ufrag = (uint32_t *)(p + off); off += fb;
    L.opdev = (DevOp *)(p + off); off += align256(sizeof(DevOp));
    L.ctr = (uint32_t *)(p + off); off += 256;
    L.bytes = off;
    return L;
}

// Projection partials of V (k_project) + optional finalisation into S_t.
template <class IT>
int project(const IT *V, const IT *Uc, uint32_t ldu, const DevMod &M, uint64_t n, uint32_t k,
            uint32_t ku, uint32_t *partial, uint32_t nctas, uint32_t *S_t, cudaStream_t st) {
    uint32_t tr = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(64, 12288 / (k + ku)));
    size_t smem = (size_t)tr * (k + ku) * sizeof(uint32_t);
    uint64_t per = (n + nctas - 1) / nctas;
    typedef unsigned __int128 u128;
    bool wide = (u128)per * (u128)(M.m - 1) * (u128)(M.m - 1) > (u128)~(uint64_t)0;
    if (k <= 64 && ku <= 64) {
        const uint32_t K4 = (k + 3) & ~3u, KU4 = (ku + 3) & ~3u;
        // 8192-word row tiles (32 KB): a few 16-byte loads in flight per thread
        const uint32_t trt = std::max<uint32_t>(PROJ_TR, std::min<uint32_t>(512, 8192 / (K4 + KU4)));
        const bool vec = sizeof(IT) == 4 && K4 == k && KU4 == ku && ldu == ku &&
                         ((uintptr_t)V & 15) == 0 && ((uintptr_t)Uc & 15) == 0;
        const size_t sm_t = std::max<size_t>((size_t)trt * (K4 + KU4), (size_t)PROJ_THREADS * 16) * 4;
        if (wide)
            k_project_t<IT, Acc96><<<nctas, PROJ_THREADS, sm_t, st>>>(V, Uc, n, k, ku, ldu, trt, vec, M, partial);
        else
            k_project_t<IT, Acc64><<<nctas, PROJ_THREADS, sm_t, st>>>(V, Uc, n, k, ku, ldu, trt, vec, M, partial);
    } else if (wide)
        k_project<IT, Acc96><<<nctas, PROJ_THREADS, smem, st>>>(V, Uc, n, k, ku, ldu, tr, M, partial);
    else
        k_project<IT, Acc64><<<nctas, PROJ_THREADS, smem, st>>>(V, Uc, n, k, ku, ldu, tr, M, partial);
    count_launch();
    if (S_t) {
        uint32_t pairs = ku * k;
        k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(partial, nctas, pairs, M, S_t);
        count_launch();
    }
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------- fused launch ---
template <class VT, int KP, class IT, int KUP, class PAcc>
int launch_step_t(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku, const IT *Vin,
                  IT *Vout, const IT *Uc, uint32_t *part_out, const uint32_t *part_prev,
                  uint32_t nprev, uint32_t *S_prev, uint32_t &nctas_out, cudaStream_t st) {
    auto kern = k_seq_step<VT, KP, IT, KUP, PAcc>;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SEQ_WARPS * 32, 0);
        occ = std::max(1, std::min<int>(occ, (int)MAX_STEP_CTAS_PER_SM));
    }
    uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    uint32_t nctas = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms() * occ, (items + SEQ_WARPS - 1) / SEQ_WARPS));
    kern<<<nctas, SEQ_WARPS * 32, 0, st>>>(op, M, k, ku, Vin, Vout, Uc, part_out, part_prev, nprev,
                                          S_prev);
    count_launch();
    nctas_out = nctas;
    return (int)cudaGetLastError();
}

template <class VT, class IT, int KUP, class PAcc>
int launch_step_kp(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku, const IT *Vin,
                   IT *Vout, const IT *Uc, uint32_t *po, const uint32_t *pp, uint32_t np,
                   uint32_t *Sp, uint32_t &nc, cudaStream_t st) {
    if (k <= 1) return launch_step_t<VT, 1, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    if (k <= 2) return launch_step_t<VT, 2, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    if (k <= 4) return launch_step_t<VT, 4, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    if (k <= 8) return launch_step_t<VT, 8, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    if (k <= 16) return launch_step_t<VT, 16, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    return launch_step_t<VT, 32, IT, KUP, PAcc>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
}

template <class IT>
int launch_step(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku, const IT *Vin, IT *Vout,
                const IT *Uc, uint32_t *po, const uint32_t *pp, uint32_t np, uint32_t *Sp,
                uint32_t &nc, cudaStream_t st) {
    // u8 iterate (m <= 256) and u16 iterate (m <= 65536): products < 2^32,
    // any n < 2^31 rows fit u64; u32 iterate: exact in u96
    if constexpr (sizeof(IT) == 1) {
        if (ku <= 16) return launch_step_kp<uint8_t, IT, 16, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
        return launch_step_kp<uint8_t, IT, 32, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    } else if constexpr (sizeof(IT) == 2) {
        if (ku <= 16) return launch_step_kp<uint16_t, IT, 16, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
        return launch_step_kp<uint16_t, IT, 32, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    } else {
        if (ku <= 16) return launch_step_kp<uint32_t, IT, 16, Acc96>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
        return launch_step_kp<uint32_t, IT, 32, Acc96>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
    }
}

// ------------------------------------------------- tensor-core projection ---
template <class VT, int KPV, int KP>
int launch_step_mma_t(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku,
                      const uint16_t *Vin, uint16_t *Vout, const uint32_t *U,
                      const uint32_t *ufrag, uint32_t *po, const uint32_t *pp, uint32_t np,
                      uint32_t *Sp, uint32_t &nc, cudaStream_t st) {
    auto kern = k_seq_step_mma<VT, KPV, KP>;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SMMA_WARPS * 32, 0);
        occ = std::max(1, std::min<int>(occ, (int)MAX_STEP_CTAS_PER_SM));
    }
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    const uint32_t nctas = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms() * occ, (items + SMMA_WARPS - 1) / SMMA_WARPS));
    kern<<<nctas, SMMA_WARPS * 32, 0, st>>>(op, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp);
    count_launch();
    nc = nctas;
    return (int)cudaGetLastError();
}

template <class VT, int LPR>
int launch_step_h_t(const DevOp &op, const DevOp *opdev, const DevMod &M, uint32_t k, uint32_t ku,
                    const uint16_t *Vin, uint16_t *Vout, const uint32_t *U, const uint32_t *ufrag,
                    uint32_t *po, const uint32_t *pp, uint32_t np, uint32_t *Sp, uint32_t &nc,
                    uint32_t *ctr, uint32_t *ctr_next, cudaStream_t st) {
    auto kern = k_seq_step_h<VT, LPR>;
    const int dsmem = FFSPMV_SEQ_AS ? SMMA_WARPS * (int)SeqRing<LPR>::bytes : 0;
    static int occ = 0;
    if (!occ) {
        if (dsmem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SMMA_WARPS * 32, dsmem);
        occ = std::max(1, std::min<int>(occ, (int)MAX_STEP_CTAS_PER_SM));
    }
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    const uint32_t nctas = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms() * occ, (items + SMMA_WARPS - 1) / SMMA_WARPS));
    kern<<<nctas, SMMA_WARPS * 32, dsmem, st>>>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp,
                                                ctr, ctr_next);
    count_launch();
    nc = nctas;
    return (int)cudaGetLastError();
}

template <class VT>
int launch_step_mma(const DevOp &op, const DevOp *opdev, const DevMod &M, uint32_t k, uint32_t ku,
                    const uint16_t *Vin, uint16_t *Vout, const uint32_t *U, const uint32_t *ufrag,
                    uint32_t *po, const uint32_t *pp, uint32_t np, uint32_t *Sp, uint32_t &nc,
                    uint32_t *ctr, uint32_t *ctr_next, cudaStream_t st) {
    // k = 8 / 16: the lean half-slice kernel (16-byte gathers, one row per lane)
    if (k == 8) return launch_step_h_t<VT, 1>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, ctr, ctr_next, st);
    if (k == 16) return launch_step_h_t<VT, 2>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, ctr, ctr_next, st);
    // remaining mma_ok widths: k = 4 (one lane per row) and k = 12 (four
    // 4-column lanes per row, the last one idle)
    if (k == 4) return launch_step_mma_t<VT, 1, 4>(op, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
    return launch_step_mma_t<VT, 4, 16>(op, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
}

int launch_step_b(const DevOp &op, const DevOp *opdev, const DevMod &M, uint32_t k, uint32_t ku,
                  const uint8_t *Vin, uint8_t *Vout, const uint32_t *U, const uint32_t *ufrag,
                  uint32_t *po, const uint32_t *pp, uint32_t np, uint32_t *Sp, uint32_t &nc,
                  uint32_t *ctr, uint32_t *ctr_next, cudaStream_t st) {
    auto kern = k_seq_step_b<uint8_t>;
    const int dsmem = FFSPMV_SEQB_AS ? SMMA_WARPS * (int)SeqRing<1>::bytes : 0;
    static int occ = 0;
    if (!occ) {
        if (dsmem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SMMA_WARPS * 32, dsmem);
        occ = std::max(1, std::min<int>(occ, (int)MAX_STEP_CTAS_PER_SM));
    }
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    const uint32_t nctas = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms() * occ, (items + SMMA_WARPS - 1) / SMMA_WARPS));
    kern<<<nctas, SMMA_WARPS * 32, dsmem, st>>>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp,
                                                ctr, ctr_next);
    count_launch();
    nc = nctas;
    return (int)cudaGetLastError();
}

// one fused tensor-core step for iterate type IT (u8: the byte kernel; u16:
// the half-slice / 4-column kernels; m <= 256 always takes the u8 iterate,
// so u16 iterates carry u16 values)
template <class IT>
int launch_step_tc(const DevOp &op, const DevOp *opdev, const DevMod &M, uint32_t k, uint32_t ku,
                   const IT *Vin, IT *Vout, const uint32_t *U, const uint32_t *ufrag, uint32_t *po,
                   const uint32_t *pp, uint32_t np, uint32_t *Sp, uint32_t &nc, uint32_t *ctr,
                   uint32_t *ctr_next, cudaStream_t st) {
    if constexpr (sizeof(IT) == 1)
        return launch_step_b(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, ctr, ctr_next, st);
    else
        return launch_step_mma<uint16_t>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, ctr,
                                         ctr_next, st);
}

template <class IT>
int run_sequence_mma(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                     const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out,
                     const SeqLayout<IT> &W, uint32_t nctas, cudaStream_t st) {
    const uint64_t n = op.rows;
    const uint32_t *Uu = U ? U : X;
    const uint32_t pairs = ku * k;
    int err;
    if ((err = (int)cudaMemcpyAsync(W.opdev, &op, sizeof(DevOp), cudaMemcpyHostToDevice, st))) return err;
    if ((err = (int)cudaMemsetAsync(W.ctr, 0, 8, st))) return err;
    {
        uint64_t tot = n * (uint64_t)k;
        uint32_t blocks = (uint32_t)std::min<uint64_t>((tot + 255) / 256, (uint64_t)num_sms() * 8);
        k_seq_prep<IT><<<std::max<uint32_t>(blocks, 1), 256, 0, st>>>(X, Uu, tot, 0, W.V[0], W.Uc);
        count_launch();
        if (op.n_slices) {
            uint64_t words = (uint64_t)op.n_slices * 256;
            uint32_t fblocks = (uint32_t)std::min<uint64_t>((words + 255) / 256, (uint64_t)num_sms() * 8);
            k_seq_ufrag<<<fblocks, 256, 0, st>>>(Uu, ku, op.perm, op.slices, op.n_slices, W.ufrag);
            count_launch();
        }
    }
    // S_0 partials straight from the caller's u32 X and U
    if ((err = project<uint32_t>(X, Uu, ku, M, n, k, ku, W.partial[0], nctas, nullptr, st)))
        return err;
    uint32_t nprev = nctas;
    L2Window win(st, n * (size_t)k * sizeof(IT));
    for (uint64_t t = 1; t < L; ++t) {
        uint32_t nc = 0;
        const IT *Vin = W.V[(t - 1) & 1];
        IT *Vout = W.V[t & 1];
        uint32_t *po = W.partial[t & 1];
        const uint32_t *pp = W.partial[(t - 1) & 1];
        uint32_t *Sp = S + (t - 1) * pairs;
        win.set(Vin);
        err = launch_step_tc<IT>(op, W.opdev, M, k, ku, Vin, Vout, Uu, W.ufrag, po, pp, nprev, Sp, nc,
                                 W.ctr + (t & 1), W.ctr + ((t + 1) & 1), st);
        if (err) return err;
        nprev = nc;
    }
    k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(W.partial[(L - 1) & 1], nprev, pairs, M,
                                                   S + (L - 1) * pairs);
    count_launch();
    if (V_out) {
        if ((err = launch_block_t<IT, uint32_t>(op, M, k, 1u, W.V[(L - 1) & 1], k, 0u, V_out, k, (void *)st)))
            return err;
    }
    return (int)cudaGetLastError();
}

template <class IT>
int run_sequence(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                 const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out, void *ws,
                 cudaStream_t st) {
    const uint64_t n = op.rows;
    const uint32_t nctas = proj_ctas(n);
    SeqLayout<IT> W = layout<IT>(ws, op, M.m, k, ku, nctas);
    if (L == 0) {
        if (V_out && n)
            return (int)cudaMemcpyAsync(V_out, X, n * (size_t)k * 4, cudaMemcpyDeviceToDevice, st);
        return 0;
    }
    if constexpr (sizeof(IT) <= 2) {
        if (mma_for<IT>(M.m, k, ku)) return run_sequence_mma<IT>(op, M, k, X, ku, U, L, S, V_out, W, nctas, st);
    }
    const bool fused = fused_ok(k, ku);
    const uint32_t ldu = fused ? kup_for(ku) : ku;
    const uint32_t pairs = ku * k;
    int err;
    {
        uint64_t tot = n * (uint64_t)(k + ldu);
        uint32_t blocks = (uint32_t)std::min<uint64_t>((tot + 255) / 256, (uint64_t)num_sms() * 8);
        if (fused) {
            if (ldu == 16)
                k_seq_prep_pad<IT, 16><<<blocks, 256, 0, st>>>(X, U ? U : X, n, k, ku, W.V[0], W.Uc);
            else
                k_seq_prep_pad<IT, 32><<<blocks, 256, 0, st>>>(X, U ? U : X, n, k, ku, W.V[0], W.Uc);
        } else {
            k_seq_prep<IT><<<blocks, 256, 0, st>>>(X, U ? U : X, n * (uint64_t)k, n * (uint64_t)ku,
                                                  W.V[0], W.Uc);
        }
        count_launch();
    }
    if (!fused) {
        for (uint64_t t = 0; t < L; ++t) {
            const IT *Vt = W.V[t & 1];
            if ((err = project<IT>(Vt, W.Uc, ldu, M, n, k, ku, W.partial[0], nctas, S + t * pairs, st)))
                return err;
            if (t + 1 < L) {
                if ((err = launch_block_t<IT, IT>(op, M, k, 1u, Vt, k, 0u, W.V[(t + 1) & 1], k, (void *)st)))
                    return err;
            } else if (V_out) {
                if ((err = launch_block_t<IT, uint32_t>(op, M, k, 1u, Vt, k, 0u, V_out, k, (void *)st)))
                    return err;
            }
        }
        return (int)cudaGetLastError();
    }
    // fused: S_0 partials from the projection kernel; step t (1..L-1) computes
    // V_t with its projection partials and finalises S_{t-1}
    if ((err = project<IT>(W.V[0], W.Uc, ldu, M, n, k, ku, W.partial[0], nctas, nullptr, st)))
        return err;
    uint32_t nprev = nctas;
    L2Window win(st, n * (size_t)k * sizeof(IT));
    for (uint64_t t = 1; t < L; ++t) {
        uint32_t nc = 0;
        win.set(W.V[(t - 1) & 1]);
        if ((err = launch_step<IT>(op, M, k, ku, W.V[(t - 1) & 1], W.V[t & 1], W.Uc,
                                   W.partial[t & 1], W.partial[(t - 1) & 1], nprev,
                                   S + (t - 1) * pairs, nc, st)))
            return err;
        nprev = nc;
    }
    k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(W.partial[(L - 1) & 1], nprev, pairs, M,
                                                   S + (L - 1) * pairs);
    count_launch();
    if (V_out) {
        if ((err = launch_block_t<IT, uint32_t>(op, M, k, 1u, W.V[(L - 1) & 1], k, 0u, V_out, k,
                                                (void *)st)))
            return err;
    }
    return (int)cudaGetLastError();
}

}  // namespace

// Stand-alone projection S = U^T V mod m (ku x k) of an n-row block, for the
// row-banded multi-GPU sequence (each rank projects its band).
size_t project_workspace(uint64_t n, uint32_t k, uint32_t ku) {
    return align256((size_t)proj_ctas(n) * ku * k * sizeof(uint32_t));
}

int launch_project(const DevMod &M, uint64_t n, uint32_t k, const uint32_t *V, uint32_t ku,
                   const uint32_t *U, uint32_t *S, void *ws, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return (int)cudaMemsetAsync(S, 0, (size_t)ku * k * 4, st);
    return project<uint32_t>(V, U, ku, M, n, k, ku, (uint32_t *)ws, proj_ctas(n), S, st);
}

__global__ void k_sum_mod(const uint32_t *__restrict__ parts, uint64_t count, uint32_t nparts,
                          DevMod M, uint32_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0;   // nparts residues < 2^32 each: exact for nparts < 2^32
        for (uint32_t p = 0; p < nparts; ++p) s += parts[(uint64_t)p * count + i];
        out[i] = mod64(s, M);
    }
}

int launch_sum_mod(const DevMod &M, uint64_t count, uint32_t nparts, const uint32_t *parts,
                   uint32_t *out, void *stream) {
    if (count == 0) return 0;
    uint32_t blocks = (uint32_t)std::min<uint64_t>((count + 255) / 256, (uint64_t)num_sms() * 8);
    k_sum_mod<<<blocks, 256, 0, (cudaStream_t)stream>>>(parts, count, nparts, M, out);
    count_launch();
    return (int)cudaGetLastError();
}

size_t sequence_workspace(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku) {
    const uint64_t n = op.rows;
    const uint32_t nctas = proj_ctas(n);
    if (M.m <= 256u) return layout<uint8_t>(nullptr, op, M.m, k, ku, nctas).bytes;
    if (M.m <= 65536u) return layout<uint16_t>(nullptr, op, M.m, k, ku, nctas).bytes;
    return layout<uint32_t>(nullptr, op, M.m, k, ku, nctas).bytes;
}

int launch_sequence(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                    const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out, void *ws,
                    size_t ws_bytes, void *stream) {
    (void)ws_bytes;
    cudaStream_t st = (cudaStream_t)stream;
    // the iterate in the narrowest type holding a residue (SURVEY a-8): u8
    // for m <= 256 ("compressed" vectors for small fields), u16, u32
    if (M.m <= 256u) return run_sequence<uint8_t>(op, M, k, X, ku, U, L, S, V_out, ws, st);
    if (M.m <= 65536u) return run_sequence<uint16_t>(op, M, k, X, ku, U, L, S, V_out, ws, st);
    return run_sequence<uint32_t>(op, M, k, X, ku, U, L, S, V_out, ws, st);
}

// ------------------------------------------------- distributed sequence ----
// Rank (i, j) of a P_r x P_c grid: band i of A (its
// columns renumbered into the padded iterate layout, q = band(c) * rows_max
// + c - b_band) and column block j of X.  The iterate V_t[:, block j] lives
// in the padded layout (P_r * rows_max rows); a step computes the band's rows
// of V_{t+1} straight into the rank's own slot of the next buffer and the
// exchange callback all-gathers the slots among the P_r ranks of block j.
// S_band[t] receives the band's projection residues U_band^T V_t[band, j].
namespace {

template <class IT>
__global__ void k_dist_prep(const uint32_t *__restrict__ X, uint32_t k, uint32_t c0, uint32_t kc,
                            uint64_t npad, uint32_t rows_max, const uint32_t *__restrict__ bstart,
                            IT *__restrict__ V0) {
    const uint64_t total = npad * kc;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = e / kc;
        const uint32_t c = (uint32_t)(e - q * kc);
        const uint32_t band = (uint32_t)(q / rows_max), r = (uint32_t)(q - (uint64_t)band * rows_max);
        const uint32_t b0 = bstart[band], h = bstart[band + 1] - b0;
        V0[e] = r < h ? (IT)X[(uint64_t)(b0 + r) * k + c0 + c] : (IT)0;
    }
}

// band copies: Xb = X[row0 .. row0 + h, c0 .. c0 + kc), Ub = U[row0 .. row0 + h, :]
__global__ void k_dist_band(const uint32_t *__restrict__ X, uint32_t k, uint32_t c0, uint32_t kc,
                            const uint32_t *__restrict__ U, uint32_t ku, uint64_t row0, uint64_t h,
                            uint32_t *__restrict__ Xb, uint32_t *__restrict__ Ub) {
    const uint64_t nx = h * kc, total = nx + h * ku;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (e < nx) {
            const uint64_t r = e / kc;
            Xb[e] = X[(row0 + r) * k + c0 + (e - r * kc)];
        } else {
            const uint64_t f = e - nx;
            Ub[f] = U[row0 * ku + f];
        }
    }
}

template <class IT, int KUP>
__global__ void k_dist_upad(const uint32_t *__restrict__ Ub, uint64_t h, uint32_t ku, IT *__restrict__ Uc) {
    const uint64_t total = h * KUP;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / KUP;
        const uint32_t a = (uint32_t)(e - r * KUP);
        Uc[e] = a < ku ? (IT)Ub[r * ku + a] : (IT)0;
    }
}

template <class IT>
struct DistLayout {
    IT *V[2];
    uint32_t *Xb, *Ub;
    IT *Uc;
    uint32_t *partial[2];
    uint32_t *ufrag;
    DevOp *opdev;
    uint32_t *bstart;
    uint32_t *ctr;
    size_t bytes;
};

template <class IT>
DistLayout<IT> dist_layout(void *ws, const DevOp &op, uint32_t m, uint32_t kc, uint32_t ku, uint32_t pr) {
    DistLayout<IT> L{};
    const uint64_t h = op.rows, npad = op.cols;
    char *p = (char *)ws;
    size_t off = 0;
    const bool mma = mma_for<IT>(m, kc, ku);
    const bool fused = mma || fused_ok(kc, ku);
    const uint32_t ucols = mma ? 0 : fused_ok(kc, ku) ? kup_for(ku) : ku;
    const uint32_t nctas = proj_ctas(h);
    const uint32_t maxc = fused ? std::max<uint32_t>(nctas, (uint32_t)num_sms() * MAX_STEP_CTAS_PER_SM) : nctas;
    auto take = [&](size_t b) { void *q = p + off; off += align256(b); return q; };
    L.V[0] = (IT *)take(npad * (size_t)kc * sizeof(IT));
    L.V[1] = (IT *)take(npad * (size_t)kc * sizeof(IT));
    L.Xb = (uint32_t *)take(h * (size_t)kc * 4);
    L.Ub = (uint32_t *)take(h * (size_t)ku * 4);
    L.Uc = (IT *)take(h * (size_t)ucols * sizeof(IT));
    L.partial[0] = (uint32_t *)take((size_t)maxc * ku * kc * 4);
    L.partial[1] = (uint32_t *)take(fused ? (size_t)maxc * ku * kc * 4 : 0);
    L.ufrag = (uint32_t *)take(mma ? (size_t)op.n_slices * 256 * 4 : 0);
    L.opdev = (DevOp *)take(sizeof(DevOp));
    L.bstart = (uint32_t *)take((size_t)(pr + 1) * 4);
    L.ctr = (uint32_t *)take(8);
    L.bytes = off;
    return L;
}

template <class IT>
int run_sequence_dist(const DevOp &op, const DevMod &M, const uint32_t *X, uint32_t k, uint32_t ku,
                      const uint32_t *U, uint64_t L, uint32_t *S_band, uint32_t *V_band, void *ws,
                      const DistSeq &d, cudaStream_t st) {
    const uint64_t h = op.rows, npad = op.cols;
    const uint32_t kc = d.kc, pairs = ku * kc;
    DistLayout<IT> W = dist_layout<IT>(ws, op, M.m, kc, ku, d.pr);
    const uint32_t *Uu = U ? U : X;
    const uint32_t grid = (uint32_t)num_sms() * 8;
    int err;
    if ((err = (int)cudaMemcpyAsync(W.opdev, &op, sizeof(DevOp), cudaMemcpyHostToDevice, st))) return err;
    if ((err = (int)cudaMemcpyAsync(W.bstart, d.bstart, (d.pr + 1) * 4ull, cudaMemcpyHostToDevice, st))) return err;
    if ((err = (int)cudaMemsetAsync(W.ctr, 0, 8, st))) return err;
    k_dist_prep<IT><<<grid, 256, 0, st>>>(X, k, d.c0, kc, npad, d.rows_max, W.bstart, W.V[0]);
    count_launch();
    if (h) {
        k_dist_band<<<grid, 256, 0, st>>>(X, k, d.c0, kc, Uu, ku, d.row0, h, W.Xb, W.Ub);
        count_launch();
    }
    const bool mma = mma_for<IT>(M.m, kc, ku);
    const bool fused = mma || fused_ok(kc, ku);
    const uint32_t ldu = mma ? ku : fused ? kup_for(ku) : ku;
    if (h && mma && op.n_slices) {
        const uint64_t words = (uint64_t)op.n_slices * 256;
        k_seq_ufrag<<<(uint32_t)std::min<uint64_t>((words + 255) / 256, grid), 256, 0, st>>>(
            W.Ub, ku, op.perm, op.slices, op.n_slices, W.ufrag);
        count_launch();
    }
    if (h && !mma && fused) {
        if (ldu == 16) k_dist_upad<IT, 16><<<grid, 256, 0, st>>>(W.Ub, h, ku, W.Uc);
        else k_dist_upad<IT, 32><<<grid, 256, 0, st>>>(W.Ub, h, ku, W.Uc);
        count_launch();
    }
    const IT *Ufused = mma ? nullptr : fused ? W.Uc : nullptr;
    const uint32_t nctas = proj_ctas(std::max<uint64_t>(h, 1));
    auto project_band = [&](const uint32_t *V32, const IT *Vn, uint32_t *S_t) -> int {
        if (!h) return (int)cudaMemsetAsync(S_t, 0, (size_t)pairs * 4, st);
        if (V32) return project<uint32_t>(V32, W.Ub, ku, M, h, kc, ku, W.partial[0], nctas, S_t, st);
        return project<IT>(Vn, W.Uc, ldu, M, h, kc, ku, W.partial[0], nctas, S_t, st);
    };
    const size_t slot = (size_t)d.rows_max * kc;   // elements of one rank's slot
    if (!fused) {
        // unfused: project the band, then the band's block apply into its slot
        if (!mma && ldu == ku && h) {
            k_seq_prep<IT><<<grid, 256, 0, st>>>(Uu + d.row0 * ku, nullptr, h * (uint64_t)ku, 0, W.Uc, nullptr);
            count_launch();
        }
        for (uint64_t t = 0; t < L; ++t) {
            const IT *Vt = W.V[t & 1];
            if ((err = t == 0 ? project_band(W.Xb, nullptr, S_band) :
                                project_band(nullptr, Vt + d.own * kc, S_band + t * pairs)))
                return err;
            if (t + 1 < L) {
                if (h && (err = launch_block_t<IT, IT>(op, M, kc, 1u, Vt, kc, 0u, W.V[(t + 1) & 1] + d.own * kc,
                                                      kc, (void *)st)))
                    return err;
                if ((err = d.exchange(d.ctx, W.V[(t + 1) & 1], slot * sizeof(IT), (void *)st))) return err;
            }
        }
    } else {
        if (h) {
            if ((err = project<uint32_t>(W.Xb, W.Ub, ku, M, h, kc, ku, W.partial[0], nctas, nullptr, st)))
                return err;                                              // S_0 partials
        } else if ((err = (int)cudaMemsetAsync(S_band, 0, (size_t)L * pairs * 4, st))) {
            return err;
        }
        uint32_t nprev = nctas;
        L2Window win(st, npad * (size_t)kc * sizeof(IT));
        for (uint64_t t = 1; t < L; ++t) {
            uint32_t nc = nprev;
            const IT *Vin = W.V[(t - 1) & 1];
            win.set(Vin);
            IT *Vout = W.V[t & 1] + d.own * kc;
            if (h) {
                uint32_t *po = W.partial[t & 1];
                const uint32_t *pp = W.partial[(t - 1) & 1];
                uint32_t *Sp = S_band + (t - 1) * pairs;
                if constexpr (sizeof(IT) <= 2) {
                    if (mma) {
                        err = launch_step_tc<IT>(op, W.opdev, M, kc, ku, Vin, Vout, W.Ub, W.ufrag, po, pp, nprev,
                                                 Sp, nc, W.ctr + (t & 1), W.ctr + ((t + 1) & 1), st);
                    } else {
                        err = launch_step<IT>(op, M, kc, ku, Vin, Vout, Ufused, po, pp, nprev, Sp, nc, st);
                    }
                } else {
                    err = launch_step<IT>(op, M, kc, ku, Vin, Vout, Ufused, po, pp, nprev, Sp, nc, st);
                }
                if (err) return err;
            }
            nprev = nc;
            if ((err = d.exchange(d.ctx, W.V[t & 1], slot * sizeof(IT), (void *)st))) return err;
        }
        if (h && L) {
            k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(W.partial[(L - 1) & 1], nprev, pairs, M,
                                                           S_band + (L - 1) * pairs);
            count_launch();
        }
    }
    if (V_band && h && L) {
        if ((err = launch_block_t<IT, uint32_t>(op, M, kc, 1u, W.V[(L - 1) & 1], kc, 0u, V_band, kc, (void *)st)))
            return err;
    }
    return (int)cudaGetLastError();
}

// S[t][a][c_j + c] = sum_i G_(i, j)[t][a][c] mod m over the P_r row bands;
// G = the all-gathered band residues, rank (i, j)'s slot at (i P_c + j)
// L ku kcmax holding L x ku x kc_j (c_j = k j / P_c, kc_j = c_{j+1} - c_j)
__device__ __forceinline__ uint32_t col_block(uint32_t col, uint32_t k, uint32_t pc) {
    uint32_t j = (uint32_t)(((uint64_t)col * pc) / k);
    while (j > 0 && (uint64_t)k * j / pc > col) --j;
    while (j + 1 < pc && (uint64_t)k * (j + 1) / pc <= col) ++j;
    return j;
}

__global__ void k_dist_sum_S(const uint32_t *__restrict__ G, uint64_t L, uint32_t ku, uint32_t k,
                             uint32_t kcmax, uint32_t pr, uint32_t pc, DevMod M, uint32_t *__restrict__ S) {
    const uint64_t total = L * ku * (uint64_t)k;
    const uint64_t slot = L * ku * (uint64_t)kcmax;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t ta = e / k;
        const uint32_t col = (uint32_t)(e - ta * k);
        const uint32_t j = col_block(col, k, pc);
        const uint32_t cj = (uint32_t)((uint64_t)k * j / pc), kcj = (uint32_t)((uint64_t)k * (j + 1) / pc) - cj;
        uint64_t s = 0;   // P_r residues: exact
        for (uint32_t i = 0; i < pr; ++i) s += G[(uint64_t)(i * pc + j) * slot + ta * kcj + (col - cj)];
        S[e] = mod64(s, M);
    }
}

// V_out[b_i + r][c_j + c] = Gv_(i, j)[r][c] (the all-gathered band blocks of
// V_L, rank (i, j)'s slot at (i P_c + j) rows_max kcmax holding h_i x kc_j)
__global__ void k_dist_put_V(const uint32_t *__restrict__ Gv, uint64_t n, uint32_t k, uint32_t kcmax,
                             uint32_t rows_max, uint32_t pr, uint32_t pc, const uint32_t *__restrict__ bstart,
                             uint32_t *__restrict__ V_out) {
    const uint64_t total = n * k;
    const uint64_t slot = (uint64_t)rows_max * kcmax;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = e / k;
        const uint32_t col = (uint32_t)(e - row * k);
        uint32_t lo = 0, hi = pr;   // band: the last i with bstart[i] <= row
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (bstart[mid] <= row) lo = mid; else hi = mid;
        }
        const uint32_t j = col_block(col, k, pc);
        const uint32_t cj = (uint32_t)((uint64_t)k * j / pc), kcj = (uint32_t)((uint64_t)k * (j + 1) / pc) - cj;
        V_out[e] = Gv[(uint64_t)(lo * pc + j) * slot + (row - bstart[lo]) * kcj + (col - cj)];
    }
}

}  // namespace

size_t sequence_dist_workspace(const DevOp &op, const DevMod &M, uint32_t kc, uint32_t ku, uint32_t pr) {
    if (M.m <= 256u) return dist_layout<uint8_t>(nullptr, op, M.m, kc, ku, pr).bytes;
    if (M.m <= 65536u) return dist_layout<uint16_t>(nullptr, op, M.m, kc, ku, pr).bytes;
    return dist_layout<uint32_t>(nullptr, op, M.m, kc, ku, pr).bytes;
}

int launch_sequence_dist(const DevOp &op, const DevMod &M, const uint32_t *X, uint32_t k, uint32_t ku,
                         const uint32_t *U, uint64_t L, uint32_t *S_band, uint32_t *V_band, void *ws,
                         const DistSeq &d, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (M.m <= 256u) return run_sequence_dist<uint8_t>(op, M, X, k, ku, U, L, S_band, V_band, ws, d, st);
    if (M.m <= 65536u) return run_sequence_dist<uint16_t>(op, M, X, k, ku, U, L, S_band, V_band, ws, d, st);
    return run_sequence_dist<uint32_t>(op, M, X, k, ku, U, L, S_band, V_band, ws, d, st);
}

int launch_dist_sum_S(const uint32_t *G, uint64_t L, uint32_t ku, uint32_t k, uint32_t kcmax, uint32_t pr,
                      uint32_t pc, const DevMod &M, uint32_t *S, void *stream) {
    const uint64_t total = L * ku * (uint64_t)k;
    if (!total) return 0;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 8);
    k_dist_sum_S<<<blocks, 256, 0, (cudaStream_t)stream>>>(G, L, ku, k, kcmax, pr, pc, M, S);
    count_launch();
    return (int)cudaGetLastError();
}

int launch_dist_prep_x(const uint32_t *X, uint32_t k, uint32_t c0, uint32_t kc, uint64_t npad,
                       uint32_t rows_max, const uint32_t *bstart_dev, uint32_t *Xp, void *stream) {
    if (!npad || !kc) return 0;
    k_dist_prep<uint32_t><<<(uint32_t)num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(X, k, c0, kc, npad, rows_max,
                                                                                    bstart_dev, Xp);
    count_launch();
    return (int)cudaGetLastError();
}

int launch_dist_put_V(const uint32_t *Gv, uint64_t n, uint32_t k, uint32_t kcmax, uint32_t rows_max,
                      uint32_t pr, uint32_t pc, const uint32_t *bstart_dev, uint32_t *V_out, void *stream) {
    const uint64_t total = n * k;
    if (!total) return 0;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 8);
    k_dist_put_V<<<blocks, 256, 0, (cudaStream_t)stream>>>(Gv, n, k, kcmax, rows_max, pr, pc, bstart_dev, V_out);
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace ffspmv

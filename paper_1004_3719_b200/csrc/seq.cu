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

#include "block.cuh"
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
                if constexpr (sizeof(IT) == 2) ua = (ws[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
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
    size_t bytes;
};

inline uint32_t kup_for(uint32_t ku) { return ku <= 16 ? 16 : 32; }
inline bool fused_ok(uint32_t k, uint32_t ku) { return k <= 32 && ku <= 32; }
// tensor-core projection: u16 iterate (2 limbs), 4 | k <= 16, ku <= 16
inline bool mma_ok(uint32_t m, uint32_t k, uint32_t ku) {
    return m <= 65536u && k % 4 == 0 && k >= 4 && k <= 16 && ku <= 16;
}
constexpr uint32_t MAX_STEP_CTAS_PER_SM = 8;

template <class IT>
SeqLayout<IT> layout(void *ws, const DevOp &op, uint32_t m, uint32_t k, uint32_t ku, uint32_t nctas) {
    SeqLayout<IT> L{};
    const uint64_t n = op.rows;
    char *p = (char *)ws;
    size_t off = 0;
    const bool mma = sizeof(IT) == 2 && mma_ok(m, k, ku);
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
    // u16 iterate (m <= 65536): products < 2^32, any n < 2^31 rows fit u64;
    // u32 iterate: exact in u96
    if constexpr (sizeof(IT) == 2) {
        if (M.vbytes == 1) {
            if (ku <= 16) return launch_step_kp<uint8_t, IT, 16, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
            return launch_step_kp<uint8_t, IT, 32, Acc64>(op, M, k, ku, Vin, Vout, Uc, po, pp, np, Sp, nc, st);
        }
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
                    cudaStream_t st) {
    auto kern = k_seq_step_h<VT, LPR>;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SMMA_WARPS * 32, 0);
        occ = std::max(1, std::min<int>(occ, (int)MAX_STEP_CTAS_PER_SM));
    }
    const uint32_t items = op.n_long + op.n_slices + op.n_groups + (op.n_zero_rows + 31) / 32;
    const uint32_t nctas = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms() * occ, (items + SMMA_WARPS - 1) / SMMA_WARPS));
    kern<<<nctas, SMMA_WARPS * 32, 0, st>>>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp);
    count_launch();
    nc = nctas;
    return (int)cudaGetLastError();
}

template <class VT>
int launch_step_mma(const DevOp &op, const DevOp *opdev, const DevMod &M, uint32_t k, uint32_t ku,
                    const uint16_t *Vin, uint16_t *Vout, const uint32_t *U, const uint32_t *ufrag,
                    uint32_t *po, const uint32_t *pp, uint32_t np, uint32_t *Sp, uint32_t &nc,
                    cudaStream_t st) {
    // k = 8 / 16: the lean half-slice kernel (16-byte gathers, one row per lane)
    if (k == 8) return launch_step_h_t<VT, 1>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
    if (k == 16) return launch_step_h_t<VT, 2>(op, opdev, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
    // remaining mma_ok widths: k = 4 (one lane per row) and k = 12 (four
    // 4-column lanes per row, the last one idle)
    if (k == 4) return launch_step_mma_t<VT, 1, 4>(op, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
    return launch_step_mma_t<VT, 4, 16>(op, M, k, ku, Vin, Vout, U, ufrag, po, pp, np, Sp, nc, st);
}

int run_sequence_mma(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                     const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out,
                     const SeqLayout<uint16_t> &W, uint32_t nctas, cudaStream_t st) {
    const uint64_t n = op.rows;
    const uint32_t *Uu = U ? U : X;
    const uint32_t pairs = ku * k;
    int err;
    if ((err = (int)cudaMemcpyAsync(W.opdev, &op, sizeof(DevOp), cudaMemcpyHostToDevice, st))) return err;
    {
        uint64_t tot = n * (uint64_t)k;
        uint32_t blocks = (uint32_t)std::min<uint64_t>((tot + 255) / 256, (uint64_t)num_sms() * 8);
        k_seq_prep<uint16_t><<<std::max<uint32_t>(blocks, 1), 256, 0, st>>>(X, Uu, tot, 0, W.V[0], W.Uc);
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
    for (uint64_t t = 1; t < L; ++t) {
        uint32_t nc = 0;
        const uint16_t *Vin = W.V[(t - 1) & 1];
        uint16_t *Vout = W.V[t & 1];
        uint32_t *po = W.partial[t & 1];
        const uint32_t *pp = W.partial[(t - 1) & 1];
        uint32_t *Sp = S + (t - 1) * pairs;
        err = M.vbytes == 1
                  ? launch_step_mma<uint8_t>(op, W.opdev, M, k, ku, Vin, Vout, Uu, W.ufrag, po, pp, nprev, Sp, nc, st)
                  : launch_step_mma<uint16_t>(op, W.opdev, M, k, ku, Vin, Vout, Uu, W.ufrag, po, pp, nprev, Sp, nc, st);
        if (err) return err;
        nprev = nc;
    }
    k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(W.partial[(L - 1) & 1], nprev, pairs, M,
                                                   S + (L - 1) * pairs);
    count_launch();
    if (V_out) {
        if ((err = launch_block_t<uint16_t, uint32_t>(op, M, k, 1u, W.V[(L - 1) & 1], k, 0u, V_out,
                                                      k, (void *)st)))
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
    if constexpr (sizeof(IT) == 2) {
        if (mma_ok(M.m, k, ku)) return run_sequence_mma(op, M, k, X, ku, U, L, S, V_out, W, nctas, st);
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
    for (uint64_t t = 1; t < L; ++t) {
        uint32_t nc = 0;
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
    if (M.m <= 65536u) return layout<uint16_t>(nullptr, op, M.m, k, ku, nctas).bytes;
    return layout<uint32_t>(nullptr, op, M.m, k, ku, nctas).bytes;
}

int launch_sequence(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                    const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out, void *ws,
                    size_t ws_bytes, void *stream) {
    (void)ws_bytes;
    cudaStream_t st = (cudaStream_t)stream;
    if (M.m <= 65536u) return run_sequence<uint16_t>(op, M, k, X, ku, U, L, S, V_out, ws, st);
    return run_sequence<uint32_t>(op, M, k, X, ku, U, L, S, V_out, ws, st);
}

}  // namespace ffspmv

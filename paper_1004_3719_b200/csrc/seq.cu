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
    uint64_t c = std::min<uint64_t>((uint64_t)num_sms() * 2, (n + 63) / 64);
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
          uint32_t ku, uint32_t tr, DevMod M, uint32_t *__restrict__ partial) {
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
            for (uint32_t i = threadIdx.x; i < nr * ku; i += PROJ_THREADS) su[i] = Uc[rb * ku + i];
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

template <class IT>
struct SeqLayout {
    IT *V[2];
    IT *Uc;
    uint32_t *partial;
    size_t bytes;
};

template <class IT>
SeqLayout<IT> layout(void *ws, uint64_t n, uint32_t k, uint32_t ku, uint32_t nctas) {
    SeqLayout<IT> L{};
    char *p = (char *)ws;
    size_t off = 0;
    size_t vb = align256(n * (size_t)k * sizeof(IT));
    size_t ub = align256(n * (size_t)ku * sizeof(IT));
    size_t pb = align256((size_t)nctas * ku * k * sizeof(uint32_t));
    L.V[0] = (IT *)(p + off); off += vb;
    L.V[1] = (IT *)(p + off); off += vb;
    L.Uc = (IT *)(p + off); off += ub;
    L.partial = (uint32_t *)(p + off); off += pb;
    L.bytes = off;
    return L;
}

template <class IT>
int project(const DevOp &op, const DevMod &M, const IT *V, const IT *Uc, uint64_t n, uint32_t k,
            uint32_t ku, uint32_t *partial, uint32_t nctas, uint32_t *S_t, cudaStream_t st) {
    uint32_t tr = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(64, 12288 / (k + ku)));
    size_t smem = (size_t)tr * (k + ku) * sizeof(uint32_t);
    uint64_t per = (n + nctas - 1) / nctas;
    typedef unsigned __int128 u128;
    bool wide = (u128)per * (u128)(M.m - 1) * (u128)(M.m - 1) > (u128)~(uint64_t)0;
    if (wide)
        k_project<IT, Acc96><<<nctas, PROJ_THREADS, smem, st>>>(V, Uc, n, k, ku, tr, M, partial);
    else
        k_project<IT, Acc64><<<nctas, PROJ_THREADS, smem, st>>>(V, Uc, n, k, ku, tr, M, partial);
    count_launch();
    uint32_t pairs = ku * k;
    k_seq_finalize<<<(pairs + 7) / 8, 256, 0, st>>>(partial, nctas, pairs, M, S_t);
    count_launch();
    (void)op;
    return (int)cudaGetLastError();
}

template <class IT>
int run_sequence(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X, uint32_t ku,
                 const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out, void *ws,
                 cudaStream_t st) {
    const uint64_t n = op.rows;
    const uint32_t nctas = proj_ctas(n);
    SeqLayout<IT> W = layout<IT>(ws, n, k, ku, nctas);
    if (L == 0) {
        if (V_out && n)
            return (int)cudaMemcpyAsync(V_out, X, n * (size_t)k * 4, cudaMemcpyDeviceToDevice, st);
        return 0;
    }
    int err;
    {
        uint64_t tot = n * (uint64_t)(k + ku);
        uint32_t blocks = (uint32_t)std::min<uint64_t>((tot + 255) / 256, (uint64_t)num_sms() * 8);
        if (blocks) {
            k_seq_prep<IT><<<blocks, 256, 0, st>>>(X, U ? U : X, n * (uint64_t)k, n * (uint64_t)ku,
                                                  W.V[0], W.Uc);
            count_launch();
        }
    }
    for (uint64_t t = 0; t < L; ++t) {
        const IT *Vt = W.V[t & 1];
        if ((err = project<IT>(op, M, Vt, W.Uc, n, k, ku, W.partial, nctas,
                               S + t * (uint64_t)ku * k, st)))
            return err;
        if (t + 1 < L) {
            if ((err = launch_block_t<IT, IT>(op, M, k, 1u, Vt, k, 0u, W.V[(t + 1) & 1], k,
                                              (void *)st)))
                return err;
        } else if (V_out) {
            if ((err = launch_block_t<IT, uint32_t>(op, M, k, 1u, Vt, k, 0u, V_out, k, (void *)st)))
                return err;
        }
    }
    return (int)cudaGetLastError();
}

}  // namespace

size_t sequence_workspace(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku) {
    const uint64_t n = op.rows;
    const uint32_t nctas = proj_ctas(n);
    if (M.m <= 65536u) return layout<uint16_t>(nullptr, n, k, ku, nctas).bytes;
    return layout<uint32_t>(nullptr, n, k, ku, nctas).bytes;
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

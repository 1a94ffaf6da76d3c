// Microbenchmark 3: random ROW gathers of R bytes from an L2-resident array
// (the X / V_t access of the block and sequence kernels), four ways:
//   ldg    LDG.128 per lane, R/16 lanes per row, 8 independent loads in flight
//   lsts   cp.async.cg 16 B per lane into a shared ring (LDGSTS), D groups deep
//   bulk   cp.async.bulk (1-D, R bytes) per row, one per lane, mbarrier ring
//   g4     cp.async.bulk.tensor.2d ... tile::gather4 (4 rows per instruction)
// Each reads every gathered byte once (sum), so the comparison is fair.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gb3 tools/gather_bench3.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R>
__global__ void k_ldg(const uint32_t *__restrict__ idx, const uint4 *__restrict__ X, uint32_t n, uint32_t *out) {
    constexpr int LPR = R / 16, RPW = 32 / LPR;   // lanes per row, rows per warp instruction
    const uint32_t lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (uint32_t base = warp * RPW * 8; base < n; base += nw * RPW * 8) {
        uint32_t r[8];
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = base + u * RPW + sub < n ? __ldg(idx + base + u * RPW + sub) : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(X + (uint64_t)r[u] * LPR + sl);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// cp.async 16 B per lane; per warp a ring of D stages x (32 lanes x 16 B x U)
template <int R, int D, int U>
__global__ void k_lsts(const uint32_t *__restrict__ idx, const uint4 *__restrict__ X, uint32_t n, uint32_t *out) {
    constexpr int LPR = R / 16, RPW = 32 / LPR;
    extern __shared__ uint4 sm[];
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5, sub = lane / LPR, sl = lane % LPR;
    uint4 *ring = sm + (size_t)wl * D * U * 32;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t per = RPW * U;              // rows per stage
    uint32_t acc = 0;
    uint32_t b = warp * per;
    auto issue = [&](uint32_t base, int st) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = base + u * RPW + sub;
            const uint32_t r = i < n ? __ldg(idx + i) : 0;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(ring + (st * U + u) * 32 + lane)),
                         "l"(X + (uint64_t)r * LPR + sl) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int s = 0; s < D - 1; ++s) issue(b + s * nw * per, s);
    int st = 0;
    for (; b < n; b += nw * per) {
        issue(b + (D - 1) * nw * per, (st + D - 1) % D);
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint4 v = ring[(st * U + u) * 32 + lane];
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        st = (st + 1) % D;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                 ::"r"(mbar), "r"(phase) : "memory");
}

// cp.async.bulk per row (lane i issues row i of the stage); D stages x 32 rows per warp
template <int R, int D>
__global__ void k_bulk(const uint32_t *__restrict__ idx, const unsigned char *__restrict__ X, uint32_t n, uint32_t *out) {
    extern __shared__ __align__(128) unsigned char smb[];
    __shared__ uint64_t mb[32 * D];
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char *ring = smb + (size_t)wl * D * 32 * R;
    const uint32_t mbw = sa(&mb[wl * D]);
    if (lane < D) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbw + 8 * lane) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    auto issue = [&](uint32_t base, int st) {
        const uint32_t i = base + lane;
        const uint32_t r = i < n ? __ldg(idx + i) : 0;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbw + 8 * st), "r"(32 * R) : "memory");
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(ring + (st * 32 + lane) * R)), "l"(X + (uint64_t)r * R), "n"(R), "r"(mbw + 8 * st) : "memory");
    };
    uint32_t b = warp * 32;
#pragma unroll
    for (int s = 0; s < D - 1; ++s) issue(b + s * nw * 32, s);
    uint32_t phase = 0;
    int st = 0;
    for (; b < n; b += nw * 32) {
        issue(b + (D - 1) * nw * 32, (st + D - 1) % D);
        mbar_wait(mbw + 8 * st, phase);
        // lane reads row `lane`
        const uint4 *rp = reinterpret_cast<const uint4 *>(ring + (st * 32 + lane) * R);
#pragma unroll
        for (int q = 0; q < R / 16; ++q) { const uint4 v = rp[q]; acc += v.x ^ v.y ^ v.z ^ v.w; }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        st = st + 1;
        if (st == D) { st = 0; phase ^= 1; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// TMA gather4: lanes 0..7 each gather 4 rows (32 rows per stage per warp)
template <int R, int D>
__global__ void k_g4(const __grid_constant__ CUtensorMap tm, const uint32_t *__restrict__ idx, uint32_t n, uint32_t *out) {
    extern __shared__ __align__(128) unsigned char smb[];
    __shared__ uint64_t mb[32 * D];
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char *ring = smb + (size_t)wl * D * 32 * R;
    const uint32_t mbw = sa(&mb[wl * D]);
    if (lane < D) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbw + 8 * lane) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    auto issue = [&](uint32_t base, int st) {
        const uint32_t i = base + lane;
        const uint32_t r = i < n ? __ldg(idx + i) : 0;
        const uint32_t r0 = __shfl_sync(~0u, r, (lane & 7) * 4), r1 = __shfl_sync(~0u, r, (lane & 7) * 4 + 1),
                       r2 = __shfl_sync(~0u, r, (lane & 7) * 4 + 2), r3 = __shfl_sync(~0u, r, (lane & 7) * 4 + 3);
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbw + 8 * st), "r"(32 * R) : "memory");
        __syncwarp();
        if (lane < 8)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                         ::"r"(sa(ring + (st * 32 + 4 * lane) * R)), "l"(&tm), "r"(mbw + 8 * st),
                         "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
    };
    uint32_t b = warp * 32;
#pragma unroll
    for (int s = 0; s < D - 1; ++s) issue(b + s * nw * 32, s);
    uint32_t phase = 0;
    int st = 0;
    for (; b < n; b += nw * 32) {
        issue(b + (D - 1) * nw * 32, (st + D - 1) % D);
        mbar_wait(mbw + 8 * st, phase);
        const uint4 *rp = reinterpret_cast<const uint4 *>(ring + (st * 32 + lane) * R);
#pragma unroll
        for (int q = 0; q < R / 16; ++q) { const uint4 v = rp[q]; acc += v.x ^ v.y ^ v.z ^ v.w; }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        st = st + 1;
        if (st == D) { st = 0; phase ^= 1; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// correctness probe for gather4: gathers rows {5, 9, 2, 7} of X into dst
__global__ void k_g4_check(const __grid_constant__ CUtensorMap tm, uint32_t *dst, int R) {
    extern __shared__ __align__(128) unsigned char smb[];
    __shared__ uint64_t mb;
    const uint32_t m = sa(&mb);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(4 * R) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                     ::"r"(sa(smb)), "l"(&tm), "r"(m), "r"(0), "r"(5), "r"(9), "r"(2), "r"(7) : "memory");
        mbar_wait(m, 0);
        for (int i = 0; i < R; i += 4) dst[i / 4] = *reinterpret_cast<uint32_t *>(smb + i);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    f();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    const uint32_t n = 1u << 24;
    uint32_t *idx, *out;
    CK(cudaMalloc(&idx, n * 4ull));
    CK(cudaMalloc(&out, 4));
    std::vector<uint32_t> h(n);
    uint64_t s = 88172645463325252ull;
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    const uint64_t xbytes = 64ull << 20;
    unsigned char *X;
    CK(cudaMalloc(&X, xbytes));
    {
        std::vector<uint32_t> hx(xbytes / 4);
        for (size_t i = 0; i < hx.size(); ++i) hx[i] = (uint32_t)i;
        CK(cudaMemcpy(X, hx.data(), xbytes, cudaMemcpyHostToDevice));
    }
    auto run = [&](auto R_) -> int {
        constexpr int R = decltype(R_)::value;
        const uint64_t nrow = xbytes / R;
        for (uint32_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % nrow); }
        CK(cudaMemcpy(idx, h.data(), n * 4ull, cudaMemcpyHostToDevice));
        float ms = timeit([&] { k_ldg<R><<<148 * 8, 256>>>(idx, (const uint4 *)X, n, out); });
        printf("R=%3d ldg   : %7.3f ms %7.1f G rows/s %7.1f GB/s\n", R, ms, n / ms / 1e6, n * (double)R / ms / 1e6);
        {
            constexpr int D = 4, U = 2;
            const int smem = 8 * D * U * 32 * 16;
            cudaFuncSetAttribute(k_lsts<R, D, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            ms = timeit([&] { k_lsts<R, D, U><<<148 * 3, 256, smem>>>(idx, (const uint4 *)X, n, out); });
            printf("R=%3d lsts  : %7.3f ms %7.1f G rows/s %7.1f GB/s (D=%d U=%d)\n", R, ms, n / ms / 1e6, n * (double)R / ms / 1e6, D, U);
        }
        for (int D : {2, 4}) {
            const int smem = 8 * D * 32 * R;
            auto kb = D == 2 ? k_bulk<R, 2> : k_bulk<R, 4>;
            cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int ctas = 148 * std::max(1, std::min(8, 200 * 1024 / smem));
            ms = timeit([&] { kb<<<ctas, 256, smem>>>(idx, X, n, out); });
            printf("R=%3d bulk  : %7.3f ms %7.1f G rows/s %7.1f GB/s (D=%d, %d CTAs)\n", R, ms, n / ms / 1e6, n * (double)R / ms / 1e6, D, ctas);
        }
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)R / 4, nrow}, strides[1] = {(cuuint64_t)R};
        cuuint32_t box[2] = {(cuuint32_t)R / 4, 1}, es[2] = {1, 1};
        CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr) { printf("encode failed %d\n", (int)cr); return 0; }
        uint32_t *dst;
        CK(cudaMalloc(&dst, R));
        k_g4_check<<<1, 32, 4 * R>>>(tm, dst, R);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> hd(R / 4);
        CK(cudaMemcpy(hd.data(), dst, R, cudaMemcpyDeviceToHost));
        printf("g4 check R=%d: first words of rows 5: %u (want %u), 9 @ %d: %u (want %u)\n", R, hd[0], 5u * R / 4,
               R / 16, R >= 16 ? hd[R / 16] : 0, 9u * R / 4);
        cudaFree(dst);
        for (int D : {2, 4}) {
            const int smem = 8 * D * 32 * R;
            auto kg = D == 2 ? k_g4<R, 2> : k_g4<R, 4>;
            cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int ctas = 148 * std::max(1, std::min(8, 200 * 1024 / smem));
            ms = timeit([&] { kg<<<ctas, 256, smem>>>(tm, idx, n, out); });
            printf("R=%3d g4    : %7.3f ms %7.1f G rows/s %7.1f GB/s (D=%d, %d CTAs) %s\n", R, ms, n / ms / 1e6,
                   n * (double)R / ms / 1e6, D, ctas, cudaGetErrorString(cudaGetLastError()));
        }
        return 0;
    };
    run(std::integral_constant<int, 32>{});
    run(std::integral_constant<int, 64>{});
    run(std::integral_constant<int, 128>{});
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}

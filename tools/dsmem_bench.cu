// Microbenchmark: random u16 gathers from a vector spread over the shared
// memory of a thread-block cluster (DSMEM), the access an apply kernel with
// x staged across a cluster would make.  Compares with local smem gathers.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dsmem_bench.cu -o /tmp/dsmem
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r));
    return d;
}
__device__ __forceinline__ uint32_t ld_dsm16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared::cluster.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

// MODE 0: mapa per gather; MODE 1: per-rank base table in smem; MODE 2: local only.
template <int MODE>
__global__ void k_dsm(const uint32_t *__restrict__ idx, uint64_t n, uint32_t wlog, uint32_t clog,
                      uint32_t *out) {
    extern __shared__ __align__(16) uint16_t sx[];
    __shared__ uint32_t base[16];
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t W = 1u << wlog;
    for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) sx[i] = (uint16_t)(i * 3 + 1);
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(sx);
    if (threadIdx.x < 16) base[threadIdx.x] = mapa(local, threadIdx.x & ((1u << clog) - 1));
    cl.sync();
    uint32_t acc = 0;
    const uint32_t mask = (1u << (wlog + clog)) - 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        const uint4 c4 = __ldg(reinterpret_cast<const uint4 *>(idx + i));
        const uint32_t c[4] = {c4.x & mask, c4.y & mask, c4.z & mask, c4.w & mask};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (MODE == 2) {
                acc += sx[c[u] & (W - 1)];
            } else {
                const uint32_t r = c[u] >> wlog, off = (c[u] & (W - 1)) * 2;
                const uint32_t a = MODE == 0 ? mapa(local + off, r) : base[r] + off;
                acc += ld_dsm16(a);
            }
        }
    }
    cl.sync();
    if (acc == 0x12345678) out[0] = acc;
}

template <int MODE>
float run(const uint32_t *idx, uint64_t n, uint32_t wlog, uint32_t clog, uint32_t *out, int blocks_per_sm) {
    cudaLaunchConfig_t cfg = {};
    const uint32_t C = 1u << clog;
    int nsm = 148;
    // grid: as many full clusters as fit (rounded down to a multiple of C)
    cfg.gridDim = dim3((nsm * blocks_per_sm / C) * C);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = (2u << wlog);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k_dsm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_dsm<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k_dsm<MODE>, &cfg);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, k_dsm<MODE>, idx, n, wlog, clog, out);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, k_dsm<MODE>, idx, n, wlog, clog, out);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("mode=%d cluster=%2u W=%6u (%4u KB/cta) grid=%u maxActiveClusters=%d: %7.3f ms %7.1f G gathers/s %s\n",
           MODE, C, 1u << wlog, (2u << wlog) >> 10, cfg.gridDim.x, ncl, ms, n / ms / 1e6,
           e ? cudaGetErrorString(e) : "");
    return ms;
}

int main() {
    const uint64_t n = 1ull << 26;
    uint32_t *idx, *out;
    cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    uint32_t *h = new uint32_t[n];
    uint64_t s = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s; }
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    for (uint32_t clog : {0u, 1u, 2u, 3u, 4u}) {
        run<2>(idx, n, 16, clog, out, 1);
        run<0>(idx, n, 16, clog, out, 1);
        run<1>(idx, n, 16, clog, out, 1);
    }
    // capacity variant: 96 KB per CTA, 2 CTAs / SM
    for (uint32_t clog : {3u, 4u}) run<1>(idx, n, 15, clog, out, 2);
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Microbenchmark 2: random ROW gathers (a group of G lanes reads a contiguous
// row of G*4 bytes at a random row index) -- the access of the block /
// sequence kernels -- and random shared-memory gathers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int G>
__global__ void k_rows(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ X, uint64_t nrows_g, uint32_t* out) {
    uint32_t acc = 0;
    const uint32_t lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t stride = nw * (32 / G);
    uint64_t i = warp * (32 / G) + sub;
    for (; i + 7 * stride < nrows_g; i += 8 * stride) {
        uint32_t r[8], v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __ldg(idx + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(X + (uint64_t)r[u] * G + sl);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; i < nrows_g; i += stride) acc += __ldg(X + (uint64_t)__ldg(idx + i) * G + sl);
    if (acc == 0x12345678) out[0] = acc;
}

__global__ void k_smem(const uint32_t* __restrict__ idx, uint64_t n, uint32_t mask, uint32_t* out) {
    extern __shared__ uint16_t sx[];
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sx[i] = i;
    __syncthreads();
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = __ldg(idx + i) & mask;
        acc += sx[c];
        acc += sx[(c * 7) & mask];
        acc += sx[(c * 13) & mask];
        acc += sx[(c * 29) & mask];
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    const uint64_t nidx = 1ull << 24;
    uint32_t *idx, *X, *out;
    cudaMalloc(&idx, nidx * 4); cudaMalloc(&out, 4);
    uint32_t* h = new uint32_t[nidx];
    uint64_t s = 88172645463325252ull;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint64_t xbytes : {64ull << 20, 128ull << 20, 256ull << 20}) {
        cudaMalloc(&X, xbytes); cudaMemset(X, 1, xbytes);
#define ROWS(G) { uint64_t nrow = xbytes / (G * 4); \
        for (uint64_t i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % nrow); } \
        cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice); \
        for (int it = 0; it < 2; ++it) k_rows<G><<<148*8, 256>>>(idx, X, nidx, out); \
        cudaEventRecord(a); for (int it = 0; it < 5; ++it) k_rows<G><<<148*8, 256>>>(idx, X, nidx, out); cudaEventRecord(b); \
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5; \
        printf("X=%4llu MB row=%3d B: %7.3f ms %7.1f G rows/s %7.1f GB/s useful\n", (unsigned long long)(xbytes>>20), G*4, ms, nidx/ms/1e6, nidx*G*4.0/ms/1e6); }
        ROWS(1) ROWS(2) ROWS(4) ROWS(8) ROWS(16) ROWS(32)
        cudaFree(X);
    }
    for (uint32_t sm_elems : {1u << 15, 1u << 16}) {
        cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int it = 0; it < 2; ++it) k_smem<<<148*2, 1024, sm_elems * 2>>>(idx, nidx, sm_elems - 1, out);
        cudaEventRecord(a); for (int it = 0; it < 5; ++it) k_smem<<<148*2, 1024, sm_elems * 2>>>(idx, nidx, sm_elems - 1, out); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("smem u16 gathers (%u elems): %7.3f ms  %7.1f G gathers/s\n", sm_elems, ms, 4 * nidx / ms / 1e6);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}

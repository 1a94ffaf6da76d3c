// Microbenchmark: shared-memory atomics vs plain stores at random addresses
// (decides the accumulation scheme of the x-panel apply).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const uint32_t* __restrict__ idx, uint64_t n, uint32_t mask, uint32_t* out) {
    extern __shared__ uint32_t s[];
    unsigned long long* s64 = (unsigned long long*)s;
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = __ldg(idx + i);
        uint32_t a = c & mask, b = (c >> 7) & mask, d = (c * 13) & mask, e = (c * 29) & mask;
        if (MODE == 0) { atomicAdd(s + a, 1u); atomicAdd(s + b, 1u); atomicAdd(s + d, 1u); atomicAdd(s + e, 1u); }
        else if (MODE == 1) { atomicAdd(s64 + (a >> 1), 1ull); atomicAdd(s64 + (b >> 1), 1ull); atomicAdd(s64 + (d >> 1), 1ull); atomicAdd(s64 + (e >> 1), 1ull); }
        else if (MODE == 2) { s[a] += 1; s[b] += 1; s[d] += 1; s[e] += 1; }
        else { uint32_t row = (uint32_t)(i >> 1) & mask; atomicAdd(s + row, 1u); atomicAdd(s + ((row + 1) & mask), 1u); atomicAdd(s + ((row+2)&mask), 1u); atomicAdd(s + ((row+3)&mask), 1u);}  // sorted-ish rows
    }
    __syncthreads();
    if (threadIdx.x == 0 && s[0] == 0x12345) out[0] = 1;
}

int main() {
    const uint64_t n = 1ull << 24;
    uint32_t *idx, *out;
    cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    uint32_t* h = new uint32_t[n];
    uint64_t st = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; h[i] = (uint32_t)st; }
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const uint32_t mask = (1u << 14) - 1;   // 16k words = 64 KB
#define RUN(M, NAME) { cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024); \
    for (int it = 0; it < 2; ++it) k<M><<<148, 1024, (mask + 1) * 4>>>(idx, n, mask, out); \
    cudaEventRecord(a); for (int it = 0; it < 5; ++it) k<M><<<148, 1024, (mask + 1) * 4>>>(idx, n, mask, out); cudaEventRecord(b); \
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5; \
    printf("%-34s %7.3f ms  %8.1f G ops/s\n", NAME, ms, 4 * n / ms / 1e6); }
    RUN(0, "smem atomicAdd u32 random")
    RUN(1, "smem atomicAdd u64 random")
    RUN(2, "smem plain RMW u32 random (racy)")
    RUN(3, "smem atomicAdd u32 sorted rows")
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}

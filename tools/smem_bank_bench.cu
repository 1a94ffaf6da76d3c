// Microbenchmark: cost of random vs bank-conflict-free shared-memory gathers
// (ld.shared.u16) and reductions (red.shared.add.u32) -- the two per-entry
// shared operations of the panel apply.  Addresses come from a register LCG
// so no global traffic is involved.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/smem_bank_bench.cu -o /tmp/sbb
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// MODE bit 0: do gathers, bit 1: do reductions, bit 2: conflict-free
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t iters, uint32_t *out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t xs = (uint32_t)__cvta_generic_to_shared(sm);                 // 128 KB x
    const uint32_t as = xs + (128u << 10);                                       // 64 KB acc
    for (uint32_t i = threadIdx.x; i < (192u << 10) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t r = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r = r * 1664525u + 1013904223u;
            uint32_t xw, aw;   // word indices
            if (MODE & 4) {
                xw = ((r >> 8) & 1023u) * 32 + lane;         // bank = lane
                aw = ((r >> 20) & 511u) * 32 + lane;
            } else {
                xw = (r >> 8) & 32767u;
                aw = (r >> 18) & 16383u;
            }
            uint32_t v = 1;
            if (MODE & 1) {
                unsigned short h;
                asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(xs + 4 * xw));
                v = h;
            }
            if (MODE & 2) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(as + 4 * aw), "r"(v));
            else acc += v;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
void run(const char *name) {
    uint32_t *out;
    cudaMalloc(&out, 4);
    const size_t smem = 192u << 10;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t iters = 4096;
    k<MODE><<<148, 1024, smem>>>(iters, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<148, 1024, smem>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_ops = 148.0 * 32 * iters * 8;   // per op kind
    const double cyc = ms * 1e-3 * 1.965e9;            // SM cycles (nominal max clock)
    printf("%-40s %8.3f ms  %6.2f cycles per warp-op per SM  (%.0f G lane-ops/s)\n", name, ms,
           cyc / (warp_ops / 148.0), warp_ops * 32 / (ms * 1e6));
    cudaFree(out);
}

int main() {
    run<1>("gather u16, random");
    run<5>("gather u16, conflict-free");
    run<2>("red.add u32, random");
    run<6>("red.add u32, conflict-free");
    run<3>("gather + red.add, random");
    run<7>("gather + red.add, conflict-free");
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

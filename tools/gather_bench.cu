// Microbenchmark: random 4-byte gather throughput on B200 through the
// different load paths (decides the x-gather design of the apply kernel).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, class T>
__global__ void k_gather(const uint32_t* __restrict__ idx, const T* __restrict__ x, uint64_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c;
        asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(c) : "l"(idx + i));
        uint32_t v;
        const T* p = x + c;
        if (MODE == 0) v = __ldg(p);
        else if (MODE == 1) { if (sizeof(T)==4) asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(p)); else { unsigned short h; asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(h) : "l"(p)); v = h; } }
        else if (MODE == 2) { if (sizeof(T)==4) asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p)); else { unsigned short h; asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(h) : "l"(p)); v = h; } }
        else { v = *(volatile const T*)p; }
        acc += v;
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    const uint64_t n = 1ull << 24;        // 16M gathers
    uint32_t* idx; uint32_t* x; uint16_t* x16; uint32_t* out;
    cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    uint32_t* h = new uint32_t[n];
    uint64_t s = 88172645463325252ull;
    for (int pass = 0; pass < 4; ++pass) {
        uint64_t xs = pass == 0 ? (1u<<20) : pass == 1 ? (1u<<22) : pass == 2 ? (1u<<16) : (1u<<26);
        cudaMalloc(&x, xs * 4); cudaMalloc(&x16, xs * 2);
        cudaMemset(x, 1, xs * 4); cudaMemset(x16, 1, xs * 2);
        for (uint64_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % xs); }
        cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        auto run = [&](auto kern, const char* name) {
            for (int occ : {1, 2}) {
            int blocks = 148 * 8 * occ;
            kern<<<blocks, 256>>>(idx, (decltype(x)) nullptr == nullptr ? nullptr : nullptr, 0, out);
            };
        };
        (void)run;
#define RUN(MODE, T, XP, NAME) { \
        for (int it = 0; it < 2; ++it) k_gather<MODE, T><<<148*8, 256>>>(idx, XP, n, out); \
        cudaEventRecord(a); for (int it = 0; it < 10; ++it) k_gather<MODE, T><<<148*8, 256>>>(idx, XP, n, out); cudaEventRecord(b); \
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10; \
        printf("x=%8llu elems %-5s %-22s %7.3f ms  %6.1f G gathers/s  idx-stream %5.0f GB/s\n", (unsigned long long)xs, sizeof(T)==4?"u32":"u16", NAME, ms, n / ms / 1e6, n*4 / ms / 1e6); }
        RUN(0, uint32_t, x, "ldg(.nc)");
        RUN(1, uint32_t, x, "ld.cg");
        RUN(2, uint32_t, x, "ld.nc.L1::no_allocate");
        RUN(3, uint32_t, x, "ld (volatile .ca)");
        RUN(0, uint16_t, x16, "ldg(.nc)");
        RUN(2, uint16_t, x16, "ld.nc.L1::no_allocate");
        cudaFree(x); cudaFree(x16);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

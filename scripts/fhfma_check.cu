// Checks that fma.rn.f32.bf16 (SASS FHFMA.BF16) equals fmaf on the bf16 values widened
// to fp32 — the identity the pruning dot relies on. Dev tool.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t h32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
__global__ void k(unsigned long long* bad, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float acc1 = 0.f, acc2 = 0.f;
    uint32_t s = i * 2654435761u;
    for (int j = 0; j < n; ++j) {
        s = h32(s + j);
        uint16_t a = (uint16_t)(s & 0xffff), b = (uint16_t)(s >> 16);
        // keep exponents moderate-to-wide (include subnormal-product ranges sometimes)
        if ((j & 7) != 0) { a = (a & 0x807f) | (((a >> 7) & 0x1f) + 112) << 7; b = (b & 0x807f) | (((b >> 7) & 0x1f) + 112) << 7; }
        float d;
        asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(acc1));
        const float fa = __uint_as_float((uint32_t)a << 16), fb = __uint_as_float((uint32_t)b << 16);
        const float e = __fmaf_rn(fa, fb, acc2);
        if (!((d == e) || (d != d && e != e))) { atomicAdd(bad, 1ull); }
        acc1 = d; acc2 = e;
        if (!(fabsf(acc1) < 1e30f)) { acc1 = 0.f; acc2 = 0.f; }
    }
}
int main() {
    unsigned long long* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
    k<<<4096, 256>>>(bad, 1024);
    unsigned long long h = 0; cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("fhfma vs fmaf mismatches: %llu of %llu (%s)\n", h, 4096ull * 256 * 1024, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

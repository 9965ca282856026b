// Throughput of FHFMA.BF16 (fma.rn.f32.bf16) vs FFMA (+ bf16 unpack) on sm_100a. Dev tool.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float fh(uint32_t a, uint32_t b, float c, bool hi) {
    float d; const uint16_t ah = hi ? a >> 16 : a & 0xffff, bh = hi ? b >> 16 : b & 0xffff;
    asm volatile("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(ah), "h"(bh), "f"(c)); return d;
}
template <int MODE>
__global__ void k(const uint32_t* in, float* out, int iters) {
    uint32_t a[8], b[8]; float acc[8];
    for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 8 + i]; acc[i] = 0.f; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) { acc[i] = fh(a[i], b[i], acc[i], false); acc[i] = fh(a[i], b[i], acc[i], true); }
            else { acc[i] = __fmaf_rn(__uint_as_float(a[i] << 16), __uint_as_float(b[i] << 16), acc[i]);
                   acc[i] = __fmaf_rn(__uint_as_float(a[i] & 0xffff0000u), __uint_as_float(b[i] & 0xffff0000u), acc[i]); }
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t* in; float* out; cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 8 * 1024 * 4); cudaMemset(in, 0x3f, 4096);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(in, out, 1000); else k<1><<<148 * 8, 256>>>(in, out, 1000);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double fmas = 148.0 * 8 * 256 * 1000 * 16;
            if (rep) printf("%s: %.3f ms, %.1f fma/clk/SM at 1.965 GHz\n", mode ? "FFMA+unpack" : "FHFMA.BF16", ms,
                            fmas / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    return 0;
}

// Dev probe (sm_100a): (1) accuracy of mma.sync m16n8k16 bf16 -> fp32 dots of length 128
// (8 chained k-steps) against the exact (fp64) dot and the reference's sequential fp32
// dot, relative to sum |q_i k_i|; (2) mma.sync issue throughput per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_check scripts/mma_check.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// keys K [16][128] (A, row-major), q Q [8][128] (B, "col": n-major rows of k) -> D[16][8]
__global__ void dots(const __nv_bfloat16* K, const __nv_bfloat16* Q, float* D, int n_tiles) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    for (int tile = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; tile < n_tiles; tile += gridDim.x * (blockDim.x / 32)) {
        const __nv_bfloat16* k = K + static_cast<size_t>(tile) * 16 * 128;
        const __nv_bfloat16* q = Q + static_cast<size_t>(tile) * 8 * 128;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        for (int ks = 0; ks < 8; ++ks) {
            uint32_t a[4], b[2];
            auto w = [](const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); };
            a[0] = w(k + g * 128 + ks * 16 + 2 * tq);
            a[1] = w(k + (g + 8) * 128 + ks * 16 + 2 * tq);
            a[2] = w(k + g * 128 + ks * 16 + 2 * tq + 8);
            a[3] = w(k + (g + 8) * 128 + ks * 16 + 2 * tq + 8);
            b[0] = w(q + g * 128 + ks * 16 + 2 * tq);
            b[1] = w(q + g * 128 + ks * 16 + 2 * tq + 8);
            mma16816(c, a, b);
        }
        float* d = D + static_cast<size_t>(tile) * 128;
        d[g * 8 + 2 * tq] = c[0];
        d[g * 8 + 2 * tq + 1] = c[1];
        d[(g + 8) * 8 + 2 * tq] = c[2];
        d[(g + 8) * 8 + 2 * tq + 1] = c[3];
    }
}

__global__ void tput(float* out, int iters) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b[2] = {11u, threadIdx.x};
    float c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mma16816(c[u], a, b);
    }
    float s = 0.f;
    for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
    const int n_tiles = 1 << 14;
    const size_t nk = static_cast<size_t>(n_tiles) * 16 * 128, nq = static_cast<size_t>(n_tiles) * 8 * 128;
    __nv_bfloat16* hk = (__nv_bfloat16*)malloc(nk * 2);
    __nv_bfloat16* hq = (__nv_bfloat16*)malloc(nq * 2);
    float* hkf = (float*)malloc(nk * 4);
    float* hqf = (float*)malloc(nq * 4);
    srand(7);
    auto gauss = []() { float s = 0; for (int i = 0; i < 12; ++i) s += rand() / (float)RAND_MAX; return s - 6.0f; };
    for (int t = 0; t < n_tiles; ++t) {
        const int mode = t % 4;  // 0 random, 1 wide dynamic range, 2 cancellation (k ~ +-q), 3 large
        for (int r = 0; r < 8; ++r)
            for (int e = 0; e < 128; ++e) {
                float x = gauss();
                if (mode == 1) x *= powf(2.0f, (float)(rand() % 17 - 8));
                if (mode == 3) x *= 1000.0f;
                hqf[(static_cast<size_t>(t) * 8 + r) * 128 + e] = bf(x);
            }
        for (int r = 0; r < 16; ++r)
            for (int e = 0; e < 128; ++e) {
                float x = gauss();
                if (mode == 1) x *= powf(2.0f, (float)(rand() % 17 - 8));
                if (mode == 2) {  // alternating-sign copy of q row 0: huge cancellation
                    x = hqf[(static_cast<size_t>(t) * 8) * 128 + e] * ((e & 1) ? 1.0f : -1.0f) * (1.0f + 0.01f * gauss());
                }
                hkf[(static_cast<size_t>(t) * 16 + r) * 128 + e] = bf(x);
            }
    }
    for (size_t i = 0; i < nk; ++i) hk[i] = __float2bfloat16(hkf[i]);
    for (size_t i = 0; i < nq; ++i) hq[i] = __float2bfloat16(hqf[i]);
    __nv_bfloat16 *dk, *dq; float* dd;
    cudaMalloc(&dk, nk * 2); cudaMalloc(&dq, nq * 2); cudaMalloc(&dd, static_cast<size_t>(n_tiles) * 128 * 4);
    cudaMemcpy(dk, hk, nk * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, hq, nq * 2, cudaMemcpyHostToDevice);
    dots<<<592, 256>>>(dk, dq, dd, n_tiles);
    float* hd = (float*)malloc(static_cast<size_t>(n_tiles) * 128 * 4);
    cudaMemcpy(hd, dd, static_cast<size_t>(n_tiles) * 128 * 4, cudaMemcpyDeviceToHost);
    double worst_exact[4] = {0, 0, 0, 0}, worst_seq[4] = {0, 0, 0, 0}, worst_cs[4] = {0, 0, 0, 0};
    for (int t = 0; t < n_tiles; ++t)
        for (int r = 0; r < 16; ++r)
            for (int n = 0; n < 8; ++n) {
                const float* k = hkf + (static_cast<size_t>(t) * 16 + r) * 128;
                const float* q = hqf + (static_cast<size_t>(t) * 8 + n) * 128;
                double ex = 0, ab = 0, nk2 = 0, nq2 = 0;
                float seq = 0.f;
                for (int e = 0; e < 128; ++e) {
                    ex += (double)q[e] * k[e];
                    ab += fabs((double)q[e] * k[e]);
                    nk2 += (double)k[e] * k[e];
                    nq2 += (double)q[e] * q[e];
                    seq = seq + q[e] * k[e];  // products exact (bf16 x bf16), sums rounded
                }
                const double tc = hd[static_cast<size_t>(t) * 128 + r * 8 + n];
                const int mode = t % 4;
                if (ab > 0) {
                    worst_exact[mode] = fmax(worst_exact[mode], fabs(tc - ex) / ab);
                    worst_seq[mode] = fmax(worst_seq[mode], fabs(tc - seq) / ab);
                    worst_cs[mode] = fmax(worst_cs[mode], fabs(tc - seq) / sqrt(nk2 * nq2));
                }
            }
    for (int m = 0; m < 4; ++m)
        printf("mode %d: max |tc-exact|/sum|qk| = %.3e (2^%.1f)  max |tc-seq|/sum|qk| = %.3e (2^%.1f)  /(|q||k|) = %.3e (2^%.1f)\n", m,
               worst_exact[m], log2(worst_exact[m]), worst_seq[m], log2(worst_seq[m]), worst_cs[m], log2(worst_cs[m]));
    // throughput: 4 independent accumulators per warp
    float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    for (int warps : {4, 8, 16, 32}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int iters = 4096;
        tput<<<148, warps * 32>>>(o, 16);
        cudaEventRecord(a);
        tput<<<148, warps * 32>>>(o, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double macs = 148.0 * warps * iters * 4 * 2048.0;
        printf("warps/SM %2d: %.1f TFLOP/s dense bf16 via mma.sync (%.0f MAC/clk/SM at 1.9 GHz)\n", warps,
               2 * macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / 148 / 1.9e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

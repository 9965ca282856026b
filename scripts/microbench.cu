// Calibration microbenchmarks for single-CTA latency-bound phases (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_chase(const int* next, int n_steps, unsigned long long* out) {
    int p = threadIdx.x;
    unsigned long long c0 = clock64(), t0 = gt();
    for (int i = 0; i < n_steps; ++i) p = __ldcg(next + p);
    unsigned long long c1 = clock64(), t1 = gt();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = t1 - t0; out[2] = p; }
}

template <int B>
__global__ void k_batched(const float* buf, int rounds, int stride, unsigned long long* out, float* sink) {
    float acc = 0.f;
    unsigned long long c0 = clock64(), t0 = gt();
    for (int r = 0; r < rounds; ++r) {
        float v[B];
#pragma unroll
        for (int k = 0; k < B; ++k) v[k] = __ldcg(buf + (r * B + k) * stride + threadIdx.x);
#pragma unroll
        for (int k = 0; k < B; ++k) acc += v[k];
        // make next round depend on this one (like a reduction loop would not) - no
    }
    unsigned long long c1 = clock64(), t1 = gt();
    sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = t1 - t0; }
}

__global__ void k_hist(const unsigned* keys, int n, int passes, unsigned long long* out, int* sink) {
    __shared__ int hist[256];
    unsigned long long c0 = clock64(), t0 = gt();
    for (int p = 0; p < passes; ++p) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int j = threadIdx.x; j < n; j += blockDim.x) atomicAdd(&hist[(keys[j] >> (p * 3)) & 255], 1);
        __syncthreads();
    }
    unsigned long long c1 = clock64(), t1 = gt();
    if (threadIdx.x < 256) sink[threadIdx.x] = hist[threadIdx.x];
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = t1 - t0; }
}

__global__ void k_sync(int n, unsigned long long* out) {
    unsigned long long c0 = clock64(), t0 = gt();
    for (int i = 0; i < n; ++i) __syncthreads();
    unsigned long long c1 = clock64(), t1 = gt();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = t1 - t0; }
}

__global__ void k_timer(unsigned long long* out) {
    unsigned long long prev = gt(), first = prev;
    int changes = 0;
    unsigned long long mind = ~0ull;
    unsigned long long c0 = clock64();
    while (changes < 64) {
        unsigned long long t = gt();
        if (t != prev) { mind = min(mind, t - prev); prev = t; ++changes; }
    }
    unsigned long long c1 = clock64();
    out[0] = mind; out[1] = prev - first; out[2] = c1 - c0;
}

int main() {
    unsigned long long* d_out;
    cudaMalloc(&d_out, 64);
    unsigned long long h[4];
    // timer resolution + clock rate
    k_timer<<<1, 1>>>(d_out);
    cudaMemcpy(h, d_out, 24, cudaMemcpyDeviceToHost);
    printf("globaltimer: min step %llu ns, 64 steps = %llu ns, clock cycles %llu -> %.3f GHz\n", h[0], h[1], h[2], (double)h[2] / h[1]);
    // pointer chase, buffer 1 MB (L2), 256 threads
    const int n = 1 << 18;
    std::vector<int> nx(n);
    for (int i = 0; i < n; ++i) nx[i] = (int)(((long long)i * 7919 + 4099) % n);
    int* d_next;
    cudaMalloc(&d_next, n * 4);
    cudaMemcpy(d_next, nx.data(), n * 4, cudaMemcpyHostToDevice);
    k_chase<<<1, 256>>>(d_next, 64, d_out);  // warm L2
    k_chase<<<1, 256>>>(d_next, 256, d_out);
    cudaMemcpy(h, d_out, 24, cudaMemcpyDeviceToHost);
    printf("L2 pointer chase: %.1f cycles/load, %.1f ns/load\n", h[0] / 256.0, h[1] / 256.0);
    // batched loads
    float* d_buf; float* d_sink;
    cudaMalloc(&d_buf, 64 << 20); cudaMalloc(&d_sink, 4096 * 4);
    cudaMemset(d_buf, 0, 64 << 20);
    for (int rep = 0; rep < 2; ++rep) {
        k_batched<16><<<1, 256>>>(d_buf, 8, 256, d_out, d_sink);
        cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
        printf("batched 16 x 8 rounds (256 thr): %llu cycles, %llu ns -> %.0f ns/round\n", h[0], h[1], h[1] / 8.0);
        k_batched<1><<<1, 256>>>(d_buf, 128, 256, d_out, d_sink);
        cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
        printf("unbatched 128 loads (256 thr): %llu cycles, %llu ns -> %.0f ns/load\n", h[0], h[1], h[1] / 128.0);
    }
    // smem histogram
    unsigned* d_keys; int* d_isink;
    std::vector<unsigned> keys(4096);
    for (int i = 0; i < 4096; ++i) keys[i] = (unsigned)(i * 2654435761u);
    cudaMalloc(&d_keys, 4096 * 4); cudaMalloc(&d_isink, 256 * 4);
    cudaMemcpy(d_keys, keys.data(), 4096 * 4, cudaMemcpyHostToDevice);
    k_hist<<<1, 128>>>(d_keys, 1024, 4, d_out, d_isink);
    k_hist<<<1, 128>>>(d_keys, 1024, 4, d_out, d_isink);
    cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("smem hist 1024 keys x 4 passes (128 thr): %llu cycles, %llu ns\n", h[0], h[1]);
    k_sync<<<1, 128>>>(1000, d_out);
    cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("__syncthreads x1000 (128 thr): %.1f cycles each, %.1f ns each\n", h[0] / 1000.0, h[1] / 1000.0);
    k_sync<<<1, 512>>>(1000, d_out);
    cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("__syncthreads x1000 (512 thr): %.1f cycles each, %.1f ns each\n", h[0] / 1000.0, h[1] / 1000.0);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

// Achievable HBM bandwidth for random 256 B row gathers (the pruning-stage access
// pattern) vs streaming reads, on this B200. Dev tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_bw scripts/gather_bw.cu && /tmp/gather_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// A: warp gathers 32 random rows per step with 16 B cp.async (2 rows per instruction)
__global__ void __launch_bounds__(128) gA(const char* buf, uint32_t nrows, int steps, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* ks = sm + w * 32 * 256;
    float acc = 0.f;
    uint32_t seed = (blockIdx.x * 4 + w) * 32 + lane;
    for (int s = 0; s < steps; ++s) {
        uint32_t row = hash32(seed * 131 + s * 7919) % nrows;
        unsigned long long p = (unsigned long long)(buf + (size_t)row * 256);
        const int c = lane & 15, sub = lane >> 4;
        for (int r = 0; r < 32; r += 2) {
            unsigned long long pp = __shfl_sync(0xffffffffu, p, r + sub);
            cp16(ks + (r + sub) * 256 + ((c ^ ((r + sub) & 15)) << 4), (const char*)pp + (c << 4));
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
        const uint4 v = *reinterpret_cast<const uint4*>(ks + lane * 256 + ((3 ^ (lane & 15)) << 4));
        acc += __uint_as_float(v.x & 0x3fffffff) * 1e-30f;
        seed += (uint32_t)(acc > 1e30f);
        __syncwarp();
    }
    if (acc == 12345.f) sink[0] = acc;
}

// B: each lane issues one 256 B bulk copy per step (mbarrier per warp)
__global__ void __launch_bounds__(128) gB(const char* buf, uint32_t nrows, int steps, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* ks = sm + w * 32 * 272;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar[w])), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    float acc = 0.f;
    uint32_t seed = (blockIdx.x * 4 + w) * 32 + lane;
    for (int s = 0; s < steps; ++s) {
        uint32_t row = hash32(seed * 131 + s * 7919) % nrows;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[w])), "r"(32 * 256) : "memory");
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(su(ks + lane * 272)), "l"(buf + (size_t)row * 256), "r"(su(&bar[w])) : "memory");
        asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su(&bar[w])), "r"(s & 1) : "memory");
        const uint4 v = *reinterpret_cast<const uint4*>(ks + lane * 272 + 48);
        acc += __uint_as_float(v.x & 0x3fffffff) * 1e-30f;
        seed += (uint32_t)(acc > 1e30f);
        __syncwarp();
    }
    if (acc == 12345.f) sink[0] = acc;
}

// D: the stage-1 descent pattern in the paged layout ([page][8 kv][64 tokens][256 B],
// chunks of 256 tokens = 4 pages): lane = chunk, warp item = (chunk group, kv head), step
// s visits token c*256 + a binary-search offset (the same for every chunk at the first
// steps, then split by per-(chunk, head) random branch bits). skew: extra bytes per page
// of pool stride (0 = the dense layout).
__global__ void __launch_bounds__(128) gD(const char* buf, uint32_t n_chunks, int steps, uint32_t skew, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* ks = sm + w * 32 * 256;
    float acc = 0.f;
    const uint32_t item = blockIdx.x * 4 + w;
    const uint32_t kvh = item & 7, grp = item >> 3;
    const uint32_t c = (grp * 32 + lane) % n_chunks;
    const uint32_t bits = hash32(c * 8 + kvh + 12345);
    const size_t page_stride = 8ull * 64 * 256 + skew;
    uint32_t first = 0, half = 128;
    for (int s = 0; s < steps; ++s) {
        const uint32_t t = c * 256 + (s == 0 ? 0 : first + half);
        if (s > 0) { if ((bits >> s) & 1) first += half; half >>= 1; if (half == 0) half = 1; }
        const size_t off = (size_t)(t >> 6) * page_stride + ((size_t)kvh * 64 + (t & 63)) * 256;
        unsigned long long p = (unsigned long long)(buf + off);
        const int cc = lane & 15, sub = lane >> 4;
        for (int r = 0; r < 32; r += 2) {
            unsigned long long pp = __shfl_sync(0xffffffffu, p, r + sub);
            cp16(ks + (r + sub) * 256 + ((cc ^ ((r + sub) & 15)) << 4), (const char*)pp + (cc << 4));
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
        const uint4 v = *reinterpret_cast<const uint4*>(ks + lane * 256 + ((3 ^ (lane & 15)) << 4));
        acc += __uint_as_float(v.x & 0x3fffffff) * 1e-30f;
        __syncwarp();
    }
    if (acc == 12345.f) sink[0] = acc;
}

// C: streaming read (coalesced 16 B per lane)
__global__ void gC(const uint4* buf, size_t n, float* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(buf + i); acc ^= v.x ^ v.w;
    }
    if (acc == 0x12345) sink[0] = acc;
}

int main() {
    const size_t bytes = 2ull << 30;
    char* buf; float* sink;
    cudaMalloc(&buf, bytes); cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    const uint32_t nrows = bytes / 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int steps = 9;
    cudaFuncSetAttribute(gA, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 256);
    cudaFuncSetAttribute(gB, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 272);
    for (int ctas_per_sm = 2; ctas_per_sm <= 8; ++ctas_per_sm) {
        for (int v = 0; v < 2; ++v) {
            int grid = 148 * ctas_per_sm;
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (v == 0) gA<<<grid, 128, 4 * 32 * 256>>>(buf, nrows, steps, sink);
                else gB<<<grid, 128, 4 * 32 * 272>>>(buf, nrows, steps, sink);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            double moved = (double)grid * 128 * steps * 256;
            printf("%s ctas/sm %d: %.1f us, %.0f GB/s (%.1f MB)  err=%s\n", v ? "bulk " : "cpasync", ctas_per_sm, best * 1e3,
                   moved / (best * 1e-3) / 1e9, moved / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // unloaded step latency: one CTA (4 warps), 64 dependent gather steps
    for (int v = 0; v < 2; ++v) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (v == 0) gA<<<1, 128, 4 * 32 * 256>>>(buf, nrows, 64, sink);
            else gB<<<1, 128, 4 * 32 * 272>>>(buf, nrows, 64, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%s unloaded: %.0f ns per gather step\n", v ? "bulk " : "cpasync", best * 1e6 / 64);
    }
    // descent pattern: 4,096 chunks (1M tokens) x 8 kv heads = 1,024 warps of 32 chunks x 8 heads... one wave
    cudaFuncSetAttribute(gD, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 256);
    for (uint32_t skew : {0u, 256u, 512u, 1024u, 4096u}) {
        const uint32_t n_chunks = 3700;  // ~0.95M tokens: 14,800 pages x (128 KB + skew) < 2 GB
        const int grid = n_chunks / 32 * 8 / 4;  // 1,024 warps of (32 chunks, 1 head) per kv head pass
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            for (int k = 0; k < 4; ++k) gD<<<grid, 128, 4 * 32 * 256>>>(buf, n_chunks, 9, skew, sink);  // 4 q-heads per kv head
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        double moved = 4.0 * grid * 128 * 9 * 256;
        printf("descent pattern skew %4u B/page: %.1f us, %.0f GB/s  err=%s\n", skew, best * 1e3, moved / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        gC<<<148 * 8, 256>>>((const uint4*)buf, bytes / 16, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("stream read 2 GB: %.1f us, %.0f GB/s\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    }
    return 0;
}

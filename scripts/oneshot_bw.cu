// One-shot gather: 148 CTAs x 256 threads, each warp gathers R random 256 B rows
// into shared memory (cp.async, 2 rows per instruction), once. Dev tool.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t h32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(256) g1(const char* buf, uint32_t nrows, int R, float* sink, uint32_t salt) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = lane & 15, sub = lane >> 4;
    unsigned char* dst = sm + w * R * 256;
    if (MODE == 0) {  // pointer per instruction from a hash (no dependent smem load)
        for (int r0 = 0; r0 < R; r0 += 2) {
            const int r = r0 + sub;
            const uint32_t row = h32(salt + (blockIdx.x * 8 + w) * 4096 + r) % nrows;
            cp16(dst + r * 256 + c * 16, buf + (size_t)row * 256 + c * 16);
        }
    } else {  // all lanes compute their row pointer first, then shuffle-broadcast
        uint64_t p = 0;
        if (lane < R) p = (uint64_t)(buf + (size_t)(h32(salt + (blockIdx.x * 8 + w) * 4096 + lane) % nrows) * 256);
        for (int r0 = 0; r0 < R; r0 += 2) {
            const int r = r0 + sub;
            const uint64_t pp = __shfl_sync(0xffffffffu, p, r & 31);
            cp16(dst + r * 256 + c * 16, (const char*)pp + c * 16);
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (sm[threadIdx.x * 4] == 123 && sm[threadIdx.x * 4 + 1] == 45) sink[0] = 1.f;
}
int main() {
    const size_t bytes = 2ull << 30;
    char* buf; float* sink;
    cudaMalloc(&buf, bytes); cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    char* fl; cudaMalloc(&fl, 512 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode)
    for (int R : {8, 16, 24, 32}) {
        size_t smem = 8 * R * 256;
        if (mode == 0) cudaFuncSetAttribute(g1<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        else cudaFuncSetAttribute(g1<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int rep = 0; rep < 7; ++rep) {
            if (getenv("NOFLUSH") == nullptr) cudaMemset(fl, rep, 512 << 20);
            else if (mode == 0) g1<0><<<148, 256, smem>>>(buf, bytes / 256, R, sink, rep * 7777 + 1);  // warm TLB, other rows
            else g1<1><<<148, 256, smem>>>(buf, bytes / 256, R, sink, rep * 7777 + 1);
            cudaEventRecord(a);
            if (mode == 0) g1<0><<<148, 256, smem>>>(buf, bytes / 256, R, sink, rep * 7777);
            else g1<1><<<148, 256, smem>>>(buf, bytes / 256, R, sink, rep * 7777);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        double moved = 148.0 * 8 * R * 256;
        printf("mode %d R=%2d rows/warp: %.2f us for %.1f MB -> %.0f GB/s (%s)\n", mode, R, best * 1e3, moved / 1e6,
               moved / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

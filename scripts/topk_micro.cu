// Dev microbenchmark: cycles per CTA-wide exact top-K (1024 / 4096 keys, 512 threads).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "topk.cuh"
using namespace hpk;

__device__ inline void cta_topk_prof(const uint32_t* keys, int cc, int K, int32_t* sel, TopkShared& sh,
                                     long long* st) {
    int ns = 0;
#define STAMP() do { __syncwarp(); if (threadIdx.x == 0) st[ns] = clock64(); ++ns; } while (0)
    STAMP();
    const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = warp_id(), nw = nt >> 5;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int j = t; j < cc; j += nt) {
        const uint32_t u = keys[j];
        kmin = min(kmin, u);
        kmax = max(kmax, u);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) { sh.wmin[w] = kmin; sh.wmax[w] = kmax; }
    for (int i = t; i < 256; i += nt) sh.hist[0][i] = 0;
    __syncthreads();
    kmin = __reduce_min_sync(0xffffffffu, lane < nw ? sh.wmin[lane] : 0xffffffffu);
    kmax = __reduce_max_sync(0xffffffffu, lane < nw ? sh.wmax[lane] : 0u);
    STAMP();
    const uint32_t range = kmax - kmin;
    const int hb = range ? 31 - __clz(range) : 0;  // highest differing bit
    int width = min(8, hb + 1);
    int shift = hb + 1 - width;                    // current digit = bits [shift, shift + width)
    uint32_t prefix = 0;                           // the target's bits above the current digit
    int need = K;
    for (int pass = 0;; ++pass) {
        int* hist = sh.hist[pass % 3];
        int* next = sh.hist[(pass + 1) % 3];  // last read two passes ago: free to clear
        for (int i = t; i < 256; i += nt) next[i] = 0;
        const int hi = shift + width;
        for (int j = t; j < cc; j += nt) {
            const uint32_t v = keys[j] - kmin;
            const uint32_t above_bits = hi >= 32 ? 0u : (v >> hi);
            if (above_bits == prefix) atomicAdd(&hist[(v >> shift) & ((1u << width) - 1u)], 1);
        }
        __syncthreads();
        STAMP();
        if (w == 0) {  // the bin holding the need-th largest: suffix sums over 8 bins per lane
            const int4 c0 = *reinterpret_cast<const int4*>(hist + lane * 8);
            const int4 c1 = *reinterpret_cast<const int4*>(hist + lane * 8 + 4);
            const int c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            int tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) tot += c[k];
            int suf = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += y;
            }
            int above = suf - tot;
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                if (above < need && need <= above + c[k]) { sh.digit = lane * 8 + k; sh.above = above; }
                above += c[k];
            }
        }
        __syncthreads();
        const int digit = sh.digit, above_d = sh.above;
        prefix = (prefix << width) | static_cast<uint32_t>(digit);
        need -= above_d;
        STAMP();
        if (shift == 0) break;
        width = min(8, shift);
        shift -= width;
    }
    const uint32_t kth = prefix + kmin;  // the K-th largest key; keep `need` of its copies
    const int per = (cc + nt - 1) / nt;
    const int j0 = min(cc, t * per), j1 = min(cc, j0 + per);
    int ties = 0, gts = 0;
    for (int j = j0; j < j1; ++j) {
        const uint32_t u = keys[j];
        ties += u == kth;
        gts += u > kth;
    }
    // one exclusive scan of (ties << 16 | gts): both counts are <= cc <= 16384
    const int packed = (ties << 16) | gts;
    int x = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    STAMP();
    if (lane == 31) sh.scan[w] = x;
    __syncthreads();
    STAMP();
    int wt = lane < nw ? sh.scan[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wt, o);
        if (lane >= o) wt += y;
    }
    const int wbase = __shfl_sync(0xffffffffu, wt, (w + 31) & 31);
    const int excl = (w ? wbase : 0) + x - packed;
    const int tie_base = excl >> 16;
    int r = (excl & 0xffff) + min(tie_base, need);  // kept before this run: greater + earlier ties
    int trank = tie_base;
    for (int j = j0; j < j1; ++j) {
        const uint32_t u = keys[j];
        bool keep = u > kth;
        if (u == kth) { keep = trank < need; ++trank; }
        if (keep) sel[r++] = j;
    }
    __syncthreads();
    STAMP();
}

__global__ void prof(const float* scores, int cc, int K, long long* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(sm);
    int32_t* sel = reinterpret_cast<int32_t*>(keys + 16384);
    __shared__ TopkShared sh;
    __shared__ long long st[64];
    for (int j = threadIdx.x; j < cc; j += blockDim.x) keys[j] = order_key(scores[j]);
    __syncthreads();
    for (int r = 0; r < 3; ++r) cta_topk_prof(keys, cc, K, sel, sh, st);
    if (threadIdx.x < 32) out[threadIdx.x] = st[threadIdx.x] - st[0];
}

__global__ void bench(const float* scores, int cc, int K, int reps, long long* out, int variant) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(sm);
    int32_t* sel = reinterpret_cast<int32_t*>(keys + 16384);
    int* whist = sel + 4096;
    __shared__ TopkShared sh;
        for (int j = threadIdx.x; j < cc; j += blockDim.x) keys[j] = order_key(scores[j]);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (variant == 0) cta_topk_smem(keys, cc, K, sel, sh);
        else __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = sel[0]; out[2] = sel[K - 1]; }
    // exactness: the fast variant's kept set equals the radix select's
    if (variant == 1) {
        int32_t* sel2 = sel + 2048;
        cta_topk_smem(keys, cc, K, sel2, sh);
        int bad = 0;
        for (int i = threadIdx.x; i < K; i += blockDim.x) bad |= sel[i] != sel2[i];
        bad = __syncthreads_or(bad);
        if (threadIdx.x == 0) out[3] = bad;
    }
}

int main() {
    const int n = 4096;
    float* h = (float*)malloc(n * 4);
    srand(1);
    for (int i = 0; i < n; ++i) {  // approx normal scores
        float s = 0; for (int k = 0; k < 12; ++k) s += rand() / (float)RAND_MAX; h[i] = (s - 6.0f) * 3.0f;
    }
    float* d; long long* o; cudaMalloc(&d, n * 4); cudaMalloc(&o, 64);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    size_t smem = 16384 * 4 + 4096 * 4 + 2 * 32 * 256 * 4;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int cfg[][2] = {{1024, 256}, {4091, 128}, {1024, 256}};
    int ci = 0;
    for (auto& c : cfg) {
        if (ci++ == 2) {  // heavy ties: few distinct values
            for (int i = 0; i < n; ++i) h[i] = (float)(rand() % 5);
            cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
        }
        for (int threads : {512, 1024})
            for (int v = 0; v < 3; ++v) {
                bench<<<1, threads, smem>>>(d, c[0], c[1], 20, o, v);
                long long r[4] = {0, 0, 0, 0}; cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
                printf("cc=%d K=%d threads=%d variant=%d: %lld cycles/call (sel %lld..%lld) mismatch=%lld %s\n", c[0], c[1], threads, v, r[0], r[1], r[2], r[3],
                       cudaGetErrorString(cudaGetLastError()));
                cudaMemset(o, 0, 64);
            }
    }
    {
        long long* po; cudaMalloc(&po, 64 * 8); cudaMemset(po, 0, 512);
        srand(1);
        for (int i = 0; i < n; ++i) { float s = 0; for (int k = 0; k < 12; ++k) s += rand() / (float)RAND_MAX; h[i] = (s - 6.0f) * 3.0f; }
        cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(prof, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int cfg2 = 0; cfg2 < 2; ++cfg2) {
            const int cc2 = cfg2 ? 4091 : 1024, k2 = cfg2 ? 128 : 256;
            cudaMemset(po, 0, 512);
            prof<<<1, 512, smem>>>(d, cc2, k2, po);
            long long r[32]; cudaMemcpy(r, po, 256, cudaMemcpyDeviceToHost);
            printf("phase stamps cc=%d K=%d (cycles): ", cc2, k2);
            for (int i = 0; i < 32; ++i) if (i == 0 || r[i]) printf("%lld ", r[i]);
            printf("\n");
        }
    }
    return 0;
}

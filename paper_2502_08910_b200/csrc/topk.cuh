// CTA-wide exact top-K over order keys in shared memory (shared by the decode
// stages and the page-cache victim selection).
#pragma once

#include "common.cuh"

namespace hpk {

// ----------------------------------------------------------------------- top-k
// Exclusive scan over the CTA for any multiple-of-32 block size.
__device__ __forceinline__ int block_scan_rt(int v, int* tmp) {
    const int lane = threadIdx.x & 31, w = warp_id(), nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = lane < nw ? tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) tmp[lane] = t;
    }
    __syncthreads();
    const int base = w ? tmp[w - 1] : 0;
    __syncthreads();
    return base + x - v;
}

// Exact top-K of cc chunk scores held in shared memory as order keys (keys[j] =
// order_key(score_j)): the K largest by (score desc, chunk asc) — the reference's
// stable_sort order (pruning.cpp:187-192) — written to sel[0..K) in ascending
// chunk order. Radix select on v = key - min(key) with 8-bit digits from the highest
// differing bit. Latency-shaped for one CTA: two barriers per pass (bins are
// rotated and cleared ahead, so no clearing barrier), one for the extrema, one for
// the emission scan — ties and greater-than counts scanned together as one packed
// word, so ties keep the lowest chunks.
struct alignas(16) TopkShared {
    int hist[3][256];
    int scan[32];
    uint32_t wmin[32], wmax[32];
    int digit, above;
};

__device__ inline void cta_topk_smem(const uint32_t* keys, int cc, int K, int32_t* sel, TopkShared& sh,
                                     int cut = -1) {
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
    trace(3, 3);
    if (cut == 10) return;  // dev-build phase cuts (decode_topk_kernel)
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
        if (shift + width == hb + 1) trace(3, 5);
        if (cut == 11) return;
        if (shift == 0) break;
        width = min(8, shift);
        shift -= width;
    }
    trace(3, 6);
    if (cut == 12) return;
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
    if (lane == 31) sh.scan[w] = x;
    __syncthreads();
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
}

}  // namespace hpk

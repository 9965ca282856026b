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
// chunk order. Radix select on v = key - min(key): the scores of one mask span a
// narrow range, so 8-bit digits start at the highest differing bit and spread over
// the 256 shared-memory bins (3 passes for a typical 20-bit range). Emission walks
// contiguous per-thread runs with two block scans, so ties keep the lowest chunks.
struct TopkShared {
    int hist[256];
    int scan[32];
    uint32_t kmin, kmax;
    int digit, above;
};

__device__ inline void cta_topk_smem(const uint32_t* keys, int cc, int K, int32_t* sel, TopkShared& sh) {
    const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = warp_id();
    uint32_t lmin = 0xffffffffu, lmax = 0u;
    for (int j = t; j < cc; j += nt) {
        const uint32_t u = keys[j];
        lmin = min(lmin, u);
        lmax = max(lmax, u);
    }
    lmin = __reduce_min_sync(0xffffffffu, lmin);
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if (t == 0) { sh.kmin = 0xffffffffu; sh.kmax = 0u; }
    __syncthreads();
    if (lane == 0) { atomicMin(&sh.kmin, lmin); atomicMax(&sh.kmax, lmax); }
    __syncthreads();
    trace(3, 3);
    const uint32_t kmin = sh.kmin, range = sh.kmax - sh.kmin;
    const int hb = range ? 31 - __clz(range) : 0;  // highest differing bit
    int width = min(8, hb + 1);
    int shift = hb + 1 - width;                    // current digit = bits [shift, shift + width)
    uint32_t prefix = 0;                           // the target's bits above the current digit
    int need = K;
    for (;;) {
        for (int i = t; i < 256; i += nt) sh.hist[i] = 0;
        __syncthreads();
        const int hi = shift + width;
        for (int j = t; j < cc; j += nt) {
            const uint32_t v = keys[j] - kmin;
            const uint32_t above_bits = hi >= 32 ? 0u : (v >> hi);
            if (above_bits == prefix) atomicAdd(&sh.hist[(v >> shift) & ((1u << width) - 1u)], 1);
        }
        __syncthreads();
        if (w == 0) {  // bin holding the need-th largest: suffix sums over 8 bins per lane
            int c[8], tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { c[k] = sh.hist[lane * 8 + k]; tot += c[k]; }
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
        prefix = (prefix << width) | static_cast<uint32_t>(sh.digit);
        need -= sh.above;
        if (shift + width == hb + 1) trace(3, 5);
        if (shift == 0) break;
        width = min(8, shift);
        shift -= width;
    }
    trace(3, 6);
    const uint32_t kth = prefix + kmin;  // the K-th largest key; keep `need` of its copies
    const int per = (cc + nt - 1) / nt;
    const int j0 = min(cc, t * per), j1 = min(cc, j0 + per);
    int ties = 0, gts = 0;
    for (int j = j0; j < j1; ++j) {
        const uint32_t u = keys[j];
        ties += u == kth;
        gts += u > kth;
    }
    const int tie_base = block_scan_rt(ties, sh.scan);
    const int take = gts + max(0, min(need - tie_base, ties));
    int r = block_scan_rt(take, sh.scan);
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

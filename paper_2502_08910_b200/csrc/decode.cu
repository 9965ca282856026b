// Fused decode path (d = 128): one kernel per pruning stage with the exact
// top-k fused into the last CTA of each mask, implicit stage lists, and a
// segment-mode split-K BSA with a fused log-sum-exp combine.
//
// Reference semantics (paths relative to /root/reference/proj):
//   stage descent / scores / top-k   pruning.cpp:69-98,153-200, tensor.cpp:88-114
//   decode stage chaining            decode.cpp:225-249 (stage i consumes stage i-1)
//   selected set for the token       sparse_attention.cpp:95-112 (1-row block)
//   attention_row                    sparse_attention.cpp:33-60
// Exactness contract as in prune.cu: sequential separately-rounded fp32 dots,
// Alg. 3 descent with strict '>', stable (score desc, chunk asc) top-k.
//
// B200 mapping. Stage 1 at 1M ctx x 8 KV groups is 131K independent descents of
// 9 dependent 256 B row gathers; it is HBM-bound only if all of them are in
// flight at once. A warp owns 32 descents (lane = chunk) of one q-head and
// stages its 32 rows per step in 8 KB of shared memory with 16 B cp.async
// (XOR-swizzled 16 B chunks: conflict-free LDS.128 without padding), so 7 CTAs
// of 4 warps (<= 72 registers/thread) fit per SM and the whole stage is one
// wave. The mask's last CTA to finish (atomic ticket) runs the radix select on
// the mask's chunk scores and emits only the kept chunk ids; the next stage
// resolves its input positions through them (hp_list_ref), so the 32K / 8K
// intermediate index lists never touch HBM on the critical path.

#include <algorithm>
#include <cmath>

#include "common.cuh"

using namespace hpk;

namespace {

constexpr int kD = 128;
constexpr int kStageWarps = 4;     // warps per stage CTA
constexpr int kBsaWarps = 8;
constexpr int kBsaKeysPerWarp = 8;
constexpr int kBsaKeysPerCta = kBsaWarps * kBsaKeysPerWarp;  // 64
constexpr int kMaxHC = 8;

__device__ __forceinline__ int64_t ref_token(const hp_list_ref& L, int mask, int64_t pos) {
#pragma unroll 1
    for (int i = L.depth - 1; i >= 0; --i) {
        const uint32_t lc = static_cast<uint32_t>(L.lc[i]);
        const uint32_t p32 = static_cast<uint32_t>(pos);  // list positions < 2^31
        const uint32_t r = p32 / lc;
        pos = static_cast<int64_t>(L.sel[i][static_cast<int64_t>(mask) * L.sel_stride[i] + r]) * lc + (p32 - r * lc);
    }
    return L.base_list ? static_cast<int64_t>(L.base_list[mask * L.base_stride + pos]) : L.range_start + pos;
}

// ----------------------------------------------------------------------------- dots
// Sequential fp32 dot of q (shared, broadcast) with the lane's staged row.
template <typename T>
__device__ __forceinline__ float dot_row(const unsigned char* row, int swz, const float* q);

template <>
__device__ __forceinline__ float dot_row<bf16_t>(const unsigned char* row, int swz, const float* q) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
        const uint4 w = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
        const float4 qa = q4[2 * c], qb = q4[2 * c + 1];
        acc = __fadd_rn(acc, __fmul_rn(qa.x, bf16_lo(w.x)));
        acc = __fadd_rn(acc, __fmul_rn(qa.y, bf16_hi(w.x)));
        acc = __fadd_rn(acc, __fmul_rn(qa.z, bf16_lo(w.y)));
        acc = __fadd_rn(acc, __fmul_rn(qa.w, bf16_hi(w.y)));
        acc = __fadd_rn(acc, __fmul_rn(qb.x, bf16_lo(w.z)));
        acc = __fadd_rn(acc, __fmul_rn(qb.y, bf16_hi(w.z)));
        acc = __fadd_rn(acc, __fmul_rn(qb.z, bf16_lo(w.w)));
        acc = __fadd_rn(acc, __fmul_rn(qb.w, bf16_hi(w.w)));
    }
    return acc;
}

// Same dot when every product q[i]*k[i] is exact in fp32 (bf16 x bf16 in range):
// fma(q, k, acc) rounds once, exactly like acc + (q*k) with an exact product.
__device__ __forceinline__ float dot_row_fma(const unsigned char* row, int swz, const float* q) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
        const uint4 w = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
        const float4 qa = q4[2 * c], qb = q4[2 * c + 1];
        acc = __fmaf_rn(qa.x, bf16_lo(w.x), acc);
        acc = __fmaf_rn(qa.y, bf16_hi(w.x), acc);
        acc = __fmaf_rn(qa.z, bf16_lo(w.y), acc);
        acc = __fmaf_rn(qa.w, bf16_hi(w.y), acc);
        acc = __fmaf_rn(qb.x, bf16_lo(w.z), acc);
        acc = __fmaf_rn(qb.y, bf16_hi(w.z), acc);
        acc = __fmaf_rn(qb.z, bf16_lo(w.w), acc);
        acc = __fmaf_rn(qb.w, bf16_hi(w.w), acc);
    }
    return acc;
}

// q is bf16-exact with |q| in [2^-63, 2^63] or 0 (so bf16 products stay exact).
__device__ __forceinline__ bool q_product_safe(float x) {
    const uint32_t u = __float_as_uint(x);
    if ((u & 0xffffu) != 0u) return false;
    const float ax = fabsf(x);
    return ax == 0.0f || (ax >= 1.0842022e-19f && ax <= 9.2233720e18f);
}

template <>
__device__ __forceinline__ float dot_row<float>(const unsigned char* row, int swz, const float* q) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
        const float4 w = *reinterpret_cast<const float4*>(row + ((c ^ swz) << 4));
        const float4 qa = q4[c];
        acc = __fadd_rn(acc, __fmul_rn(qa.x, w.x));
        acc = __fadd_rn(acc, __fmul_rn(qa.y, w.y));
        acc = __fadd_rn(acc, __fmul_rn(qa.z, w.z));
        acc = __fadd_rn(acc, __fmul_rn(qa.w, w.w));
    }
    return acc;
}

template <typename T>
__device__ __forceinline__ float elem(const unsigned char* row, int swz, int i) {
    constexpr int per = 16 / sizeof(T);
    const int c = i / per, o = i - c * per;
    const T* p = reinterpret_cast<const T*>(row + ((c ^ swz) << 4));
    return load_elem(p, o);
}

// Rotated dot: apply_rope_inplace (tensor.cpp:61-79) then the sequential dot.
template <typename T>
__device__ __forceinline__ float dot_row_rot(const unsigned char* row, int swz, const float* q,
                                             const float* cs, const float* sn) {
    float acc = 0.0f;
    constexpr int half = kD / 2;
#pragma unroll 2
    for (int i = 0; i < half; ++i) {
        const float x = elem<T>(row, swz, i), y = elem<T>(row, swz, i + half);
        const float r = __fsub_rn(__fmul_rn(x, __ldg(cs + i)), __fmul_rn(y, __ldg(sn + i)));
        acc = __fadd_rn(acc, __fmul_rn(q[i], r));
    }
#pragma unroll 2
    for (int i = 0; i < half; ++i) {
        const float x = elem<T>(row, swz, i), y = elem<T>(row, swz, i + half);
        const float r = __fadd_rn(__fmul_rn(x, __ldg(sn + i)), __fmul_rn(y, __ldg(cs + i)));
        acc = __fadd_rn(acc, __fmul_rn(q[half + i], r));
    }
    return acc;
}

// ------------------------------------------------------------------------ staging
template <typename T>
struct RowGeom {
    static constexpr int bytes = kD * sizeof(T);        // 256 or 512
    static constexpr int chunks = bytes / 16;           // 16 or 32
    static constexpr int rows_per_instr = 32 / chunks;  // 2 or 1
};

// Gather one key row per active lane into the warp's swizzled staging area.
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Optionally warms L2 with the lane's two possible next-step rows (pf0/pf1, -1 = none)
// while this step's gather is in flight: the descent direction is unknown until the
// compare, but both candidates are (used for latency-bound stages only — it costs
// one wasted row per step in DRAM traffic).
template <typename T>
__device__ __forceinline__ void stage_rows(const hp_kv_view& kv, int kvh, int64_t tok,
                                           unsigned char* ks, int lane, int64_t pf0 = -1,
                                           int64_t pf1 = -1) {
    using G = RowGeom<T>;
    const char* p = tok >= 0 ? kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, tok, sizeof(T)) : nullptr;
    const unsigned long long pu = reinterpret_cast<unsigned long long>(p);
    const int c = lane % G::chunks, sub = lane / G::chunks;
#pragma unroll
    for (int r = 0; r < 32; r += G::rows_per_instr) {
        const int row = r + sub;
        const unsigned long long pp = __shfl_sync(0xffffffffu, pu, row);
        if (pp) cp_async16(ks + row * G::bytes + ((c ^ (row & (G::chunks - 1))) << 4),
                           reinterpret_cast<const char*>(pp) + (c << 4));
    }
    if (pf0 >= 0) {
        const char* q0 = kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, pf0, sizeof(T));
#pragma unroll
        for (int o = 0; o < G::bytes; o += 128) prefetch_l2(q0 + o);
    }
    if (pf1 >= 0) {
        const char* q1 = kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, pf1, sizeof(T));
#pragma unroll
        for (int o = 0; o < G::bytes; o += 128) prefetch_l2(q1 + o);
    }
    cp_async_wait_all();
    __syncwarp();
}

// ----------------------------------------------------------------------- top-k
// Exclusive scan over the CTA for any multiple-of-32 block size.
__device__ __forceinline__ int block_scan_rt(int v, int* tmp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
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

// Exact top-K of `cc` chunk scores for one mask by the whole CTA: radix select
// on order keys (-0 folded onto +0), ties to the lowest chunk index, survivors
// emitted in ascending chunk order (pruning.cpp:187-192).
__device__ void cta_topk(const float* sc, int64_t cc, int K, int32_t* sel_out, uint32_t* skeys,
                         int smem_cap, int trace_id) {
    __shared__ int hist[256];
    __shared__ int scan_tmp[32];
    __shared__ int sh_digit, sh_above;
    const int nt = blockDim.x;
    const bool in_smem = cc <= smem_cap;
    if (in_smem) {
        // batched loads: 8 independent L2 reads in flight per thread
        for (int64_t b0 = 0; b0 < cc; b0 += 8 * nt) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t j = b0 + k * nt + threadIdx.x;
                v[k] = j < cc ? __ldcg(sc + j) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t j = b0 + k * nt + threadIdx.x;
                if (j < cc) skeys[j] = order_key(v[k]);
            }
        }
        __syncthreads();
    }
    // Radix select on v = key - kmin: chunk scores of one mask span a narrow range, so
    // digits start at the highest bit that differs and the bins spread out (plain
    // shared atomics, no same-address serialisation). Order is unchanged by the shift.
    trace(trace_id, 6);
    __shared__ uint32_t sh_min, sh_max;
    uint32_t lmin = 0xffffffffu, lmax = 0u;
    for (int64_t j = threadIdx.x; j < cc; j += nt) {
        const uint32_t u = in_smem ? skeys[j] : order_key(__ldcg(sc + j));
        lmin = min(lmin, u);
        lmax = max(lmax, u);
    }
    lmin = __reduce_min_sync(0xffffffffu, lmin);
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if (threadIdx.x == 0) { sh_min = 0xffffffffu; sh_max = 0u; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { atomicMin(&sh_min, lmin); atomicMax(&sh_max, lmax); }
    __syncthreads();
    const uint32_t kmin = sh_min, range = sh_max - sh_min;
    auto key = [&](int64_t j) -> uint32_t { return (in_smem ? skeys[j] : order_key(__ldcg(sc + j))) - kmin; };
    // 4-bit digits counted with warp ballots: each element contributes 5 ballots
    // (validity + 4 digit bit-planes) and lane b < 16 popcounts bin b's mask. Shared
    // atomics cost ~2 cycles per lane on this part; the ballot histogram has no
    // contention and no atomics at all.
    int* whist = hist;  // [nwarp (<= 16)][16] per-warp bin counts
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = nt >> 5;
    uint32_t prefix = 0, pmask = 0;
    int need = K;
    const int hb = range ? 31 - __clz(range) : 0;  // highest differing bit
    int s = hb >= 3 ? hb - 3 : 0;                  // digit = bits [s, s+3]
    for (;;) {
        int cnt = 0;
        for (int64_t b0 = static_cast<int64_t>(wid) * 32; b0 < cc; b0 += nt) {
            const int64_t j = b0 + lane;
            const uint32_t u = j < cc ? key(j) : 0u;
            const uint32_t dg = (u >> s) & 15u;
            const unsigned vb = __ballot_sync(0xffffffffu, j < cc && (u & pmask) == prefix);
            const unsigned p0 = __ballot_sync(0xffffffffu, dg & 1u);
            const unsigned p1 = __ballot_sync(0xffffffffu, dg & 2u);
            const unsigned p2 = __ballot_sync(0xffffffffu, dg & 4u);
            const unsigned p3 = __ballot_sync(0xffffffffu, dg & 8u);
            const unsigned m = vb & ((lane & 1) ? p0 : ~p0) & ((lane & 2) ? p1 : ~p1) &
                               ((lane & 4) ? p2 : ~p2) & ((lane & 8) ? p3 : ~p3);
            cnt += __popc(m);
        }
        if (lane < 16) whist[wid * 16 + lane] = cnt;
        __syncthreads();
        if (wid == 0) {
            int c = 0;
            if (lane < 16)
                for (int w2 = 0; w2 < nwarp; ++w2) c += whist[w2 * 16 + lane];
            int suf = c;  // inclusive suffix over bins [lane, 15]
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 16) suf += y;
            }
            const int above = suf - c;
            const unsigned hit = __ballot_sync(0xffffffffu, lane < 16 && above < need && need <= above + c);
            if (lane == __ffs(hit) - 1) { sh_digit = lane; sh_above = above; }
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(sh_digit) << s;
        pmask |= 15u << s;
        need -= sh_above;
        if (s == 0) break;
        s = s >= 4 ? s - 4 : 0;  // a final overlapping digit re-reads fixed bits: harmless
    }
    trace(trace_id, 7);
    // Each thread owns a contiguous run of chunk indices so ranks follow index order.
    const int64_t per = (cc + nt - 1) / nt;
    const int64_t j0 = min64(cc, threadIdx.x * per), j1 = min64(cc, j0 + per);
    int ties = 0, gts = 0;
    for (int64_t j = j0; j < j1; ++j) {
        const uint32_t u = key(j);
        ties += u == prefix;
        gts += u > prefix;
    }
    const int tie_base = block_scan_rt(ties, scan_tmp);
    const int take = gts + max(0, min(need - tie_base, ties));
    int r = block_scan_rt(take, scan_tmp);
    int trank = tie_base;
    for (int64_t j = j0; j < j1; ++j) {
        const uint32_t u = key(j);
        bool s = u > prefix;
        if (u == prefix) { s = trank < need; ++trank; }
        if (s) sel_out[r++] = static_cast<int32_t>(j);
    }
    __syncthreads();
}

// Histogram-guided exact top-K (the fast path). Every descent CTA has already added
// its chunks' order keys to two global per-mask histograms — coarse (key >> 24) and
// fine (key >> 16) — so the last CTA only walks two 256-bin slices to find the
// 16-bit bin holding the K-th largest key, resolves that bin's few members exactly
// by (key desc, chunk asc) rank, and compacts the survivors in chunk order. It
// resets every bin it consumed for the next launch. Returns false (nothing written)
// when the inputs do not fit its shared buffers; the caller then runs cta_topk.
constexpr int kTopkSmemKeys = 4096;
constexpr int kCandCap = 512;

__device__ bool cta_topk_hist(const float* sc, int64_t cc, int K, int32_t* sel_out,
                              unsigned char* buf, int* coarse, int* fine, int trace_id) {
    __shared__ int scan_tmp[32];
    __shared__ int sh_c, sh_above_c, sh_f, sh_above_f, sh_ncand;
    if (cc > kTopkSmemKeys) return false;
    const int nt = blockDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* keys = reinterpret_cast<uint32_t*>(buf);                    // [cc]
    uint32_t* cand_key = keys + kTopkSmemKeys;                             // [kCandCap]
    int* cand_idx = reinterpret_cast<int*>(cand_key + kCandCap);           // [kCandCap]
    uint32_t* selbits = reinterpret_cast<uint32_t*>(cand_idx + kCandCap);  // [kTopkSmemKeys/32]
    int* h = reinterpret_cast<int*>(selbits + kTopkSmemKeys / 32);         // [256]
    int* hc = h + 256;                                                     // [256] coarse copy
    // batched key loads + coarse histogram fetch
    for (int64_t b0 = 0; b0 < cc; b0 += 8 * nt) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t j = b0 + k * nt + threadIdx.x;
            v[k] = __ldcg(sc + min64(j, cc - 1));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t j = b0 + k * nt + threadIdx.x;
            if (j < cc) keys[j] = order_key(v[k]);
        }
    }
    for (int i = threadIdx.x; i < 256; i += nt) h[i] = hc[i] = __ldcg(coarse + i);
    for (int i = threadIdx.x; i < kTopkSmemKeys / 32; i += nt) selbits[i] = 0u;
    if (threadIdx.x == 0) sh_ncand = 0;
    __syncthreads();
    trace(trace_id, 6);
    // one warp finds the bin holding the K-th largest from the top (8 bins per lane)
    auto find_digit = [&](int need, int* out_digit, int* out_above) {
        if (wid == 0) {
            int c[8], tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { c[k] = h[lane * 8 + k]; tot += c[k]; }
            int suf = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += y;
            }
            int above = suf - tot;
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                if (above < need && need <= above + c[k]) { *out_digit = lane * 8 + k; *out_above = above; }
                above += c[k];
            }
        }
        __syncthreads();
    };
    find_digit(K, &sh_c, &sh_above_c);
    const int cstar = sh_c;
    for (int i = threadIdx.x; i < 256; i += nt) h[i] = __ldcg(fine + cstar * 256 + i);
    __syncthreads();
    find_digit(K - sh_above_c, &sh_f, &sh_above_f);
    const uint32_t t16 = (static_cast<uint32_t>(cstar) << 8) | static_cast<uint32_t>(sh_f);
    const int need = K - sh_above_c - sh_above_f;  // members of bin t16 to keep (>= 1)
    const int m = h[sh_f];
    if (m > kCandCap) {
        // pathological concentration: leave the histograms to be reset by the caller path
        return false;
    }
    // gather the threshold bin's members
    for (int64_t j = threadIdx.x; j < cc; j += nt) {
        const uint32_t u = keys[j];
        if ((u >> 16) == t16) {
            const int p = atomicAdd(&sh_ncand, 1);
            cand_key[p] = u;
            cand_idx[p] = static_cast<int>(j);
        }
    }
    __syncthreads();
    // exact rank inside the bin: (key desc, chunk asc) == the reference's stable order
    for (int i = threadIdx.x; i < m; i += nt) {
        const uint32_t ki = cand_key[i];
        const int ii = cand_idx[i];
        int rank = 0;
        for (int c = 0; c < m; ++c) {
            const uint32_t kc = cand_key[c];
            rank += kc > ki || (kc == ki && cand_idx[c] < ii);
        }
        if (rank < need) atomicOr(&selbits[ii >> 5], 1u << (ii & 31));
    }
    __syncthreads();
    trace(trace_id, 7);
    // ordered emission over contiguous per-thread runs; reset the consumed bins
    const int64_t per = (cc + nt - 1) / nt;
    const int64_t j0 = min64(cc, threadIdx.x * per), j1 = min64(cc, j0 + per);
    int take = 0;
    for (int64_t j = j0; j < j1; ++j) {
        const uint32_t u16 = keys[j] >> 16;
        take += u16 > t16 || (u16 == t16 && ((selbits[j >> 5] >> (j & 31)) & 1u));
    }
    // reset: every coarse bin, plus the fine slice under each occupied coarse bin
    for (int b = threadIdx.x; b < 256; b += nt) {
        if (hc[b] > 0) {
            int4* f4 = reinterpret_cast<int4*>(fine + b * 256);
            for (int i = 0; i < 64; ++i) f4[i] = make_int4(0, 0, 0, 0);
        }
        coarse[b] = 0;
    }
    int r = block_scan_rt(take, scan_tmp);
    for (int64_t j = j0; j < j1; ++j) {
        const uint32_t u16 = keys[j] >> 16;
        if (u16 > t16 || (u16 == t16 && ((selbits[j >> 5] >> (j & 31)) & 1u))) sel_out[r++] = static_cast<int32_t>(j);
    }
    __syncthreads();
    return true;
}

// ------------------------------------------------------------------ stage kernel
template <typename T, bool EXT>
__global__ void __launch_bounds__(kStageWarps * 32, 7)
decode_stage_kernel(const hp_decode_stage_args a, float* scores, int* tickets, int* hist_coarse,
                    int* hist_fine, int cg, int prefetch) {
    extern __shared__ __align__(128) unsigned char smem[];
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    const int m = blockIdx.y;
    const int64_t n_in = a.in_count ? a.in_count[m] : a.in_count_const;
    const int lc = a.chunk_size;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int K = a.keep / lc;
    const int chunks_per_cta = 32 * cg;
    const int64_t chunk0 = static_cast<int64_t>(blockIdx.x) * chunks_per_cta;

    if (n_in <= a.keep || cc <= K) {  // identity (pruning.cpp:159-168): keep every chunk
        if (blockIdx.x == 0) {
            for (int64_t j = threadIdx.x; j < cc; j += blockDim.x) a.sel_out[static_cast<int64_t>(m) * a.sel_stride + j] = static_cast<int32_t>(j);
            if (threadIdx.x == 0) a.out_count[m] = static_cast<int32_t>(n_in);
        }
        return;
    }
    if (chunk0 >= cc) return;
    trace(10 + lc, 0);

    const int nwarps = blockDim.x >> 5;
    // staging first so every derived pointer stays a shared-window pointer (LDS, not LD.E)
    unsigned char* stage = smem;                                      // [nwarps][32][row]
    float* qs = reinterpret_cast<float*>(smem + static_cast<size_t>(nwarps) * 32 * G::bytes);  // [hpm][128]
    float* red = qs + hpm * kD;                                       // [hpm][chunks_per_cta]

    bool q_safe = true;
    for (int i = threadIdx.x; i < hpm * kD; i += blockDim.x) {
        const float x = a.q[static_cast<int64_t>(m * hpm) * kD + i];
        qs[i] = x;
        q_safe &= q_product_safe(x);
    }
    // FFMA path only without rotation, with bf16 keys certified in range, and bf16-exact q
    trace(10 + lc, 1);
    const bool use_fma = __syncthreads_and(q_safe) && !EXT && sizeof(T) == 2 &&
                         a.keys_exact != nullptr && *a.keys_exact != 0;
    if constexpr (EXT) {
        constexpr int half = kD / 2;
        const int64_t qp = rope_q_position(a.rope, a.query_position, a.stream_tokens, cc);
        for (int i = threadIdx.x; i < hpm * half; i += blockDim.x) {
            const int hh = i / half, e = i - hh * half;
            float* row = qs + hh * kD;
            const float c = a.rope.cos_tab[qp * half + e], s = a.rope.sin_tab[qp * half + e];
            const float x = row[e], y = row[e + half];
            row[e] = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, s));
            row[e + half] = __fadd_rn(__fmul_rn(x, s), __fmul_rn(y, c));
        }
        __syncthreads();
    }

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* ks = stage + static_cast<size_t>(w) * 32 * G::bytes;
    const unsigned char* myrow = ks + lane * G::bytes;
    const int swz = lane & (G::chunks - 1);

    for (int item = w; item < hpm * cg; item += nwarps) {
        const int hh = item % hpm, grp = item / hpm;
        const int qh = m * hpm + hh;
        const int kvh = qh / (a.n_q_heads / a.keys.n_kv);
        const float* qrow = qs + hh * kD;
        const int64_t j = chunk0 + grp * 32 + lane;
        const bool active = j < cc;
        const int64_t base = j * lc;
        const int len = active ? static_cast<int>(min64(lc, n_in - base)) : 0;
        int64_t t_first = 0;
        bool contiguous = true;
        if (active) {
            t_first = ref_token(a.in, m, base);
            if (len > 1) contiguous = ref_token(a.in, m, base + len - 1) - t_first == len - 1;
        }
        auto token = [&](int i) -> int64_t { return contiguous ? t_first + i : ref_token(a.in, m, base + i); };
        const float* cs1 = nullptr; const float* sn1 = nullptr;
        const float* cs2 = nullptr; const float* sn2 = nullptr;
        bool same_rot = true;
        if constexpr (EXT) {
            constexpr int half = kD / 2;
            const int64_t p1 = rope_k_position(a.rope, 1, j), p2 = rope_k_position(a.rope, 2, j);
            cs1 = a.rope.cos_tab + p1 * half; sn1 = a.rope.sin_tab + p1 * half;
            cs2 = a.rope.cos_tab + p2 * half; sn2 = a.rope.sin_tab + p2 * half;
            same_rot = p1 == p2;
        }
        int first = 1, last = len, it = 0, iters = 0;
        while ((1 << iters) < len) ++iters;
        float s1 = 0.f, s2 = 0.f;
        const int mid0 = (1 + len + 1) >> 1;  // first step's mid is known up front
        stage_rows<T>(a.keys, kvh, active ? token(0) : -1, ks, lane,
                      prefetch && active && iters > 0 ? token(mid0 - 1) : -1);
        if (active) {
            if constexpr (EXT) {
                s1 = dot_row_rot<T>(myrow, swz, qrow, cs1, sn1);
                s2 = same_rot ? s1 : dot_row_rot<T>(myrow, swz, qrow, cs2, sn2);
            } else {
                s1 = s2 = use_fma ? dot_row_fma(myrow, swz, qrow) : dot_row<T>(myrow, swz, qrow);
            }
        }
        for (;;) {
            const bool go = active && it < iters && first < last;
            if (!__any_sync(0xffffffffu, go)) break;
            const int mid = (first + last + 1) >> 1;
            __syncwarp();
            int64_t pf_r = -1, pf_l = -1;
            if (prefetch && go && it + 1 < iters) {
                if (mid < last) pf_r = token(((mid + last + 1) >> 1) - 1);       // if it goes right
                if (first < mid - 1) pf_l = token(((first + mid) >> 1) - 1);     // if it goes left
            }
            stage_rows<T>(a.keys, kvh, go ? token(mid - 1) : -1, ks, lane, pf_r, pf_l);
            if (go) {
                float m1, m2;
                if constexpr (EXT) {
                    m1 = dot_row_rot<T>(myrow, swz, qrow, cs1, sn1);
                    m2 = same_rot ? m1 : dot_row_rot<T>(myrow, swz, qrow, cs2, sn2);
                } else {
                    m1 = m2 = use_fma ? dot_row_fma(myrow, swz, qrow) : dot_row<T>(myrow, swz, qrow);
                }
                if (m2 > s1) { first = mid; s1 = m1; s2 = m2; } else { last = mid - 1; }
                ++it;
            }
        }
        red[hh * chunks_per_cta + grp * 32 + lane] = s2;
        __syncwarp();
    }
    __syncthreads();
    for (int c0 = 0; c0 < chunks_per_cta; c0 += blockDim.x) {  // warp-uniform trip count
        const int c = c0 + threadIdx.x;
        const int64_t jj = chunk0 + c;
        const bool valid = c < chunks_per_cta && jj < cc;
        float best = -INFINITY;
        if (valid) {
            for (int h = 0; h < hpm; ++h) {
                const float s = red[h * chunks_per_cta + c];
                best = (best < s) ? s : best;  // std::max (pruning.cpp:182)
            }
            scores[static_cast<int64_t>(m) * a.max_chunks + jj] = best;
        }
        // Feed the selection histograms. A mask's scores share one or two coarse bins,
        // so same-bin lanes are merged first (one RED per distinct bin per warp) to
        // keep thousands of same-address atomics off the L2 slice.
        const uint32_t u = order_key(best);
        const int cb = valid ? static_cast<int>(u >> 24) : -1;
        const int fb = valid ? static_cast<int>(u >> 16) : -1;
        const unsigned cpeers = __match_any_sync(0xffffffffu, cb);
        const unsigned fpeers = __match_any_sync(0xffffffffu, fb);
        const int lane = threadIdx.x & 31;
        if (valid && lane == __ffs(cpeers) - 1) atomicAdd(hist_coarse + m * 256 + cb, __popc(cpeers));
        if (valid && lane == __ffs(fpeers) - 1) atomicAdd(hist_fine + static_cast<int64_t>(m) * 65536 + fb, __popc(fpeers));
    }
    trace(10 + lc, 2);
    (void)tickets;
}

// ----------------------------------------------------------------- top-k kernel
// Exact top-(k/l_c) chunk selection for one mask by a 1024-thread CTA (32 warps:
// every phase has enough warps to hide latency; a 4-warp "last CTA" did not).
// The descent kernel already built the mask's coarse (key >> 24) and fine
// (key >> 16) histograms, so: two 256-bin searches locate the 16-bit bin holding
// the K-th largest order key, that bin's members are ranked exactly by
// (key desc, chunk asc) — the reference's stable_sort order (pruning.cpp:187-192)
// — and one block scan emits the kept chunk ids in ascending order. A radix
// select over the keys covers the pathological case of a crowded bin.
constexpr int kTopkThreads2 = 1024;
constexpr int kTopkMaxKeys = 16384;

__device__ __forceinline__ int block_scan_1024(int v, int* tmp) { return block_scan_rt(v, tmp); }

// Finds bin b with above(b) < need <= above(b) + h[b], above(b) = sum_{b' > b} h[b'].
// h: 256 shared counts; all threads call; result in *digit / *above.
__device__ __forceinline__ void find_bin_256(const int* h, int need, int* tmp, int* digit, int* above) {
    const int t = threadIdx.x;
    const int c = t < 256 ? h[255 - t] : 0;  // reversed: bin 255 first
    const int ex = block_scan_rt(c, tmp);     // count of bins above (255 - t)
    if (t < 256 && ex < need && need <= ex + c) { *digit = 255 - t; *above = ex; }
    __syncthreads();
}

__global__ void __launch_bounds__(kTopkThreads2)
decode_topk_kernel(const hp_decode_stage_args a, const float* scores, int* hist_coarse, int* hist_fine) {
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ int scan_tmp[32];
    __shared__ int sh_c, sh_ac, sh_f, sh_af, sh_ncand;
    const int m = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
    const int n_in = a.in_count ? a.in_count[m] : static_cast<int>(a.in_count_const);
    const int lc = a.chunk_size;
    const int cc = (n_in + lc - 1) / lc;
    const int K = a.keep / lc;
    int32_t* sel = a.sel_out + static_cast<int64_t>(m) * a.sel_stride;
    if (n_in <= a.keep || cc <= K) {  // identity: every chunk kept (pruning.cpp:159-168)
        for (int j = t; j < cc; j += nt) sel[j] = j;
        if (t == 0) a.out_count[m] = n_in;
        if (a.list_out)
            for (int i = t; i < n_in; i += nt)
                a.list_out[m * a.list_out_stride + i] = static_cast<int32_t>(ref_token(a.in, m, i));
        return;
    }
    trace(3, 0);
    const float* sc = scores + static_cast<int64_t>(m) * a.max_chunks;
    int* co = hist_coarse + m * 256;
    int* fi = hist_fine + static_cast<int64_t>(m) * 65536;
    uint32_t* keys = reinterpret_cast<uint32_t*>(tsm);              // [cc]
    uint32_t* selbits = keys + kTopkMaxKeys;                         // [kTopkMaxKeys / 32]
    uint32_t* cand_key = selbits + kTopkMaxKeys / 32;                // [kCandCap]
    int* cand_idx = reinterpret_cast<int*>(cand_key + kCandCap);     // [kCandCap]
    int* h = cand_idx + kCandCap;                                    // [256]
    int* hc = h + 256;                                               // [256]
    constexpr int kPer = kTopkMaxKeys / kTopkThreads2;               // 16
    {
        float v[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = k * nt + t;
            v[k] = j < cc ? __ldcg(sc + j) : 0.f;
        }
        if (t < 256) h[t] = hc[t] = __ldcg(co + t);
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = k * nt + t;
            if (j < cc) keys[j] = order_key(v[k]);
        }
        for (int i = t; i < (cc + 31) / 32; i += nt) selbits[i] = 0u;
        if (t == 0) sh_ncand = 0;
    }
    __syncthreads();
    trace(3, 1);
    find_bin_256(h, K, scan_tmp, &sh_c, &sh_ac);
    const int cstar = sh_c;
    if (t < 256) h[t] = __ldcg(fi + cstar * 256 + t);
    __syncthreads();
    find_bin_256(h, K - sh_ac, scan_tmp, &sh_f, &sh_af);
    const uint32_t t16 = (static_cast<uint32_t>(cstar) << 8) | static_cast<uint32_t>(sh_f);
    const int need = K - sh_ac - sh_af;  // members of bin t16 to keep (>= 1)
    const int mc = h[sh_f];
    trace(3, 2);
    if (mc <= kCandCap) {
        for (int j = t; j < cc; j += nt) {
            const uint32_t u = keys[j];
            if ((u >> 16) == t16) {
                const int p = atomicAdd(&sh_ncand, 1);
                cand_key[p] = u;
                cand_idx[p] = j;
            }
        }
        __syncthreads();
        for (int i = t; i < mc; i += nt) {
            const uint32_t ki = cand_key[i];
            const int ii = cand_idx[i];
            int rank = 0;
            for (int c = 0; c < mc; ++c) {
                const uint32_t kc = cand_key[c];
                rank += kc > ki || (kc == ki && cand_idx[c] < ii);
            }
            if (rank < need) atomicOr(&selbits[ii >> 5], 1u << (ii & 31));
        }
    } else {
        // crowded threshold bin: exact 4-bit ballot radix select among its members
        // (low 16 bits), then mark the first `need` of the chosen key by chunk order
        uint32_t prefix = 0, pmask = 0;
        int nd = need;
        for (int s = 12;; s -= 4) {
            int cnt = 0;
            const int lane = t & 31, wid = t >> 5;
            for (int b0 = wid * 32; b0 < cc; b0 += nt) {
                const int j = b0 + lane;
                const uint32_t u = j < cc ? keys[j] : 0u;
                const bool in = j < cc && (u >> 16) == t16 && ((u & 0xffffu) & pmask) == prefix;
                const uint32_t dg = (u >> s) & 15u;
                const unsigned vb = __ballot_sync(0xffffffffu, in);
                const unsigned p0 = __ballot_sync(0xffffffffu, dg & 1u), p1 = __ballot_sync(0xffffffffu, dg & 2u);
                const unsigned p2 = __ballot_sync(0xffffffffu, dg & 4u), p3 = __ballot_sync(0xffffffffu, dg & 8u);
                cnt += __popc(vb & ((lane & 1) ? p0 : ~p0) & ((lane & 2) ? p1 : ~p1) &
                              ((lane & 4) ? p2 : ~p2) & ((lane & 8) ? p3 : ~p3));
            }
            if (t < 256) h[t] = 0;
            __syncthreads();
            if (lane < 16 && cnt) atomicAdd(&h[lane], cnt);
            __syncthreads();
            find_bin_256(h, nd, scan_tmp, &sh_f, &sh_af);  // bins 16..255 are empty
            prefix |= static_cast<uint32_t>(sh_f) << s;
            pmask |= 15u << s;
            nd -= sh_af;
            if (s == 0) break;
        }
        // keys equal to (t16, prefix): keep the first nd by chunk index; greater keys all kept
        const uint32_t kth = (t16 << 16) | prefix;
        const int per = (cc + nt - 1) / nt;
        const int j0 = min(cc, t * per), j1 = min(cc, j0 + per);
        int eq = 0;
        for (int j = j0; j < j1; ++j) eq += keys[j] == kth;
        int r = block_scan_rt(eq, scan_tmp);
        for (int j = j0; j < j1; ++j) {
            const uint32_t u = keys[j];
            if ((u >> 16) == t16 && (u > kth || (u == kth && r++ < nd))) atomicOr(&selbits[j >> 5], 1u << (j & 31));
        }
    }
    __syncthreads();
    trace(3, 3);
    // ordered emission over contiguous per-thread runs
    const int per = (cc + nt - 1) / nt;
    const int j0 = min(cc, t * per), j1 = min(cc, j0 + per);
    int take = 0;
    for (int j = j0; j < j1; ++j) {
        const uint32_t u16 = keys[j] >> 16;
        take += u16 > t16 || (u16 == t16 && ((selbits[j >> 5] >> (j & 31)) & 1u));
    }
    int r = block_scan_rt(take, scan_tmp);
    for (int j = j0; j < j1; ++j) {
        const uint32_t u16 = keys[j] >> 16;
        if (u16 > t16 || (u16 == t16 && ((selbits[j >> 5] >> (j & 31)) & 1u))) sel[r++] = j;
    }
    // reset the histograms for the next stage / launch
    if (t < 256) {
        if (hc[t] > 0) {
            int4* f4 = reinterpret_cast<int4*>(fi + t * 256);
            for (int i = 0; i < 64; ++i) f4[i] = make_int4(0, 0, 0, 0);
        }
        co[t] = 0;
    }
    __syncthreads();
    const int lastc = sel[K - 1];
    const int n_out = (K - 1) * lc + min(lc, n_in - lastc * lc);
    if (t == 0) a.out_count[m] = n_out;
    if (a.list_out) {  // materialize: output position o -> chunk sel[o / lc] -> input list
        for (int o = t; o < n_out; o += nt) {
            const int r = o / lc;
            a.list_out[m * a.list_out_stride + o] =
                static_cast<int32_t>(ref_token(a.in, m, static_cast<int64_t>(sel[r]) * lc + (o - r * lc)));
        }
    }
    trace(3, 4);
}

// -------------------------------------------------------------------- BSA kernel
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T> struct Pair;
template <> struct Pair<bf16_t> {
    using V = uint32_t;
    static __device__ __forceinline__ V ld(const void* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }
    static __device__ __forceinline__ float lo(V v) { return bf16_lo(v); }
    static __device__ __forceinline__ float hi(V v) { return bf16_hi(v); }
};
template <> struct Pair<float> {
    using V = float2;
    static __device__ __forceinline__ V ld(const void* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
    static __device__ __forceinline__ float lo(V v) { return v.x; }
    static __device__ __forceinline__ float hi(V v) { return v.y; }
};

// grid = (splits, n_q_heads / HC); CTA covers 64 consecutive selected positions for
// HC q-heads sharing one kv head and one mask. Lane L holds elements 2L, 2L+1 and
// their RoPE partners 64+2L, 65+2L. The last CTA of each head group merges.
template <typename T, int HC, bool EXT>
__global__ void __launch_bounds__(kBsaWarps * 32, 3)
decode_bsa_kernel(const hp_decode_bsa_args a, float* part, int* tickets, int splits) {
    using P = Pair<T>;
    __shared__ float sm_m[kBsaWarps][HC], sm_l[kBsaWarps][HC];
    __shared__ float sm_o[kBsaWarps][HC][kD];
    __shared__ int sh_last;
    const int split = blockIdx.x, hg = blockIdx.y;
    const int h0 = hg * HC;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int mask = h0 / a.heads_per_mask;
    const int kvh = h0 / (a.n_q_heads / a.kv.n_kv);
    const int64_t pos = a.query_position;
    const int64_t sink_end = min64(a.sink_tokens, pos + 1);
    int64_t stream_begin = pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0;
    stream_begin = max64(stream_begin, sink_end);
    const int64_t n_mask = a.mask_count[mask];
    const int64_t n_sel = sink_end + n_mask + (pos + 1 - stream_begin);
    const float scale = 1.0f / sqrtf(static_cast<float>(kD));
    constexpr int half = kD / 2;

    float qx[HC][2], qy[HC][2];
#pragma unroll
    for (int hh = 0; hh < HC; ++hh) {
        const float* qr = a.q + static_cast<int64_t>(h0 + hh) * kD;
        float x0 = qr[2 * lane], x1 = qr[2 * lane + 1], y0 = qr[half + 2 * lane], y1 = qr[half + 2 * lane + 1];
        if constexpr (EXT) {
            const float* c = a.rope.cos_tab + pos * half;
            const float* s = a.rope.sin_tab + pos * half;
            const float c0 = c[2 * lane], c1 = c[2 * lane + 1], s0 = s[2 * lane], s1 = s[2 * lane + 1];
            const float nx0 = x0 * c0 - y0 * s0, ny0 = x0 * s0 + y0 * c0;
            const float nx1 = x1 * c1 - y1 * s1, ny1 = x1 * s1 + y1 * c1;
            x0 = nx0; y0 = ny0; x1 = nx1; y1 = ny1;
        }
        qx[hh][0] = x0; qx[hh][1] = x1; qy[hh][0] = y0; qy[hh][1] = y1;
    }

    trace(2, 0);
    // this warp's 8 positions
    const int64_t p0 = static_cast<int64_t>(split) * kBsaKeysPerCta + w * kBsaKeysPerWarp;
    int64_t tok_l = -1;
    if (lane < kBsaKeysPerWarp) {
        const int64_t p = p0 + lane;
        if (p < n_sel) {
            if (p < sink_end) tok_l = p;
            else if (p < sink_end + n_mask) tok_l = ref_token(a.mask, mask, p - sink_end);
            else tok_l = stream_begin + (p - sink_end - n_mask);
        }
    }
    typename P::V kr[kBsaKeysPerWarp][2], vr[kBsaKeysPerWarp][2];
    int64_t toks[kBsaKeysPerWarp];
#pragma unroll
    for (int k = 0; k < kBsaKeysPerWarp; ++k) {
        toks[k] = __shfl_sync(0xffffffffu, tok_l, k);
        if (toks[k] >= 0) {
            const char* kp = kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kvh, toks[k], sizeof(T));
            const char* vp = kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kvh, toks[k], sizeof(T));
            kr[k][0] = P::ld(kp + 2 * lane * sizeof(T));
            kr[k][1] = P::ld(kp + (half + 2 * lane) * sizeof(T));
            vr[k][0] = P::ld(vp + 2 * lane * sizeof(T));
            vr[k][1] = P::ld(vp + (half + 2 * lane) * sizeof(T));
        } else {
            kr[k][0] = kr[k][1] = vr[k][0] = vr[k][1] = typename P::V{};
        }
    }
    trace(2, 1);
    float kx[kBsaKeysPerWarp][2], ky[kBsaKeysPerWarp][2];
#pragma unroll
    for (int k = 0; k < kBsaKeysPerWarp; ++k) {
        float x0 = P::lo(kr[k][0]), x1 = P::hi(kr[k][0]), y0 = P::lo(kr[k][1]), y1 = P::hi(kr[k][1]);
        if constexpr (EXT) {
            if (toks[k] >= 0) {
                const int64_t kp = pos + 1 - n_sel + (p0 + k);  // streaming_positions (rope_policy.cpp:59-72)
                const float* c = a.rope.cos_tab + kp * half;
                const float* s = a.rope.sin_tab + kp * half;
                const float c0 = c[2 * lane], c1 = c[2 * lane + 1], s0 = s[2 * lane], s1 = s[2 * lane + 1];
                const float nx0 = x0 * c0 - y0 * s0, ny0 = x0 * s0 + y0 * c0;
                const float nx1 = x1 * c1 - y1 * s1, ny1 = x1 * s1 + y1 * c1;
                x0 = nx0; y0 = ny0; x1 = nx1; y1 = ny1;
            }
        }
        kx[k][0] = x0; kx[k][1] = x1; ky[k][0] = y0; ky[k][1] = y1;
    }
#pragma unroll
    for (int hh = 0; hh < HC; ++hh) {
        float s[kBsaKeysPerWarp];
        float mt = -INFINITY;
#pragma unroll
        for (int k = 0; k < kBsaKeysPerWarp; ++k) {
            float part_dot = qx[hh][0] * kx[k][0] + qx[hh][1] * kx[k][1] + qy[hh][0] * ky[k][0] + qy[hh][1] * ky[k][1];
            part_dot = warp_sum(part_dot);
            s[k] = toks[k] >= 0 ? part_dot * scale : -INFINITY;
            mt = fmaxf(mt, s[k]);
        }
        float l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
        if (mt != -INFINITY) {
#pragma unroll
            for (int k = 0; k < kBsaKeysPerWarp; ++k) {
                const float p = toks[k] >= 0 ? expf(s[k] - mt) : 0.f;
                l += p;
                o0 += p * P::lo(vr[k][0]); o1 += p * P::hi(vr[k][0]);
                o2 += p * P::lo(vr[k][1]); o3 += p * P::hi(vr[k][1]);
            }
        }
        if (lane == 0) { sm_m[w][hh] = mt; sm_l[w][hh] = l; }
        sm_o[w][hh][2 * lane] = o0; sm_o[w][hh][2 * lane + 1] = o1;
        sm_o[w][hh][half + 2 * lane] = o2; sm_o[w][hh][half + 2 * lane + 1] = o3;
    }
    __syncthreads();
    trace(2, 2);
    // CTA partial per head -> workspace [hg][split][hh][2 + 128]
    for (int idx = threadIdx.x; idx < HC * kD; idx += blockDim.x) {
        const int hh = idx / kD, e = idx - hh * kD;
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < kBsaWarps; ++ww) M = fmaxf(M, sm_m[ww][hh]);
        float L = 0.f, o = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int ww = 0; ww < kBsaWarps; ++ww) {
                const float f = sm_m[ww][hh] == -INFINITY ? 0.f : expf(sm_m[ww][hh] - M);
                L += sm_l[ww][hh] * f;
                o += sm_o[ww][hh][e] * f;
            }
        }
        float* pp = part + ((static_cast<int64_t>(hg) * splits + split) * HC + hh) * (kD + 2);
        if (e == 0) { pp[0] = M; pp[1] = L; }
        pp[2 + e] = o;
    }
    const bool last_cta = cta_ticket_last(&tickets[hg], splits, &sh_last);
    trace(2, 6);
    if (!last_cta) return;
    trace(2, 3);
    // Merge all splits of this head group (log-sum-exp). Phase 1 pulls every (m, l)
    // in one parallel load, phase 2 forms per-split weights, phase 3 streams the o's
    // with independent (pipelined) loads.
    constexpr int kMaxSplitsSmem = 128;
    float* wgt = &sm_o[0][0][0];                  // reuse: [kMaxSplitsSmem][HC] weights
    float* ml = wgt + kMaxSplitsSmem * HC;        // [splits][HC][2]
    const bool fits = splits <= kMaxSplitsSmem && 3 * kMaxSplitsSmem * HC <= kBsaWarps * HC * kD;
    const float* pbase = part + static_cast<int64_t>(hg) * splits * HC * (kD + 2);
    trace(2, 7);
    if (fits) {
        for (int i = threadIdx.x; i < splits * HC; i += blockDim.x) {
            const float* pp = pbase + static_cast<int64_t>(i) * (kD + 2);
            ml[2 * i] = __ldcg(pp);
            ml[2 * i + 1] = __ldcg(pp + 1);
        }
        __syncthreads();
        if (w < HC) {
            const int hh = w;
            float M = -INFINITY;
            for (int s = lane; s < splits; s += 32)
                if (ml[2 * (s * HC + hh) + 1] > 0.f) M = fmaxf(M, ml[2 * (s * HC + hh)]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            float L = 0.f;
            for (int s = lane; s < splits; s += 32) {
                const float l = ml[2 * (s * HC + hh) + 1];
                const float f = l > 0.f ? expf(ml[2 * (s * HC + hh)] - M) : 0.f;
                wgt[s * HC + hh] = f;
                L += l * f;
            }
            L = warp_sum(L);
            if (lane == 0) { sm_m[0][hh] = M; sm_l[0][hh] = L; }
        }
        __syncthreads();
    }
    trace(2, 5);
    for (int idx = threadIdx.x; idx < HC * kD; idx += blockDim.x) {
        const int hh = idx / kD, e = idx - hh * kD;
        const float* pb = pbase + static_cast<int64_t>(hh) * (kD + 2);
        float M, L, o = 0.f;
        if (fits) {
            M = sm_m[0][hh];
            L = sm_l[0][hh];
            constexpr int kBatch = 16;  // independent loads in flight per thread
            for (int s0 = 0; s0 < splits; s0 += kBatch) {
                // unconditional loads (clamped index, zero weight past the end) so the
                // batch issues back to back instead of load->use->load on one register
                float vals[kBatch];
#pragma unroll
                for (int k = 0; k < kBatch; ++k) {
                    const int s = min(s0 + k, splits - 1);
                    vals[k] = __ldcg(pb + static_cast<int64_t>(s) * HC * (kD + 2) + 2 + e);
                }
#pragma unroll
                for (int k = 0; k < kBatch; ++k) {
                    const int s = s0 + k;
                    o += vals[k] * (s < splits ? wgt[min(s, splits - 1) * HC + hh] : 0.f);
                }
            }
        } else {
            M = -INFINITY;
            for (int s = 0; s < splits; ++s) {
                const float* pp = pb + static_cast<int64_t>(s) * HC * (kD + 2);
                if (__ldcg(pp + 1) > 0.f) M = fmaxf(M, __ldcg(pp));
            }
            L = 0.f;
            for (int s = 0; s < splits; ++s) {
                const float* pp = pb + static_cast<int64_t>(s) * HC * (kD + 2);
                const float l = __ldcg(pp + 1);
                if (l > 0.f) {
                    const float f = expf(__ldcg(pp) - M);
                    L += l * f;
                    o += __ldcg(pp + 2 + e) * f;
                }
            }
        }
        const int64_t h = h0 + hh;
        a.out[h * kD + e] = L > 0.f ? o / L : NAN;
        if (a.part_o) a.part_o[h * kD + e] = L > 0.f ? o / L : 0.f;
        if (e == 0 && a.part_m) { a.part_m[h] = M; a.part_l[h] = L; }
    }
    trace(2, 4);
}

// ------------------------------------------------------------------ materialize
struct MatArgs {
    hp_list_ref ref[4];
    const int32_t* count[4];
    int32_t* out[4];
    int64_t stride[4];
};

__global__ void materialize_kernel(const MatArgs a) {
    const int l = blockIdx.z, m = blockIdx.y;
    const int64_t n = a.count[l][m];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        a.out[l][m * a.stride[l] + i] = static_cast<int32_t>(ref_token(a.ref[l], m, i));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int bsa_hc(int n_q_heads, int n_kv, int hpm) {
    const int g = n_q_heads / n_kv;
    int hc = std::__gcd(g, hpm);
    hc = std::__gcd(hc, kMaxHC);
    return std::max(1, hc);
}

template <typename T, bool EXT>
cudaError_t launch_stage(const hp_decode_stage_args& a, float* scores, int* tickets, int* coarse,
                         int* fine, cudaStream_t s) {
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    int cg = std::max(1, kStageWarps / hpm);
    const int warps = std::min(kStageWarps, std::max(hpm * cg, 1));
    const int threads = std::max(32, std::min(warps, hpm * cg) * 32);
    const int nw = threads / 32;
    const size_t smem = static_cast<size_t>(hpm) * kD * 4 + static_cast<size_t>(hpm) * 32 * cg * 4 + 128 +
                        static_cast<size_t>(nw) * 32 * G::bytes;
    auto kern = decode_stage_kernel<T, EXT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid((a.max_chunks + 32 * cg - 1) / (32 * cg), a.n_masks);
    // speculative next-row prefetch only where the stage is latency-bound (few descents)
    const int64_t lanes = static_cast<int64_t>(a.n_masks) * a.max_chunks * hpm;
    const int prefetch = lanes <= 65536 ? 1 : 0;
    kern<<<grid, threads, smem, s>>>(a, scores, tickets, coarse, fine, cg, prefetch);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t tsmem = static_cast<size_t>(kTopkMaxKeys) * 4 + kTopkMaxKeys / 8 + kCandCap * 8 + 512 * 4;
    e = cudaFuncSetAttribute(decode_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem));
    if (e != cudaSuccess) return e;
    decode_topk_kernel<<<a.n_masks, kTopkThreads2, tsmem, s>>>(a, scores, coarse, fine);
    return cudaGetLastError();
}

template <typename T, int HC, bool EXT>
cudaError_t launch_bsa(const hp_decode_bsa_args& a, float* part, int* tickets, int splits, cudaStream_t s) {
    dim3 grid(splits, a.n_q_heads / HC);
    decode_bsa_kernel<T, HC, EXT><<<grid, kBsaWarps * 32, 0, s>>>(a, part, tickets, splits);
    return cudaGetLastError();
}

template <typename T, bool EXT>
cudaError_t dispatch_bsa_hc(const hp_decode_bsa_args& a, int hc, float* part, int* tickets, int splits, cudaStream_t s) {
    switch (hc) {
        case 1: return launch_bsa<T, 1, EXT>(a, part, tickets, splits, s);
        case 2: return launch_bsa<T, 2, EXT>(a, part, tickets, splits, s);
        case 4: return launch_bsa<T, 4, EXT>(a, part, tickets, splits, s);
        default: return launch_bsa<T, 8, EXT>(a, part, tickets, splits, s);
    }
}

}  // namespace

// Developer instrumentation: record per-CTA phase stamps of kernel `kernel_id`
// (1 = decode stage, 2 = decode BSA) into buf [n_cta][8] (NULL disables).
extern "C" int hp_trace_enable(unsigned long long* buf, int kernel_id) {
    if (int rc = hph::check_cuda(cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(buf)), "hp_trace_enable")) return rc;
    return hph::check_cuda(cudaMemcpyToSymbol(g_trace_kernel, &kernel_id, sizeof(int)), "hp_trace_enable");
}

extern "C" size_t hp_decode_stage_workspace_bytes(int32_t n_masks, int32_t max_chunks) {
    return align_up(static_cast<size_t>(n_masks) * 4, 256) +             // tickets
           align_up(static_cast<size_t>(n_masks) * 256 * 4, 256) +       // coarse histograms
           static_cast<size_t>(n_masks) * 65536 * 4 +                     // fine histograms
           align_up(static_cast<size_t>(n_masks) * std::max(1, max_chunks) * 4, 256);  // scores
}

extern "C" int hp_decode_stage(const hp_decode_stage_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: null args");
    const hp_decode_stage_args& a = *ap;
    if (a.chunk_size <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: b_q and l_c must be >= 1");
    if (a.keep <= 0 || a.keep % a.chunk_size) return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: k must be a positive multiple of l_c");
    if (a.keys.d != kD) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: fused decode path needs head_dim 128");
    if (a.n_masks <= 0 || a.heads_per_mask <= 0 || a.heads_per_mask > 32 || a.n_q_heads != a.n_masks * a.heads_per_mask ||
        a.keys.n_kv <= 0 || a.n_q_heads % a.keys.n_kv)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: bad head geometry");
    if (a.in.depth < 0 || a.in.depth > 4) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: list depth");
    if (a.sel_stride < a.keep / a.chunk_size) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: sel_stride < k/l_c");
    if (a.max_chunks <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: max_chunks must be >= 1");
    if (a.max_chunks > kTopkMaxKeys)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: %d chunks per list exceed the fused selection limit %d",
                              a.max_chunks, kTopkMaxKeys);
    const size_t need = hp_decode_stage_workspace_bytes(a.n_masks, a.max_chunks);
    if (!a.workspace || a.workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: workspace too small");
    if (a.rope.extension) {
        const int pol = a.rope.layer > a.rope.early_cutoff ? a.rope.late_policy : a.rope.early_policy;
        if (pol != HP_ROPE_CHUNK_INDEXED && pol != HP_ROPE_RELATIVE)
            return hph::set_error(HP_LOGIC_ERROR, "query_position: policy not applicable to pruning");
        const int64_t need_q = pol == HP_ROPE_RELATIVE ? a.stream_tokens + 1 : min64(a.query_position, a.max_chunks + a.stream_tokens);
        const int64_t need_k = pol == HP_ROPE_RELATIVE ? 1 : a.max_chunks - 1;
        if (std::max(need_q, need_k) >= a.rope.rope_max)
            return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                                  static_cast<long long>(std::max(need_q, need_k)), static_cast<long long>(a.rope.rope_max));
    }
    // Fixed-offset regions first (tickets, selection histograms): they must stay zero
    // between launches and every stage shares this workspace; scores last (size varies).
    char* ws = static_cast<char*>(a.workspace);
    int* tickets = reinterpret_cast<int*>(ws);
    size_t off = align_up(static_cast<size_t>(a.n_masks) * 4, 256);
    int* coarse = reinterpret_cast<int*>(ws + off);
    off += align_up(static_cast<size_t>(a.n_masks) * 256 * 4, 256);
    int* fine = reinterpret_cast<int*>(ws + off);
    off += static_cast<size_t>(a.n_masks) * 65536 * 4;
    float* scores = reinterpret_cast<float*>(ws + off);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool ext = a.rope.extension != 0;
    cudaError_t e;
    if (a.keys.dtype == HP_BF16) e = ext ? launch_stage<bf16_t, true>(a, scores, tickets, coarse, fine, s) : launch_stage<bf16_t, false>(a, scores, tickets, coarse, fine, s);
    else e = ext ? launch_stage<float, true>(a, scores, tickets, coarse, fine, s) : launch_stage<float, false>(a, scores, tickets, coarse, fine, s);
    return hph::check_cuda(e, "decode_stage_kernel");
}

extern "C" size_t hp_decode_bsa_workspace_bytes(int32_t n_q_heads, int32_t max_sel) {
    const int splits = std::max(1, (max_sel + kBsaKeysPerCta - 1) / kBsaKeysPerCta);
    return align_up(static_cast<size_t>(n_q_heads) * splits * (kD + 2) * 4, 256) + align_up(static_cast<size_t>(n_q_heads) * 4, 256);
}

extern "C" int hp_decode_bsa(const hp_decode_bsa_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: null args");
    const hp_decode_bsa_args& a = *ap;
    if (a.kv.d != kD) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: fused decode path needs head_dim 128");
    if (a.n_q_heads <= 0 || a.heads_per_mask <= 0 || a.kv.n_kv <= 0 || a.n_q_heads % a.kv.n_kv || a.n_q_heads % a.heads_per_mask)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: bad head geometry");
    if (!a.q || !a.out || !a.mask_count || !a.kv.k_pool || !a.kv.v_pool) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: null pointer");
    const int64_t pos = a.query_position;
    const int64_t sink_end = std::min<int64_t>(a.sink_tokens, pos + 1);
    const int64_t stream_begin = std::max<int64_t>(pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0, sink_end);
    const int64_t max_sel = sink_end + a.max_mask + (pos + 1 - stream_begin);
    if (max_sel <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "attention_row: empty selected set");
    if (a.rope.extension) {
        if (pos >= a.rope.rope_max) return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                                                          static_cast<long long>(pos), static_cast<long long>(a.rope.rope_max));
        if (max_sel > pos + 1) return hph::set_error(HP_LOGIC_ERROR, "streaming_positions: selected tokens cannot fit below position");
    }
    const int splits = static_cast<int>((max_sel + kBsaKeysPerCta - 1) / kBsaKeysPerCta);
    const size_t need = hp_decode_bsa_workspace_bytes(a.n_q_heads, static_cast<int32_t>(max_sel));
    if (!a.workspace || a.workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: workspace too small");
    char* ws = static_cast<char*>(a.workspace);
    int* tickets = reinterpret_cast<int*>(ws);
    float* part = reinterpret_cast<float*>(ws + align_up(static_cast<size_t>(a.n_q_heads) * 4, 256));
    const int hc = bsa_hc(a.n_q_heads, a.kv.n_kv, a.heads_per_mask);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool ext = a.rope.extension != 0;
    cudaError_t e;
    if (a.kv.dtype == HP_BF16) e = ext ? dispatch_bsa_hc<bf16_t, true>(a, hc, part, tickets, splits, s) : dispatch_bsa_hc<bf16_t, false>(a, hc, part, tickets, splits, s);
    else e = ext ? dispatch_bsa_hc<float, true>(a, hc, part, tickets, splits, s) : dispatch_bsa_hc<float, false>(a, hc, part, tickets, splits, s);
    return hph::check_cuda(e, "decode_bsa_kernel");
}

__global__ void append_kernel(const hp_kv_view kv, const unsigned char* k_rows,
                              const unsigned char* v_rows, int64_t token, int32_t* keys_exact) {
    const int eb = kv.dtype == HP_BF16 ? 2 : 4;
    const int row_bytes = kv.d * eb;
    const int h = blockIdx.x;
    char* kd = const_cast<char*>(kv_row_ptr(kv, kv.k_pool, kv.k_host, h, token, eb));
    char* vd = kv.v_pool ? const_cast<char*>(kv_row_ptr(kv, kv.v_pool, kv.v_host, h, token, eb)) : nullptr;
    bool ok = true;
    for (int i = threadIdx.x; i < row_bytes; i += blockDim.x) {
        kd[i] = k_rows[h * row_bytes + i];
        if (vd) vd[i] = v_rows[h * row_bytes + i];
    }
    if (eb == 2) {
        for (int i = threadIdx.x; i < kv.d; i += blockDim.x) {
            const uint16_t bits = reinterpret_cast<const uint16_t*>(k_rows + h * row_bytes)[i];
            const float x = fabsf(__uint_as_float(static_cast<uint32_t>(bits) << 16));
            ok &= x == 0.0f || (x >= 1.0842022e-19f && x <= 9.2233720e18f);
        }
    } else {
        ok = false;
    }
    if (!__syncthreads_and(ok) && threadIdx.x == 0 && keys_exact) atomicAnd(keys_exact, 0);
}

extern "C" int hp_decode_append(const hp_kv_view* kv, const void* k_rows, const void* v_rows,
                                int64_t token, int32_t* keys_exact, void* stream) {
    if (!kv || !k_rows) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_append: null pointer");
    if (token < 0 || token >= static_cast<int64_t>(kv->num_pages) * kv->page_size)
        return hph::set_error(HP_OUT_OF_RANGE, "hp_decode_append: token beyond the cache capacity");
    append_kernel<<<kv->n_kv, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        *kv, static_cast<const unsigned char*>(k_rows), static_cast<const unsigned char*>(v_rows), token, keys_exact);
    return hph::check_cuda(cudaGetLastError(), "append_kernel");
}

extern "C" int hp_decode_materialize(const hp_list_ref* refs, const int32_t* const* counts,
                                     int32_t* const* outs, const int64_t* out_strides,
                                     int32_t n_lists, int32_t n_masks, int32_t max_count,
                                     void* stream) {
    if (n_lists <= 0 || n_lists > 4 || n_masks <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_materialize: 1..4 lists");
    MatArgs m{};
    for (int i = 0; i < n_lists; ++i) {
        m.ref[i] = refs[i];
        m.count[i] = counts[i];
        m.out[i] = outs[i];
        m.stride[i] = out_strides[i];
    }
    const int blocks = std::max(1, std::min(64, (max_count + 255) / 256));
    materialize_kernel<<<dim3(blocks, n_masks, n_lists), 256, 0, static_cast<cudaStream_t>(stream)>>>(m);
    return hph::check_cuda(cudaGetLastError(), "materialize_kernel");
}

// Hierarchical context-pruning stage (InfiniteHiP Alg. 2-3) on sm_100a.
//
// Replaces run_pruning_stage + select_rep_rotated + block_scores
// (reference proj/src/pruning.cpp:69-98,153-200, tensor.cpp:88-114) with
// index-exact results:
//   * every score is the reference's sequential fp32 dot: acc = acc + q[i]*k[i],
//     i = 0..d-1, each product and sum separately rounded (__fmul_rn/__fadd_rn,
//     never contracted to FMA), σ = max over the query-block rows with strict '>';
//   * the descent is Alg. 3 verbatim: 1-based [first,last], mid rounds half up,
//     right only on strict σ2 > σ1, ⌈log2 n⌉ iterations or until first == last;
//   * RoPE (extension on) rotates keys at key_position(branch, chunk) and queries
//     at query_position, x*c - y*s / x*s + y*c with separate roundings, from the
//     host-built table (fused into the key gather);
//   * chunk score = max over the mask's q-heads of the branch-2 rep score; the
//     kept chunks are the top k/l_c by (score desc, chunk index asc) — the
//     reference's stable_sort order — found by an exact radix select.
//
// Layout of work: a warp owns 32 consecutive chunks of one (mask, block) for
// one q-head (lane = chunk). Each descent step the warp gathers its 32 key rows
// with coalesced 16-byte cp.async into shared memory (one row per lane,
// padded stride), then every lane runs its own sequential dot. Rows already
// scored are never re-read: σ1 of the next iteration is the score just computed
// for the surviving branch (ties and policies handled exactly, see below), so a
// descent over l_c keys reads 1 + ⌈log2 l_c⌉ rows instead of the reference's
// 2⌈log2 l_c⌉ + 1.

#include <algorithm>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

using namespace hpk;

namespace {

constexpr int kTopkThreads = 512;

struct StageGeom {
    int cg;          // chunk groups (of 32) per CTA
    int rows_max;    // q rows staged per head
    int key_stride;  // bytes per staged key row
    size_t q_bytes, red_bytes, key_bytes;
};

__device__ __forceinline__ int64_t list_token(const hp_stage_args& a, int mb, int64_t pos) {
    return a.in_list ? static_cast<int64_t>(a.in_list[static_cast<int64_t>(mb) * a.in_stride + pos])
                     : static_cast<int64_t>(a.in_start[mb]) + pos;
}

// σ = max over rows of the sequential dot of q_t with the (optionally rotated) key.
template <typename T, int D, bool ROT>
__device__ __forceinline__ float block_score(const unsigned char* krow, const float* qs,
                                             int rows, int d, const float* cs, const float* sn) {
    const T* k = reinterpret_cast<const T*>(krow);
    float best = 0.0f;
    for (int t = 0; t < rows; ++t) {
        const float* qt = qs + t * d;
        float acc = 0.0f;
        if constexpr (!ROT) {
            if constexpr (D == 128 && sizeof(T) == 2) {
                const uint4* k4 = reinterpret_cast<const uint4*>(krow);
                const float4* q4 = reinterpret_cast<const float4*>(qt);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const uint4 w = k4[c];
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
            } else if constexpr (D == 128 && sizeof(T) == 4) {
                const float4* k4 = reinterpret_cast<const float4*>(krow);
                const float4* q4 = reinterpret_cast<const float4*>(qt);
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const float4 w = k4[c];
                    const float4 qa = q4[c];
                    acc = __fadd_rn(acc, __fmul_rn(qa.x, w.x));
                    acc = __fadd_rn(acc, __fmul_rn(qa.y, w.y));
                    acc = __fadd_rn(acc, __fmul_rn(qa.z, w.z));
                    acc = __fadd_rn(acc, __fmul_rn(qa.w, w.w));
                }
            } else {
                for (int i = 0; i < d; ++i) acc = __fadd_rn(acc, __fmul_rn(qt[i], load_elem(k, i)));
            }
        } else {
            // apply_rope_inplace (tensor.cpp:61-79) on the fly, then the sequential dot.
            const int half = d >> 1;
            for (int i = 0; i < half; ++i) {
                const float x = load_elem(k, i), y = load_elem(k, i + half);
                const float r = __fsub_rn(__fmul_rn(x, __ldg(cs + i)), __fmul_rn(y, __ldg(sn + i)));
                acc = __fadd_rn(acc, __fmul_rn(qt[i], r));
            }
            for (int i = 0; i < half; ++i) {
                const float x = load_elem(k, i), y = load_elem(k, i + half);
                const float r = __fadd_rn(__fmul_rn(x, __ldg(sn + i)), __fmul_rn(y, __ldg(cs + i)));
                acc = __fadd_rn(acc, __fmul_rn(qt[half + i], r));
            }
        }
        if (t == 0 || acc > best) best = acc;
    }
    return best;
}

// σ with one FHFMA per element (keys certified and q bf16-exact: every product is
// exact, so fma == the separately rounded multiply-add): the key row is held in
// registers across the query rows, the packed q rows are shared-memory broadcasts.
__device__ __forceinline__ float block_score_fma(const unsigned char* krow, const uint32_t* qb, int rows) {
    uint4 k[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) k[c] = reinterpret_cast<const uint4*>(krow)[c];
    float best = 0.0f;
    int t = 0;
    for (; t + 4 <= rows; t += 4) {  // four query rows as independent FHFMA chains
        const uint4* q4 = reinterpret_cast<const uint4*>(qb + t * 64);
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < 16; ++c) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint4 q = q4[u * 16 + c];
                acc[u] = fma_bf16(q.x, k[c].x, acc[u], false); acc[u] = fma_bf16(q.x, k[c].x, acc[u], true);
                acc[u] = fma_bf16(q.y, k[c].y, acc[u], false); acc[u] = fma_bf16(q.y, k[c].y, acc[u], true);
                acc[u] = fma_bf16(q.z, k[c].z, acc[u], false); acc[u] = fma_bf16(q.z, k[c].z, acc[u], true);
                acc[u] = fma_bf16(q.w, k[c].w, acc[u], false); acc[u] = fma_bf16(q.w, k[c].w, acc[u], true);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t + u == 0 || acc[u] > best) best = acc[u];  // rows in order, strict '>'
    }
    for (; t < rows; ++t) {
        const uint4* q4 = reinterpret_cast<const uint4*>(qb + t * 64);
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const uint4 q = q4[c];
            acc = fma_bf16(q.x, k[c].x, acc, false); acc = fma_bf16(q.x, k[c].x, acc, true);
            acc = fma_bf16(q.y, k[c].y, acc, false); acc = fma_bf16(q.y, k[c].y, acc, true);
            acc = fma_bf16(q.z, k[c].z, acc, false); acc = fma_bf16(q.z, k[c].z, acc, true);
            acc = fma_bf16(q.w, k[c].w, acc, false); acc = fma_bf16(q.w, k[c].w, acc, true);
        }
        if (t == 0 || acc > best) best = acc;
    }
    return best;
}

// Gather one key row per active lane (tok >= 0) of this warp into shared memory.
template <typename T, int D>
__device__ __forceinline__ void stage_rows(const hp_stage_args& a, int kv, int64_t tok,
                                           unsigned char* ks, int stride, int lane) {
    const int eb = sizeof(T);
    const char* p = tok >= 0 ? kv_row_ptr(a.keys, a.keys.k_pool, a.keys.k_host, kv, tok, eb) : nullptr;
    const unsigned long long pu = reinterpret_cast<unsigned long long>(p);
    if constexpr (D == 128) {
        constexpr int kSegs = D * static_cast<int>(sizeof(T)) / 16;  // 16 (bf16) or 32 (fp32)
        constexpr int kRpi = 32 / kSegs;                             // rows per instruction
        const int seg = lane % kSegs, sub = lane / kSegs;
#pragma unroll 4
        for (int r = 0; r < 32; r += kRpi) {
            const int src = r + sub;
            const unsigned long long pp = __shfl_sync(0xffffffffu, pu, src);
            if (pp) cp_async16(ks + src * stride + seg * 16,
                               reinterpret_cast<const char*>(pp) + seg * 16);
        }
        cp_async_wait_all();
    } else {
        const int d = a.keys.d;
        for (int r = 0; r < 32; ++r) {
            const unsigned long long pp = __shfl_sync(0xffffffffu, pu, r);
            if (pp) {
                const T* src = reinterpret_cast<const T*>(pp);
                T* dst = reinterpret_cast<T*>(ks + r * stride);
                for (int e = lane; e < d; e += 32) dst[e] = src[e];
            }
        }
    }
    __syncwarp();
}

template <typename T, int D, bool EXT>
__global__ void __launch_bounds__(256) prune_descent_kernel(const hp_stage_args a, float* scores,
                                                            int max_chunks, StageGeom g) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int d = D ? D : a.keys.d;
    const int hpm = a.heads_per_mask;
    const int mb = blockIdx.y;
    const int m = mb / a.n_blocks, b = mb % a.n_blocks;
    const int64_t n_in = a.in_count[mb];
    const int lc = a.chunk_size;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int64_t keep_chunks = a.keep / lc;
    if (!a.descend_always && (n_in <= a.keep || cc <= keep_chunks)) return;  // identity (pruning.cpp:159-168)
    const int64_t chunk0 = static_cast<int64_t>(blockIdx.x) * 32 * g.cg;
    if (chunk0 >= cc) return;

    const int r0 = b * a.query_block;
    const int rows = min(a.query_block, a.q_rows - r0);
    float* qs = reinterpret_cast<float*>(smem);
    float* red = reinterpret_cast<float*>(smem + g.q_bytes);
    unsigned char* keys = smem + g.q_bytes + g.red_bytes;

    // rotate_queries (pruning.cpp:39-52): once per stage per head.
    bool q_safe = true;
    for (int i = threadIdx.x; i < hpm * rows * d; i += blockDim.x) {
        const int hh = i / (rows * d), rem = i - hh * rows * d, t = rem / d, e = rem - t * d;
        const float x = a.q[(static_cast<int64_t>(m * hpm + hh) * a.q_rows + r0 + t) * d + e];
        qs[(hh * g.rows_max + t) * d + e] = x;
        q_safe &= q_product_safe(x);
    }
    const bool all_safe = __syncthreads_and(q_safe);
    // exact-product fast path: q rows re-packed as bf16 pairs over the fp32 copy
    // ([head][row][64] words; the fp32 rows are not read again on this path)
    const bool use_fma = !EXT && D == 128 && sizeof(T) == 2 && all_safe && a.keys_exact != nullptr &&
                         *a.keys_exact != 0;
    uint32_t* qb = reinterpret_cast<uint32_t*>(qs);
    if (use_fma) {
        for (int i = threadIdx.x; i < hpm * rows * 64; i += blockDim.x) {
            const int hh = i / (rows * 64), rem = i - hh * rows * 64, t = rem >> 6, e = rem & 63;
            const float2 x = *reinterpret_cast<const float2*>(
                a.q + (static_cast<int64_t>(m * hpm + hh) * a.q_rows + r0 + t) * 128 + 2 * e);
            qb[(hh * g.rows_max + t) * 64 + e] = (__float_as_uint(x.x) >> 16) | (__float_as_uint(x.y) & 0xffff0000u);
        }
    }
    __syncthreads();
    if constexpr (EXT) {
        const int half = d >> 1;
        for (int i = threadIdx.x; i < hpm * rows * half; i += blockDim.x) {
            const int hh = i / (rows * half), rem = i - hh * rows * half, t = rem / half,
                      e = rem - t * half;
            const int64_t pos = rope_q_position(a.rope, a.query_offset + r0 + t, a.stream_tokens, cc);
            float* row = qs + (hh * g.rows_max + t) * d;
            const float c = a.rope.cos_tab[pos * half + e], s = a.rope.sin_tab[pos * half + e];
            const float x = row[e], y = row[e + half];
            row[e] = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, s));
            row[e + half] = __fadd_rn(__fmul_rn(x, s), __fmul_rn(y, c));
        }
        __syncthreads();
    }

    const int lane = threadIdx.x & 31, w = warp_id();
    const int n_warps = blockDim.x >> 5;
    unsigned char* ks = keys + static_cast<size_t>(w) * 32 * g.key_stride;
    unsigned char* myrow = ks + lane * g.key_stride;
    // work items (head hh, chunk group grp), looped when hpm * cg exceeds the CTA's warps
    for (int item = w; item < hpm * g.cg; item += n_warps) {
    const int hh = item % hpm, grp = item / hpm;
    const int qh = m * hpm + hh;
    const int kv = qh / (a.n_q_heads / a.keys.n_kv);
    const float* qrows = qs + hh * g.rows_max * d;
    const uint32_t* qbrows = qb + hh * g.rows_max * 64;

    const int64_t j = chunk0 + grp * 32 + lane;
    const bool active = j < cc;
    const int64_t base = j * lc;
    const int len = active ? static_cast<int>(min64(lc, n_in - base)) : 0;
    // contiguous chunk => token(i) = first + i, no list reads during the descent
    int64_t t_first = active ? list_token(a, mb, base) : 0;
    bool contiguous = true;
    if (active && a.in_list && len > 1) contiguous = list_token(a, mb, base + len - 1) - t_first == len - 1;
    auto token = [&](int i) -> int64_t { return contiguous ? t_first + i : list_token(a, mb, base + i); };

    // key positions for the two branches (rope_policy.cpp:37-57)
    const float* cs1 = nullptr; const float* sn1 = nullptr;
    const float* cs2 = nullptr; const float* sn2 = nullptr;
    bool same_rot = true;
    if constexpr (EXT) {
        const int half = d >> 1;
        const int64_t p1 = rope_k_position(a.rope, 1, j), p2 = rope_k_position(a.rope, 2, j);
        cs1 = a.rope.cos_tab + p1 * half; sn1 = a.rope.sin_tab + p1 * half;
        cs2 = a.rope.cos_tab + p2 * half; sn2 = a.rope.sin_tab + p2 * half;
        same_rot = p1 == p2;
    }
    auto score2 = [&](float& s1, float& s2) {
        if constexpr (EXT) {
            s1 = block_score<T, D, true>(myrow, qrows, rows, d, cs1, sn1);
            s2 = same_rot ? s1 : block_score<T, D, true>(myrow, qrows, rows, d, cs2, sn2);
        } else if (use_fma) {
            if constexpr (D == 128 && sizeof(T) == 2) s1 = s2 = block_score_fma(myrow, qbrows, rows);
        } else {
            s1 = s2 = block_score<T, D, false>(myrow, qrows, rows, d, nullptr, nullptr);
        }
    };

    // state: [first,last] 1-based; s1/s2 = branch-1/branch-2 scores of chunk[first-1]
    int first = 1, last = len, it = 0;
    int iters = 0;
    while ((1 << iters) < len) ++iters;
    float s1 = 0.0f, s2 = 0.0f;
    uint32_t path = 0;  // branch decisions (bit it = went right)
    stage_rows<T, D>(a, kv, active ? token(0) : -1, ks, g.key_stride, lane);
    if (active) score2(s1, s2);
    for (;;) {
        const bool go = active && it < iters && first < last;
        if (!__any_sync(0xffffffffu, go)) break;
        const int mid = (first + last + 1) >> 1;
        __syncwarp();
        stage_rows<T, D>(a, kv, go ? token(mid - 1) : -1, ks, g.key_stride, lane);
        if (go) {
            float m1, m2;
            score2(m1, m2);
            if (m2 > s1) {  // right only on strict sigma2 > sigma1 (pruning.cpp:91)
                first = mid; s1 = m1; s2 = m2;
                path |= 1u << it;
            } else {
                last = mid - 1;
            }
            ++it;
        }
    }
    const int ch = grp * 32 + lane;
    red[hh * (32 * g.cg) + ch] = s2;  // branch-2 score of the representative (pruning.cpp:181)
    if (a.path_out && active) a.path_out[(static_cast<int64_t>(mb) * max_chunks + j) * hpm + hh] = path;
    __syncwarp();
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 32 * g.cg; c += blockDim.x) {
        const int64_t jj = chunk0 + c;
        if (jj >= cc) continue;
        float best = -__int_as_float(0x7f800000);
        for (int h = 0; h < hpm; ++h) {
            const float s = red[h * (32 * g.cg) + c];
            best = (best < s) ? s : best;  // std::max (pruning.cpp:182)
        }
        scores[static_cast<int64_t>(mb) * max_chunks + jj] = best;
    }
}

// Exact top-(k/l_c) chunk selection + ordered emission of the survivors.
__global__ void __launch_bounds__(kTopkThreads) prune_topk_kernel(const hp_stage_args a,
                                                                  const float* scores,
                                                                  int32_t* sel_ws, int max_chunks,
                                                                  int kmax, int* status) {
    const int mb = blockIdx.x;
    const int64_t n_in = a.in_count[mb];
    const int lc = a.chunk_size;
    int32_t* out = a.out_list + static_cast<int64_t>(mb) * a.out_stride;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int64_t K = a.keep / lc;
    if (n_in <= a.keep || cc <= K) {
        if (n_in > a.out_stride) {
            if (threadIdx.x == 0) { atomicOr(status, 2); a.out_count[mb] = -1; }
            return;
        }
        for (int64_t i = threadIdx.x; i < n_in; i += blockDim.x) out[i] = static_cast<int32_t>(list_token(a, mb, i));
        if (threadIdx.x == 0) a.out_count[mb] = static_cast<int32_t>(n_in);
        return;
    }
    if (cc > max_chunks || K > kmax) {
        if (threadIdx.x == 0) { atomicOr(status, 1); a.out_count[mb] = -1; }
        return;
    }
    const float* sc = scores + static_cast<int64_t>(mb) * max_chunks;
    int32_t* sel = sel_ws + static_cast<int64_t>(mb) * kmax;
    __shared__ int hist[256];
    __shared__ int scan_tmp[32];
    __shared__ uint32_t sh_digit;
    __shared__ int sh_above;

    // Radix select (MSB first) of the K-th largest order key.
    uint32_t prefix = 0, pmask = 0;
    int need = static_cast<int>(K);
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t jj = threadIdx.x; jj < cc; jj += blockDim.x) {
            const uint32_t u = order_key(sc[jj]);
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int c[8], tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { c[k] = hist[lane * 8 + k]; tot += c[k]; }
            // exclusive suffix sum of lane totals (counts of digits above this lane's range)
            int suf = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += y;
            }
            int above = suf - tot;
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                if (above < need && need <= above + c[k]) { sh_digit = lane * 8 + k; sh_above = above; }
                above += c[k];
            }
        }
        __syncthreads();
        prefix |= sh_digit << shift;
        pmask |= 255u << shift;
        need -= sh_above;
        __syncthreads();
    }
    // Select: keys above the threshold, plus the first `need` ties by chunk index.
    int tie_base = 0, sel_base = 0;
    for (int64_t tile = 0; tile < cc; tile += blockDim.x) {
        const int64_t jj = tile + threadIdx.x;
        const bool in = jj < cc;
        const uint32_t u = in ? order_key(sc[jj]) : 0u;
        const int is_tie = in && u == prefix;
        const int is_gt = in && u > prefix;
        int tie_tot, s_tot;
        const int tie_rank = block_exclusive_scan<kTopkThreads>(is_tie, scan_tmp, &tie_tot) + tie_base;
        const int s = is_gt || (is_tie && tie_rank < need);
        const int r = block_exclusive_scan<kTopkThreads>(s, scan_tmp, &s_tot) + sel_base;
        if (s) sel[r] = static_cast<int32_t>(jj);
        tie_base += tie_tot;
        sel_base += s_tot;
    }
    __syncthreads();
    // Survivors in original order: chunk r of the kept set lands at r * l_c (only the
    // final chunk of the list can be short, and it is last in ascending order).
    for (int64_t o = threadIdx.x; o < K * lc; o += blockDim.x) {
        const int64_t r = o / lc, i = o - r * lc;
        const int64_t jj = sel[r];
        const int64_t len = min64(lc, n_in - jj * lc);
        if (i < len) out[o] = static_cast<int32_t>(list_token(a, mb, jj * lc + i));
    }
    if (threadIdx.x == 0) {
        const int64_t last = sel[K - 1];
        a.out_count[mb] = static_cast<int32_t>((K - 1) * lc + min64(lc, n_in - last * lc));
    }
}

__global__ void remap_kernel(const int32_t* in_list, const int32_t* in_count, int64_t in_stride,
                             int n_blocks, int next_blocks, int bq_next, int ratio, int t_q,
                             int64_t offset, int stream, int32_t* out_list, int32_t* out_count,
                             int64_t out_stride) {
    __shared__ int scan_tmp[32];
    const int mb2 = blockIdx.x;
    const int m = mb2 / next_blocks, m2 = mb2 % next_blocks;
    const int parent = min(m2 / ratio, n_blocks - 1);
    const int64_t end = offset + min(static_cast<int64_t>(m2 + 1) * bq_next, static_cast<int64_t>(t_q));
    const int64_t upper = end > stream ? end - stream : 0;
    const int32_t* src = in_list + (static_cast<int64_t>(m) * n_blocks + parent) * in_stride;
    const int n = in_count[m * n_blocks + parent];
    int32_t* dst = out_list + static_cast<int64_t>(mb2) * out_stride;
    int base = 0;
    for (int tile = 0; tile < n; tile += blockDim.x) {
        const int i = tile + threadIdx.x;
        const int keep = i < n && src[i] < upper;
        int tot;
        const int r = block_exclusive_scan<256>(keep, scan_tmp, &tot) + base;
        if (keep) dst[r] = src[i];
        base += tot;
    }
    if (threadIdx.x == 0) out_count[mb2] = base;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" size_t hp_stage_workspace_bytes(int32_t n_lists, int32_t max_chunks, int32_t keep,
                                           int32_t chunk_size) {
    const size_t kmax = chunk_size > 0 ? static_cast<size_t>(keep / chunk_size) : 0;
    return align_up(static_cast<size_t>(n_lists) * max_chunks * 4, 256) +
           align_up(static_cast<size_t>(n_lists) * (kmax ? kmax : 1) * 4, 256) + 256;
}

template <typename T, int D, bool EXT>
static cudaError_t launch_descent(const hp_stage_args& a, float* scores, const StageGeom& g,
                                  cudaStream_t s) {
    auto kern = prune_descent_kernel<T, D, EXT>;
    const size_t smem = g.q_bytes + g.red_bytes + g.key_bytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid((a.max_chunks + 32 * g.cg - 1) / (32 * g.cg), a.n_masks * a.n_blocks);
    dim3 block(32 * std::min(8, g.cg * a.heads_per_mask));
    kern<<<grid, block, smem, s>>>(a, scores, a.max_chunks, g);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch_descent(const hp_stage_args& a, float* scores, const StageGeom& g,
                                    cudaStream_t s) {
    const bool ext = a.rope.extension != 0;
    if (a.keys.d == 128) return ext ? launch_descent<T, 128, true>(a, scores, g, s)
                                    : launch_descent<T, 128, false>(a, scores, g, s);
    return ext ? launch_descent<T, 0, true>(a, scores, g, s) : launch_descent<T, 0, false>(a, scores, g, s);
}

extern "C" int hp_prune_stage(const hp_stage_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: null args");
    const hp_stage_args& a = *ap;
    // StageConfig::validate (pruning.cpp:102-109)
    if (a.query_block <= 0 || a.chunk_size <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: b_q and l_c must be >= 1");
    if (a.keep <= 0 || a.keep % a.chunk_size != 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: k must be a positive multiple of l_c");
    if (a.n_masks <= 0 || a.heads_per_mask <= 0 || a.n_blocks <= 0 || a.q_rows <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: empty batch geometry");
    if (a.n_q_heads != a.n_masks * a.heads_per_mask)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: n_q_heads != n_masks * heads_per_mask");
    if (a.keys.n_kv <= 0 || a.n_q_heads % a.keys.n_kv != 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: n_q_heads must be a multiple of n_kv");
    if (a.heads_per_mask > 32) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: heads_per_mask > 32");
    if (a.keys.d <= 0 || a.keys.d > 1024) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: head_dim out of range");
    if (a.keys.dtype != HP_F32 && a.keys.dtype != HP_BF16) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: dtype");
    if (!a.q || !a.in_count || (!a.in_list && !a.in_start) || !a.out_list || !a.out_count || !a.keys.k_pool)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: null pointer");
    if (a.max_chunks < 0) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: max_chunks < 0");
    const int n_lists = a.n_masks * a.n_blocks;
    const int max_chunks = a.max_chunks > 0 ? a.max_chunks : 1;
    const size_t need = hp_stage_workspace_bytes(n_lists, max_chunks, a.keep, a.chunk_size);
    if (!a.workspace || a.workspace_bytes < need)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: workspace too small (%zu < %zu)", a.workspace_bytes, need);
    if (a.rope.extension) {
        const int pol_e = a.rope.early_policy, pol_l = a.rope.late_policy;
        const int pol = a.rope.layer > a.rope.early_cutoff ? pol_l : pol_e;
        if (pol != HP_ROPE_CHUNK_INDEXED && pol != HP_ROPE_RELATIVE)
            return hph::set_error(HP_LOGIC_ERROR, "query_position: policy not applicable to pruning");
        if (a.keys.d % 2) return hph::set_error(HP_INVALID_ARGUMENT, "apply_rope: head_dim must be even");
        if (!a.rope.cos_tab || !a.rope.sin_tab) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: rope table missing");
        const int64_t qpos_max = a.query_offset + a.q_rows - 1;
        const int64_t need_q = pol == HP_ROPE_RELATIVE ? a.stream_tokens + 1
                                                       : min64(qpos_max, max_chunks + a.stream_tokens);
        const int64_t need_k = pol == HP_ROPE_RELATIVE ? 1 : max_chunks - 1;
        const int64_t p = std::max(need_q, need_k);
        if (p >= a.rope.rope_max)
            return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                                  static_cast<long long>(p), static_cast<long long>(a.rope.rope_max));
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* ws = static_cast<char*>(a.workspace);
    float* scores = reinterpret_cast<float*>(ws);
    const int kmax = a.keep / a.chunk_size;
    int32_t* sel = reinterpret_cast<int32_t*>(ws + align_up(static_cast<size_t>(n_lists) * max_chunks * 4, 256));
    int* status = reinterpret_cast<int*>(ws + need - 256);

    hp_stage_args la = a;
    la.max_chunks = max_chunks;
    if (a.max_chunks > 0) {
        StageGeom g{};
        const int eb = a.keys.dtype == HP_BF16 ? 2 : 4;
        g.rows_max = std::min(a.query_block, a.q_rows);
        g.key_stride = static_cast<int>(align_up(static_cast<size_t>(a.keys.d) * eb, 16) + 16);
        g.cg = std::max(1, 8 / a.heads_per_mask);
        for (;;) {
            g.q_bytes = align_up(static_cast<size_t>(a.heads_per_mask) * g.rows_max * a.keys.d * 4, 16);
            g.red_bytes = align_up(static_cast<size_t>(a.heads_per_mask) * 32 * g.cg * 4, 16);
            g.key_bytes = static_cast<size_t>(std::min(8, a.heads_per_mask * g.cg)) * 32 * g.key_stride;
            if (g.q_bytes + g.red_bytes + g.key_bytes <= 220 * 1024 || g.cg == 1) break;
            g.cg = std::max(1, g.cg / 2);
        }
        if (g.q_bytes + g.red_bytes + g.key_bytes > 227 * 1024)
            return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage: query block x heads too large for shared memory");
        const cudaError_t e = a.keys.dtype == HP_BF16 ? dispatch_descent<bf16_t>(la, scores, g, s)
                                                      : dispatch_descent<float>(la, scores, g, s);
        if (int rc = hph::check_cuda(e, "prune_descent_kernel")) return rc;
    }
    prune_topk_kernel<<<n_lists, kTopkThreads, 0, s>>>(la, scores, sel, max_chunks, kmax, status);
    return hph::check_cuda(cudaGetLastError(), "prune_topk_kernel");
}

extern "C" int hp_remap_blocks(const int32_t* in_list, const int32_t* in_count, int64_t in_stride,
                               int32_t n_masks, int32_t n_blocks, int32_t bq, int32_t bq_next,
                               int32_t t_q, int64_t query_offset, int32_t stream_tokens,
                               int32_t* out_list, int32_t* out_count, int64_t out_stride,
                               void* stream) {
    if (bq_next <= 0 || bq % bq_next != 0 || n_blocks <= 0 || n_masks <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "PruningPlan: successive b_q must be non-increasing and divisible");
    const int next_blocks = (t_q + bq_next - 1) / bq_next;
    remap_kernel<<<n_masks * next_blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        in_list, in_count, in_stride, n_blocks, next_blocks, bq_next, bq / bq_next, t_q,
        query_offset, stream_tokens, out_list, out_count, out_stride);
    return hph::check_cuda(cudaGetLastError(), "remap_kernel");
}

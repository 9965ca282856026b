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
#include <cstdlib>

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

// ---------------------------------------------------------------- tensor-core descent
// Query-block stages (prefill, b_q rows >= 16) with bf16 keys certified exact-product
// (keys_exact) and bf16-exact q: the descent's row scores are computed on the tensor
// cores (mma.sync m16n8k16, bf16 in, fp32 accumulate: a warp scores its 32 key rows
// against the block's q rows as one 32 x 128 x 64 product, σ = max over the rows), each
// with a certified bound on its distance from the reference's sequential fp32 value:
//   |σ_tc - σ_ref| <= E = 2^-15 · max_r ||q_r|| · ||k||
// (the sequential 128-term fp32 sum is within ~2^-17 Σ|q_i k_i| of the exact dot, the
// tensor-core sum measured within 2^-19.8 of it, scripts/mma_check.cu; Σ|q_i k_i| <=
// ||q|| ||k||). A descent comparison σ2 > σ1 whose operands are not separated by their
// bounds is re-decided on the exact values (the reference's sequential fp32 dots, FHFMA,
// the whole warp on one row), so every branch decision is the reference's. The chunk
// keys (max over the heads, order keys, atomicMax) stay approximate with the list's
// bound; prune_topk_kernel keeps the chunks certainly above the K-th key, drops those
// certainly below, and scores the representatives of the few in between exactly (the
// descent records each head's representative) (pruning.cpp:69-98,170-192). One CTA per
// (mask-block, head, 256 chunks).
constexpr int kTcRow = 272;                   // padded bf16 row (ldmatrix rows hit distinct banks)
constexpr int kTcWarps = 8;
constexpr int kTcQBytes = 64 * 128 * 4;       // fp32 q rows (fallback) or padded bf16 q rows
constexpr size_t kTcSmem = kTcQBytes + static_cast<size_t>(kTcWarps) * 32 * kTcRow;
constexpr float kTcBound = 1.0f / 32768.0f;   // 2^-15
constexpr int kTcMaxHeads = 8;                // heads per mask on this path (rep offsets per chunk)

__device__ __forceinline__ void ldsm_x4(uint32_t* r, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Approximate σ of this lane's staged row (warp rows at ks, q rows at qa, both kTcRow
// apart): keys are the A operand (2 m-tiles of 16), q rows the B operand (n-tiles of 8).
__device__ __forceinline__ float tc_sigma(uint32_t ks, uint32_t qa, int rows, int lane) {
    const int tq = lane & 3, mi = lane >> 3, r8 = lane & 7;
    float mx[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
    uint32_t a[2][8][4];  // both m-tiles' A fragments: every B fragment feeds two MMAs
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int k = 0; k < 8; ++k)
            ldsm_x4(a[mt][k], ks + (mt * 16 + (mi & 1) * 8 + r8) * kTcRow + (k * 16 + (mi >> 1) * 8) * 2);
#pragma unroll 1
    for (int nt = 0; nt * 8 < rows; ++nt) {
        float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
            uint32_t b[4];
            ldsm_x4(b, qa + (nt * 8 + r8) * kTcRow + ((2 * kp + (mi >> 1)) * 16 + (mi & 1) * 8) * 2);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                mma16816(c[mt], a[mt][2 * kp], b[0], b[1]);
                mma16816(c[mt], a[mt][2 * kp + 1], b[2], b[3]);
            }
        }
        const bool v0 = nt * 8 + 2 * tq < rows, v1 = nt * 8 + 2 * tq + 1 < rows;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            mx[mt][0] = fmaxf(mx[mt][0], fmaxf(v0 ? c[mt][0] : -INFINITY, v1 ? c[mt][1] : -INFINITY));
            mx[mt][1] = fmaxf(mx[mt][1], fmaxf(v0 ? c[mt][2] : -INFINITY, v1 ? c[mt][3] : -INFINITY));
        }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            mx[mt][h] = fmaxf(mx[mt][h], __shfl_xor_sync(0xffffffffu, mx[mt][h], 1));
            mx[mt][h] = fmaxf(mx[mt][h], __shfl_xor_sync(0xffffffffu, mx[mt][h], 2));
        }
    // key L = mt * 16 + h * 8 + g lives in lanes 4g..4g+3
    const int src = (lane & 7) * 4;
    const float x00 = __shfl_sync(0xffffffffu, mx[0][0], src), x01 = __shfl_sync(0xffffffffu, mx[0][1], src);
    const float x10 = __shfl_sync(0xffffffffu, mx[1][0], src), x11 = __shfl_sync(0xffffffffu, mx[1][1], src);
    const int mt = lane >> 4, h = (lane >> 3) & 1;
    return mt ? (h ? x11 : x10) : (h ? x01 : x00);
}

// Exact σ of one key row (any address space) by the whole warp: lane l runs the
// reference's sequential dots of q rows l and l + 32 (FHFMA, exact products).
__device__ __noinline__ float exact_sigma_warp(const unsigned char* krow, const uint32_t* qw, int rows, int lane) {
    const uint4* k4 = reinterpret_cast<const uint4*>(krow);
    const bool h0 = lane < rows, h1 = lane + 32 < rows;
    const uint4* q0 = reinterpret_cast<const uint4*>(qw + lane * (kTcRow / 4));
    const uint4* q1 = reinterpret_cast<const uint4*>(qw + (h1 ? lane + 32 : lane) * (kTcRow / 4));
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
        const uint4 k = k4[c], x = q0[c], y = q1[c];
        a0 = fma_bf16(x.x, k.x, a0, false); a0 = fma_bf16(x.x, k.x, a0, true);
        a1 = fma_bf16(y.x, k.x, a1, false); a1 = fma_bf16(y.x, k.x, a1, true);
        a0 = fma_bf16(x.y, k.y, a0, false); a0 = fma_bf16(x.y, k.y, a0, true);
        a1 = fma_bf16(y.y, k.y, a1, false); a1 = fma_bf16(y.y, k.y, a1, true);
        a0 = fma_bf16(x.z, k.z, a0, false); a0 = fma_bf16(x.z, k.z, a0, true);
        a1 = fma_bf16(y.z, k.z, a1, false); a1 = fma_bf16(y.z, k.z, a1, true);
        a0 = fma_bf16(x.w, k.w, a0, false); a0 = fma_bf16(x.w, k.w, a0, true);
        a1 = fma_bf16(y.w, k.w, a1, false); a1 = fma_bf16(y.w, k.w, a1, true);
    }
    // σ = the largest row dot (the value the reference's strict-'>' scan keeps; the sign
    // of a zero maximum never changes a comparison or an order key)
    float v = h0 ? a0 : -INFINITY;
    if (h1) v = fmaxf(v, a1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// the separately rounded fp32 path (q not bf16-exact or keys not certified), kept out of
// line so the tensor-core path's registers are not sized for it
__device__ __noinline__ float block_score_bf16_call(const unsigned char* krow, const float* qf, int rows) {
    const uint32_t* k = reinterpret_cast<const uint32_t*>(krow);
    float best = 0.0f;
#pragma unroll 1
    for (int t = 0; t < rows; ++t) {
        float acc = 0.0f;
#pragma unroll 4
        for (int i = 0; i < 64; ++i) {
            const uint32_t w = k[i];
            acc = __fadd_rn(acc, __fmul_rn(qf[t * 128 + 2 * i], bf16_lo(w)));
            acc = __fadd_rn(acc, __fmul_rn(qf[t * 128 + 2 * i + 1], bf16_hi(w)));
        }
        if (t == 0 || acc > best) best = acc;
    }
    return best;
}

// ||k|| of this lane's staged bf16 row, rounded up
__device__ __forceinline__ float row_norm_up(const unsigned char* krow) {
    const uint4* k4 = reinterpret_cast<const uint4*>(krow);
    float s = 0.f;
#pragma unroll 2
    for (int c = 0; c < 16; ++c) {
        const uint4 w = k4[c];
        s = fmaf(bf16_lo(w.x), bf16_lo(w.x), s); s = fmaf(bf16_hi(w.x), bf16_hi(w.x), s);
        s = fmaf(bf16_lo(w.y), bf16_lo(w.y), s); s = fmaf(bf16_hi(w.y), bf16_hi(w.y), s);
        s = fmaf(bf16_lo(w.z), bf16_lo(w.z), s); s = fmaf(bf16_hi(w.z), bf16_hi(w.z), s);
        s = fmaf(bf16_lo(w.w), bf16_lo(w.w), s); s = fmaf(bf16_hi(w.w), bf16_hi(w.w), s);
    }
    return sqrtf(s * 1.0001f) * 1.0001f;
}

__global__ void __launch_bounds__(kTcWarps * 32, 2) prune_descent_tc_kernel(const hp_stage_args a, uint32_t* keys_out,
                                                                          uint32_t* list_bound, uint16_t* rep_out,
                                                                          int max_chunks) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int hpm = a.heads_per_mask;
    const int mb = blockIdx.z, hh = blockIdx.y;
    const int m = mb / a.n_blocks, b = mb % a.n_blocks;
    const int64_t n_in = a.in_count[mb];
    const int lc = a.chunk_size;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int64_t keep_chunks = a.keep / lc;
    if (!a.descend_always && (n_in <= a.keep || cc <= keep_chunks)) return;  // identity (pruning.cpp:159-168)
    const int64_t chunk0 = static_cast<int64_t>(blockIdx.x) * 32 * kTcWarps;
    if (chunk0 >= cc) return;
    const int r0 = b * a.query_block;
    const int rows = min(a.query_block, a.q_rows - r0);
    const int qh = m * hpm + hh;
    const int kv = qh / (a.n_q_heads / a.keys.n_kv);
    const float* qg = a.q + (static_cast<int64_t>(qh) * a.q_rows + r0) * 128;

    // q: exact-product safe -> padded bf16 rows (B operand + exact dots); else fp32 rows
    bool safe = true;
    for (int i = threadIdx.x; i < rows * 128; i += blockDim.x) safe &= q_product_safe(qg[i]);
    const bool use_fma = __syncthreads_and(safe) && a.keys_exact != nullptr && *a.keys_exact != 0;
    uint32_t* qw = reinterpret_cast<uint32_t*>(smem);
    float* qf = reinterpret_cast<float*>(smem);
    __shared__ float sh_qn;
    if (use_fma) {
        for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
            const int t = i >> 6, e = i & 63;
            uint32_t wv = 0u;
            if (t < rows) {
                const float2 x = *reinterpret_cast<const float2*>(qg + t * 128 + 2 * e);
                wv = (__float_as_uint(x.x) >> 16) | (__float_as_uint(x.y) & 0xffff0000u);
            }
            qw[t * (kTcRow / 4) + e] = wv;  // rows >= rows are zero (masked from the max)
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // max_r ||q_r||, rounded up
            float nmax = 0.f;
            for (int t = threadIdx.x; t < rows; t += 32) {
                float s = 0.f;
#pragma unroll 4
                for (int e = 0; e < 64; ++e) {
                    const uint32_t x = qw[t * (kTcRow / 4) + ((e + t) & 63)];  // rotated: no bank conflicts
                    s = fmaf(bf16_lo(x), bf16_lo(x), s);
                    s = fmaf(bf16_hi(x), bf16_hi(x), s);
                }
                nmax = fmaxf(nmax, s);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
            if (threadIdx.x == 0) sh_qn = sqrtf(nmax * 1.0001f) * 1.0001f;
        }
    } else {
        for (int i = threadIdx.x; i < rows * 128; i += blockDim.x) qf[i] = qg[i];
    }
    __syncthreads();
    const float qn = use_fma ? sh_qn : 0.f;

    const int lane = threadIdx.x & 31, w = warp_id();
    unsigned char* ks = smem + kTcQBytes + static_cast<size_t>(w) * 32 * kTcRow;
    unsigned char* myrow = ks + lane * kTcRow;
    const uint32_t ks_a = smem_u32(ks), q_a = smem_u32(qw);

    const int64_t j = chunk0 + w * 32 + lane;
    const bool active = j < cc;
    const int64_t base = j * lc;
    const int len = active ? static_cast<int>(min64(lc, n_in - base)) : 0;
    int64_t t_first = active ? list_token(a, mb, base) : 0;
    bool contiguous = true;
    if (active && a.in_list && len > 1) contiguous = list_token(a, mb, base + len - 1) - t_first == len - 1;
    auto token = [&](int i) -> int64_t { return contiguous ? t_first + i : list_token(a, mb, base + i); };

    // gather this lane's row (tok >= 0) into the warp's staging; returns its address
    auto stage = [&](int64_t tok) -> const char* {
        const char* p = tok >= 0 ? kv_row_ptr(a.keys, a.keys.k_pool, a.keys.k_host, kv, tok, 2) : nullptr;
        const unsigned long long pu = reinterpret_cast<unsigned long long>(p);
        const int seg = lane & 15, sub = lane >> 4;
#pragma unroll 4
        for (int r = 0; r < 32; r += 2) {
            const unsigned long long pp = __shfl_sync(0xffffffffu, pu, r + sub);
            if (pp) cp_async16(ks + (r + sub) * kTcRow + seg * 16, reinterpret_cast<const char*>(pp) + seg * 16);
        }
        cp_async_wait_all();
        __syncwarp();
        return p;
    };
    // (σ, bound) of the staged rows: tensor cores + bound, or exact per lane
    auto score = [&](float& s, float& e) {
        if (use_fma) {
            s = tc_sigma(ks_a, q_a, rows, lane);
            e = kTcBound * qn * row_norm_up(myrow);
        } else {
            s = block_score_bf16_call(myrow, qf, rows);
            e = 0.f;
        }
    };

    int first = 1, last = len, it = 0;
    int iters = 0;
    while ((1 << iters) < len) ++iters;
    float s1 = 0.f, e1 = 0.f;
    uint32_t path = 0;
    const char* rep = stage(active ? token(0) : -1);
    score(s1, e1);
    for (;;) {
        const bool go = active && it < iters && first < last;
        if (!__any_sync(0xffffffffu, go)) break;
        const int mid = (first + last + 1) >> 1;
        __syncwarp();
        const char* p = stage(go ? token(mid - 1) : -1);
        float m2, em;
        score(m2, em);
        bool right = false, amb = false;
        if (go) {
            const float tol = (e1 + em) * 1.01f;
            if (tol == 0.f) right = m2 > s1;
            else if (m2 - s1 > tol) right = true;
            else if (!(s1 - m2 >= tol)) amb = true;
        }
        // undecided comparisons: the exact operands, one lane at a time (rare)
        for (unsigned am = __ballot_sync(0xffffffffu, amb); am; am &= am - 1) {
            const int L = __ffs(am) - 1;
            const float mx = exact_sigma_warp(ks + L * kTcRow, qw, rows, lane);
            const float e1L = __shfl_sync(0xffffffffu, e1, L);
            float sx = __shfl_sync(0xffffffffu, s1, L);
            const unsigned long long rL = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rep), L);
            if (e1L != 0.f) sx = exact_sigma_warp(reinterpret_cast<const unsigned char*>(rL), qw, rows, lane);
            if (lane == L) { m2 = mx; em = 0.f; s1 = sx; e1 = 0.f; right = m2 > s1; }
        }
        if (go) {
            if (right) {  // right only on strict σ2 > σ1 (pruning.cpp:91)
                first = mid; s1 = m2; e1 = em; rep = p;
                path |= 1u << it;
            } else {
                last = mid - 1;
            }
            ++it;
        }
    }
    // approximate chunk key (max over the heads) and the list's bound; prune_topk_kernel
    // certifies the kept set and rescores the chunks near its boundary exactly
    if (active) {
        atomicMax(keys_out + static_cast<int64_t>(mb) * max_chunks + j, order_key(s1));  // max over heads (pruning.cpp:182)
        rep_out[(static_cast<int64_t>(mb) * max_chunks + j) * kTcMaxHeads + hh] = static_cast<uint16_t>(first - 1);
        if (a.path_out) a.path_out[(static_cast<int64_t>(mb) * max_chunks + j) * hpm + hh] = path;
    }
    float eb = active ? e1 : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eb = fmaxf(eb, __shfl_xor_sync(0xffffffffu, eb, o));
    if (lane == 0 && eb > 0.f) atomicMax(list_bound + 2 * mb, __float_as_uint(eb));  // non-negative floats order as ints
    if (threadIdx.x == 0 && !use_fma) atomicOr(list_bound + 2 * mb + 1, 1u << hh);  // this head's dots are fp32-rounded
}


// Exact σ of one key row (bf16) with q rows read from global fp32: lane l runs the
// reference's sequential dots of rows l and l + 32 (FHFMA when q is bf16-exact and the
// products exact, else separately rounded), σ = the largest.
__device__ __noinline__ float exact_sigma_gq(const unsigned char* krow, const float* q, int rows, int lane, bool fma) {
    const uint4* k4 = reinterpret_cast<const uint4*>(krow);
    const bool h0 = lane < rows, h1 = lane + 32 < rows;
    const float4* q0 = reinterpret_cast<const float4*>(q + (h0 ? lane : 0) * 128);
    const float4* q1 = reinterpret_cast<const float4*>(q + (h1 ? lane + 32 : 0) * 128);
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 2
    for (int c = 0; c < 16; ++c) {
        const uint4 k = k4[c];
        const float4 x0 = q0[2 * c], x1 = q0[2 * c + 1], y0 = q1[2 * c], y1 = q1[2 * c + 1];
        const uint32_t kw[4] = {k.x, k.y, k.z, k.w};
        const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const float ys[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t kk = kw[e >> 1];
            if (fma) {  // exact products: one rounding per element, as the reference's fl(acc + fl(q k))
                const uint32_t xq = __float_as_uint(xs[e]) >> 16, yq = __float_as_uint(ys[e]) >> 16;
                a0 = fma_bf16(xq, kk >> ((e & 1) * 16), a0, false);
                a1 = fma_bf16(yq, kk >> ((e & 1) * 16), a1, false);
            } else {
                const float kf = (e & 1) ? bf16_hi(kk) : bf16_lo(kk);
                a0 = __fadd_rn(a0, __fmul_rn(xs[e], kf));
                a1 = __fadd_rn(a1, __fmul_rn(ys[e], kf));
            }
        }
    }
    float v = h0 ? a0 : -INFINITY;
    if (h1) v = fmaxf(v, a1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float key_to_float(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}


// Settle the approximate chunk keys of one list around the approximate K-th value T:
// keys more than `band` above T are certainly kept (their exact score exceeds the exact
// K-th), keys more than `band` below certainly dropped; the chunks in between have every
// head's representative (recorded by the descent, whose branch decisions are exact)
// scored with exact dots (rare: the band is ~1e-4 of the score scale) and take their
// exact key. Kept / dropped become the extreme keys so the second select
// returns exactly the reference's set (pruning.cpp:170-192).
__device__ void refine_band(const hp_stage_args& a, int mb, float* scw, int64_t cc, float T, float band,
                            uint32_t fallback_heads, const uint16_t* reps, int max_chunks, int* scan_tmp) {
    uint32_t* kw = reinterpret_cast<uint32_t*>(scw);
    __shared__ int idx[kTopkThreads];
    __shared__ uint32_t xkey[kTopkThreads];
    const int hpm = a.heads_per_mask, m = mb / a.n_blocks, b = mb % a.n_blocks;
    const int r0 = b * a.query_block, rows = min(a.query_block, a.q_rows - r0);
    const int lane = threadIdx.x & 31, w = warp_id(), nw = blockDim.x >> 5;
    const int lc = a.chunk_size;
    for (int64_t tile = 0; tile < cc; tile += blockDim.x) {
        const int64_t jj = tile + threadIdx.x;
        int is_band = 0;
        if (jj < cc) {
            const float v = key_to_float(kw[jj]);
            if (v - T > band) kw[jj] = 0xffffffffu;
            else if (T - v > band) kw[jj] = 0u;
            else is_band = 1;
        }
        int n_band;
        const int r = block_exclusive_scan<kTopkThreads>(is_band, scan_tmp, &n_band);
        if (is_band) { idx[r] = static_cast<int>(jj); xkey[r] = 0u; }
        __syncthreads();
        for (int task = w; task < n_band * hpm; task += nw) {  // (chunk, head) descents, one per warp
            const int e = task / hpm, h = task - e * hpm;
            const int64_t j = idx[e], base = j * lc;
            const int qh = m * hpm + h;
            const int kv = qh / (a.n_q_heads / a.keys.n_kv);
            const bool fb = fallback_heads >> h & 1u;
            const float* qg = a.q + (static_cast<int64_t>(qh) * a.q_rows + r0) * 128;  // L1-resident after the first row
            auto sigma = [&](int i) {
                const unsigned char* row = reinterpret_cast<const unsigned char*>(
                    kv_row_ptr(a.keys, a.keys.k_pool, a.keys.k_host, kv, list_token(a, mb, base + i), 2));
                return exact_sigma_gq(row, qg, rows, lane, !fb);
            };
            // the representative's exact score (its branch decisions were already exact)
            const float s1 = sigma(reps[(static_cast<int64_t>(mb) * max_chunks + j) * kTcMaxHeads + h]);
            if (lane == 0) atomicMax(&xkey[e], order_key(s1));  // max over heads (pruning.cpp:182)
        }
        __syncthreads();
        if (is_band) kw[jj] = xkey[r];
        __syncthreads();
    }
}

// Exact top-(k/l_c) chunk selection + ordered emission of the survivors.
__global__ void __launch_bounds__(kTopkThreads, 2) prune_topk_kernel(const hp_stage_args a,
                                                                  const float* scores,
                                                                  int32_t* sel_ws, int max_chunks,
                                                                  int kmax, int* status, bool keyed,
                                                                  const uint32_t* list_bound, const uint16_t* reps) {
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

    // keys from the tensor-core descent are approximate within the list's bound: the first
    // pass finds the approximate K-th key, the chunks that bound cannot settle are rescored
    // exactly, and the second pass selects on settled keys
    const float bound = list_bound ? __uint_as_float(list_bound[2 * mb]) : 0.f;
    const bool refine = keyed && bound > 0.f;
    uint32_t prefix = 0, pmask = 0;
    int need = static_cast<int>(K);
    for (int pass = 0; pass < (refine ? 2 : 1); ++pass) {
    if (pass == 1) {
        refine_band(a, mb, const_cast<float*>(sc), cc, key_to_float(prefix), 2.f * bound * 1.01f, list_bound[2 * mb + 1],
                    reps, max_chunks, scan_tmp);
        prefix = 0; pmask = 0; need = static_cast<int>(K);
    }
    // Radix select (MSB first) of the K-th largest order key.
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t jj = threadIdx.x; jj < cc; jj += blockDim.x) {
            const uint32_t u = keyed ? __float_as_uint(sc[jj]) : order_key(sc[jj]);
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
    }
    // Select: keys above the threshold, plus the first `need` ties by chunk index.
    int tie_base = 0, sel_base = 0;
    for (int64_t tile = 0; tile < cc; tile += blockDim.x) {
        const int64_t jj = tile + threadIdx.x;
        const bool in = jj < cc;
        const uint32_t u = in ? (keyed ? __float_as_uint(sc[jj]) : order_key(sc[jj])) : 0u;
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

// HP_TC_DESCENT=0 keeps query-block stages on the CUDA-core kernel (A/B timing, tests)
bool hp_tc_descent_disabled() {
    static const bool off = [] {
        const char* e = std::getenv("HP_TC_DESCENT");
        return e != nullptr && e[0] == '0';
    }();
    return off;
}

}  // namespace

extern "C" size_t hp_stage_workspace_bytes(int32_t n_lists, int32_t max_chunks, int32_t keep,
                                           int32_t chunk_size) {
    const size_t kmax = chunk_size > 0 ? static_cast<size_t>(keep / chunk_size) : 0;
    return align_up(static_cast<size_t>(n_lists) * max_chunks * 4, 256) +
           align_up(static_cast<size_t>(n_lists) * (kmax ? kmax : 1) * 4, 256) +
           align_up(static_cast<size_t>(n_lists) * 8, 256) +                   // per-list score bound, fp32-head mask
           align_up(static_cast<size_t>(n_lists) * max_chunks * kTcMaxHeads * 2, 256) + 256;  // rep offsets
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

static bool prune_uses_tc(const hp_stage_args& a) {
    const int rows_max = std::min(a.query_block, a.q_rows);
    return a.max_chunks > 0 && a.keys.dtype == HP_BF16 && a.keys.d == 128 && !a.rope.extension &&
           a.keys_exact != nullptr && rows_max >= 16 && a.query_block <= 64 && a.heads_per_mask <= kTcMaxHeads &&
           a.chunk_size <= 65536 &&
           !hp_tc_descent_disabled();
}

extern "C" int hp_prune_stage_variant(const hp_stage_args* ap, int32_t* variant) {
    if (!ap || !variant) return hph::set_error(HP_INVALID_ARGUMENT, "hp_prune_stage_variant: null pointer");
    *variant = prune_uses_tc(*ap) ? HP_PRUNE_TENSOR_CORE : HP_PRUNE_CUDA_CORE;
    return HP_OK;
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
    uint32_t* list_bound = reinterpret_cast<uint32_t*>(
        ws + align_up(static_cast<size_t>(n_lists) * max_chunks * 4, 256) +
        align_up(static_cast<size_t>(n_lists) * (kmax ? kmax : 1) * 4, 256));
    uint16_t* reps = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(list_bound) +
                                                 align_up(static_cast<size_t>(n_lists) * 8, 256));

    hp_stage_args la = a;
    la.max_chunks = max_chunks;
    // query-block stages on the tensor cores (bf16 keys with the exact-product flag, d = 128,
    // no RoPE, 16..64 q rows); the kernel itself checks q and the flag and falls back to
    // exact per-lane dots
    const bool tc = prune_uses_tc(a);
    if (tc) {
        const size_t keys_bytes = static_cast<size_t>(n_lists) * max_chunks * 4;
        if (int rc = hph::check_cuda(cudaMemsetAsync(scores, 0, keys_bytes, s), "hp_prune_stage: memset")) return rc;
        if (int rc = hph::check_cuda(cudaMemsetAsync(list_bound, 0, static_cast<size_t>(n_lists) * 8, s), "hp_prune_stage: memset"))
            return rc;
        auto kern = prune_descent_tc_kernel;
        if (int rc = hph::check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          static_cast<int>(kTcSmem)), "prune_descent_tc_kernel"))
            return rc;
        dim3 grid((max_chunks + 32 * kTcWarps - 1) / (32 * kTcWarps), a.heads_per_mask, n_lists);
        kern<<<grid, kTcWarps * 32, kTcSmem, s>>>(la, reinterpret_cast<uint32_t*>(scores), list_bound, reps, max_chunks);
        if (int rc = hph::check_cuda(cudaGetLastError(), "prune_descent_tc_kernel")) return rc;
    } else if (a.max_chunks > 0) {
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
    prune_topk_kernel<<<n_lists, kTopkThreads, 0, s>>>(la, scores, sel, max_chunks, kmax, status, tc,
                                                        tc ? list_bound : nullptr, reps);
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

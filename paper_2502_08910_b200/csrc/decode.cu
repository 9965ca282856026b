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
#include "topk.cuh"
#include "decode_dev.cuh"

using namespace hpk;
using namespace hpk::dec;

namespace {


size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
constexpr int kStageWarps = 4;     // warps per stage CTA
#ifndef HP_LOOKAHEAD
#define HP_LOOKAHEAD 1
#endif
constexpr bool kLookahead = HP_LOOKAHEAD != 0;  // two-comparison rounds for the classic stage path
constexpr int kMaxHC = 8;

// ------------------------------------------------------------------ stage kernel
template <typename T, bool EXT>
__global__ void __launch_bounds__(kStageWarps * 32, 6)
decode_stage_kernel(const hp_decode_stage_args a, float* scores, int* tickets, int cg, int prefetch) {
    pdl_trigger();
    pdl_wait();
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

    // identity (pruning.cpp:159-168): keep every chunk — decided here unless this is one
    // shard of a sequence-sharded stage (scores_out), whose selection is global
    if (a.scores_out == nullptr && (n_in <= a.keep || cc <= K)) {
        if (blockIdx.x == 0 && a.sel_out) {
            for (int64_t j = threadIdx.x; j < cc; j += blockDim.x) a.sel_out[static_cast<int64_t>(m) * a.sel_stride + j] = static_cast<int32_t>(j);
            if (threadIdx.x == 0) a.out_count[m] = static_cast<int32_t>(n_in);
        }
        return;
    }
    if (chunk0 >= cc) return;
    trace(10 + lc, 0);

    const int nwarps = blockDim.x >> 5;
    // staging first so every derived pointer stays a shared-window pointer (LDS, not LD.E)
    unsigned char* stage = smem;                                                   // [nwarps][32][stride]
    float* qs = reinterpret_cast<float*>(smem + static_cast<size_t>(nwarps) * 32 * G::stride);  // [hpm][128]
    uint32_t* qb = reinterpret_cast<uint32_t*>(qs + hpm * kD);                    // [hpm][64] bf16 pairs
    float* red = reinterpret_cast<float*>(qb + hpm * (kD / 2));                   // [hpm][chunks_per_cta]
    const int lane = threadIdx.x & 31, w = warp_id();
    bool q_safe = true;
    for (int i = threadIdx.x; i < hpm * kD; i += blockDim.x) {
        const float x = a.q[static_cast<int64_t>(m * hpm) * kD + i];
        qs[i] = x;
        q_safe &= q_product_safe(x);
    }
    // FHFMA path only without rotation, with bf16 keys certified in range, and bf16-exact q
    trace(10 + lc, 1);
    const bool use_fma = __syncthreads_and(q_safe) && !EXT && sizeof(T) == 2 &&
                         a.keys_exact != nullptr && *a.keys_exact != 0;
    if (use_fma) {
        for (int i = threadIdx.x; i < hpm * (kD / 2); i += blockDim.x)
            qb[i] = (__float_as_uint(qs[2 * i]) >> 16) | (__float_as_uint(qs[2 * i + 1]) & 0xffff0000u);
    }
    // unconditional barrier: a __syncthreads under a branch makes the compiler treat the
    // rest of the kernel as possibly warp-divergent (every shuffle becomes a
    // WARPSYNC.COLLECTIVE emulation loop)
    __syncthreads();
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

    unsigned char* wstage = stage + static_cast<size_t>(w) * 32 * G::stride;
    const unsigned char* myrow = wstage + lane * G::stride;
    const int swz = lane & (G::bytes / 16 - 1);

    // Items are (head, chunk group) pairs. The trip count is the same for every thread
    // and a warp past the end redoes the last item (its results are discarded): a
    // loop bounded by the warp index would read as divergent control flow around the
    // shuffles below and compile them to WARPSYNC.COLLECTIVE loops.
    const int n_items = hpm * cg;
    const int per_warp = (n_items + nwarps - 1) / nwarps;
    for (int k = 0; k < per_warp; ++k) {
        const int item_raw = w + k * nwarps;
        const bool item_ok = item_raw < n_items;
        const int item = item_ok ? item_raw : n_items - 1;
        const int hh = item % hpm, grp = item / hpm;
        const int qh = m * hpm + hh;
        const int kvh = qh / (a.n_q_heads / a.keys.n_kv);
        const float* qrow = qs + hh * kD;
        const uint32_t* qbrow = qb + hh * (kD / 2);
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
        auto score = [&](const float* cs, const float* sn) -> float {
            if constexpr (EXT) return dot_row_rot<T>(myrow, swz, qrow, cs, sn);
            else return use_fma ? dot_row_bf16x(myrow, swz, qbrow) : dot_row<T>(myrow, swz, qrow);
        };
        const float* cs1 = nullptr; const float* sn1 = nullptr;
        const float* cs2 = nullptr; const float* sn2 = nullptr;
        bool same_rot = true, plain1 = false;
        if constexpr (EXT) {
            constexpr int half = kD / 2;
            const int64_t p1 = rope_k_position(a.rope, 1, j), p2 = rope_k_position(a.rope, 2, j);
            cs1 = a.rope.cos_tab + p1 * half; sn1 = a.rope.sin_tab + p1 * half;
            cs2 = a.rope.cos_tab + p2 * half; sn2 = a.rope.sin_tab + p2 * half;
            same_rot = p1 == p2;
        plain1 = p1 == 0;
        }
        int first = 1, last = len, it = 0, iters = 0;
        while ((1 << iters) < len) ++iters;
        float s1 = 0.f, s2 = 0.f;
        const int mid0 = (1 + len + 1) >> 1;  // first step's mid is known up front
        __syncwarp();
        stage_rows<T>(a.keys, kvh, active ? token(0) : -1, wstage, lane,
                      prefetch && active && iters > 0 ? token(mid0 - 1) : -1);
        if (k == 0) trace(10 + lc, 3);
        // both branches' scores of the staged row (one pass for bf16 rows with RoPE)
        auto score2 = [&](float& b1, float& b2) {
            if constexpr (EXT && sizeof(T) == 2) {
                dot_row_rot2_bf16(myrow, swz, qrow, cs1, sn1, cs2, sn2, same_rot, b1, b2, plain1);
            } else {
                b1 = score(cs1, sn1);
                b2 = same_rot ? b1 : score(cs2, sn2);
            }
        };
        if (active) score2(s1, s2);
        if (k == 0) trace(10 + lc, 4);
        for (;;) {
            const bool go = active && it < iters && first < last;
            if (!__any_sync(0xffffffffu, go)) break;
            const int mid = (first + last + 1) >> 1;
            int64_t pf_r = -1, pf_l = -1;
            if (prefetch && go && it + 1 < iters) {
                if (mid < last) pf_r = token(((mid + last + 1) >> 1) - 1);       // if it goes right
                if (first < mid - 1) pf_l = token(((first + mid) >> 1) - 1);     // if it goes left
            }
            __syncwarp();
            stage_rows<T>(a.keys, kvh, go ? token(mid - 1) : -1, wstage, lane, pf_r, pf_l);
            if (k == 0 && it == 0) trace(10 + lc, 5);
            if (go) {
                float m1, m2;
                score2(m1, m2);
                if (m2 > s1) { first = mid; s1 = m1; s2 = m2; } else { last = mid - 1; }
                ++it;
            }
            if (k == 0 && it == 1) trace(10 + lc, 6);
        }
        if (item_ok) red[hh * chunks_per_cta + grp * 32 + lane] = s2;
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
            (a.scores_out ? a.scores_out : scores)[static_cast<int64_t>(m) * a.max_chunks + jj] = best;
        }
    }
    trace(10 + lc, 2);
    (void)tickets;
}

// ------------------------------------------------ lookahead stage kernel (bf16, no RoPE)
// The classic kernel's descent is one dependent row gather per comparison (6 for
// l_c = 32). Here every round after the first gathers the step's mid row AND both
// possible next mids (the direction is unknown until the compare, the candidates are
// not), then makes two comparisons: l_c = 32 takes 3 rounds (2 + 3 + 3 rows) instead
// of 6. The three dots run as independent chains over one q read. Same comparisons
// on the same fp32 values as the classic kernel, so the same representatives.
__global__ void __launch_bounds__(kStageWarps * 32, 2)
decode_stage_look_kernel(const hp_decode_stage_args a, float* scores, int cg, int prefetch) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem[];
    using T = bf16_t;
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    const int m = blockIdx.y;
    const int64_t n_in = a.in_count ? a.in_count[m] : a.in_count_const;
    const int lc = a.chunk_size;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int K = a.keep / lc;
    const int chunks_per_cta = 32 * cg;
    const int64_t chunk0 = static_cast<int64_t>(blockIdx.x) * chunks_per_cta;
    if (a.scores_out == nullptr && (n_in <= a.keep || cc <= K)) {  // identity (pruning.cpp:159-168)
        if (blockIdx.x == 0 && a.sel_out) {
            for (int64_t j = threadIdx.x; j < cc; j += blockDim.x) a.sel_out[static_cast<int64_t>(m) * a.sel_stride + j] = static_cast<int32_t>(j);
            if (threadIdx.x == 0) a.out_count[m] = static_cast<int32_t>(n_in);
        }
        return;
    }
    if (chunk0 >= cc) return;
    const int nwarps = blockDim.x >> 5;
    unsigned char* stage = smem;  // [nwarps][kLookSlots][32][stride]
    // per-warp q of its current head (fp32 + packed bf16 pairs): warp-private, so the
    // prologue needs no CTA barrier and q staging overlaps the first gather
    float* qw_all = reinterpret_cast<float*>(smem + static_cast<size_t>(nwarps) * kLookSlots * 32 * G::stride);
    float* red = qw_all + nwarps * (kD + kD / 2);  // [hpm][chunks_per_cta]
    const int lane = threadIdx.x & 31, w = warp_id();
    float* qrow = qw_all + w * (kD + kD / 2);
    uint32_t* qbrow = reinterpret_cast<uint32_t*>(qrow + kD);
    const bool keys_ok = a.keys_exact != nullptr && *a.keys_exact != 0;
    unsigned char* wstage = stage + static_cast<size_t>(w) * kLookSlots * 32 * G::stride;
    const unsigned char* row0 = wstage + lane * G::stride;
    const unsigned char* row1 = row0 + 32 * G::stride;
    const unsigned char* row2 = row1 + 32 * G::stride;
    const int swz = lane & (G::bytes / 16 - 1);
    const int n_items = hpm * cg;
    const int per_warp = (n_items + nwarps - 1) / nwarps;
    for (int k = 0; k < per_warp; ++k) {
        const int item_raw = w + k * nwarps;
        const bool item_ok = item_raw < n_items;
        const int item = item_ok ? item_raw : n_items - 1;
        const int hh = item % hpm, grp = item / hpm;
        const int qh = m * hpm + hh;
        const int kvh = qh / (a.n_q_heads / a.keys.n_kv);
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
        bool use_fma = false;
        auto dots = [&](float& d0, float& d1, float& d2) {
            if (use_fma) {
                dot3_bf16x(row0, row1, row2, swz, qbrow, d0, d1, d2);
            } else {
                d0 = dot_row<T>(row0, swz, qrow);
                d1 = dot_row<T>(row1, swz, qrow);
                d2 = dot_row<T>(row2, swz, qrow);
            }
        };
        int first = 1, last = len, it = 0, iters = 0;
        while ((1 << iters) < len) ++iters;
        float s1 = 0.f;
        // round 1: row 0 and the first mid (its two successors warmed in L2)
        const int mid0 = (1 + len + 1) >> 1;
        const bool step0 = active && iters > 0;
        __syncwarp();
        {
            int64_t pr = -1, pl = -1;
            if (prefetch && step0 && iters > 1) {
                if (mid0 < last) pr = token(((mid0 + last + 1) >> 1) - 1);
                if (first < mid0 - 1) pl = token(((first + mid0) >> 1) - 1);
            }
            stage_rows3<false>(a.keys, kvh, active ? token(0) : -1, step0 ? token(mid0 - 1) : -1, -1, wstage, lane);
            if (pr >= 0) {
                const char* p = kv_row_ptr(a.keys, a.keys.k_pool, a.keys.k_host, kvh, pr, 2);
                prefetch_l2(p); prefetch_l2(p + 128);
            }
            if (pl >= 0) {
                const char* p = kv_row_ptr(a.keys, a.keys.k_pool, a.keys.k_host, kvh, pl, 2);
                prefetch_l2(p); prefetch_l2(p + 128);
            }
        }
        {  // this head's q while the rows are in flight (the previous item's dots are done: __syncwarp above)
            bool safe = true;
#pragma unroll
            for (int i = 0; i < kD / 32; ++i) {
                const float x = a.q[static_cast<int64_t>(qh) * kD + i * 32 + lane];
                qrow[i * 32 + lane] = x;
                safe &= q_product_safe(x);
            }
            use_fma = __all_sync(0xffffffffu, safe) && keys_ok;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < kD / 64; ++i) {
                const int e = i * 32 + lane;
                qbrow[e] = (__float_as_uint(qrow[2 * e]) >> 16) | (__float_as_uint(qrow[2 * e + 1]) & 0xffff0000u);
            }
            cp_async_wait_all();
            __syncwarp();
        }
        if (active) {
            float d0, d1, d2;
            dots(d0, d1, d2);
            s1 = d0;
            if (step0) {
                if (d1 > s1) { first = mid0; s1 = d1; } else { last = mid0 - 1; }
                ++it;
            }
        }
        // rounds of two comparisons: the mid row and both candidate next mids
        for (;;) {
            const bool go = active && it < iters && first < last;
            if (!__any_sync(0xffffffffu, go)) break;
            const int mid = (first + last + 1) >> 1;
            const bool more = it + 1 < iters;
            const int mid_r = (go && more && mid < last) ? ((mid + last + 1) >> 1) : 0;
            const int mid_l = (go && more && first < mid - 1) ? ((first + mid) >> 1) : 0;
            __syncwarp();
            stage_rows3(a.keys, kvh, go ? token(mid - 1) : -1, mid_r ? token(mid_r - 1) : -1,
                        mid_l ? token(mid_l - 1) : -1, wstage, lane);
            if (go) {
                float dm, dr, dl;
                dots(dm, dr, dl);
                float nx;
                int nmid;
                if (dm > s1) { first = mid; s1 = dm; nx = dr; nmid = mid_r; } else { last = mid - 1; nx = dl; nmid = mid_l; }
                ++it;
                if (it < iters && first < last) {  // nmid == (first + last + 1) >> 1, staged above
                    if (nx > s1) { first = nmid; s1 = nx; } else { last = nmid - 1; }
                    ++it;
                }
            }
        }
        if (item_ok) red[hh * chunks_per_cta + grp * 32 + lane] = s1;
        __syncwarp();
    }
    __syncthreads();
    for (int c0 = 0; c0 < chunks_per_cta; c0 += blockDim.x) {
        const int c = c0 + threadIdx.x;
        const int64_t jj = chunk0 + c;
        const bool valid = c < chunks_per_cta && jj < cc;
        float best = -INFINITY;
        if (valid) {
            for (int h = 0; h < hpm; ++h) {
                const float sc = red[h * chunks_per_cta + c];
                best = (best < sc) ? sc : best;  // std::max (pruning.cpp:182)
            }
            (a.scores_out ? a.scores_out : scores)[static_cast<int64_t>(m) * a.max_chunks + jj] = best;
        }
    }
}

// ------------------------------------------------------ one-wave stage kernel (big stages)
// The long-chunk descents (stage 1: 4,091 chunks x 32 q-heads at 1M) need every warp
// resident at once: a warp of 32 descents stages 32 rows (8 KB), and a second wave of
// CTAs would run the whole 9-step dependent chain again at low occupancy. Here a CTA
// is 7 warps (56 KB of staging, nothing else in shared memory): 4 CTAs fill an SM's
// 228 KB, 148 x 4 x 7 = 4,144 warps >= 4,096 items. Each warp is one (mask, chunk
// group, head) item; q is read through L1 (a broadcast), and each warp writes its
// head's representative scores to [mask][head][chunk] — the selection takes the max
// over heads in head order, as the reference does.
constexpr int kWideWarps = 7;

// EXT (RoPE extension, rope_policy.cpp:18-72): each warp rotates its head's q once into
// its own 512 B of shared memory (rotate_queries, pruning.cpp:39-52) and every staged
// key row is rotated element by element inside the sequential dot at the chunk's
// branch-1 / branch-2 key positions (separately rounded, as apply_rope_inplace).
template <typename T, bool EXT = false>
__global__ void __launch_bounds__(kWideWarps * 32, 4)
decode_stage_wide_kernel(const hp_decode_stage_args a, float* hscores, int groups) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem[];
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    const int lc = a.chunk_size;
    const int lane = threadIdx.x & 31, w = warp_id();
    const int per_mask = groups * hpm;
    const int item_raw = blockIdx.x * kWideWarps + w;
    const bool item_ok = item_raw < a.n_masks * per_mask;
    const int item = item_ok ? item_raw : 0;
    const int m = item / per_mask, rem = item - m * per_mask;
    const int g = rem / hpm, hh = rem - g * hpm;  // the heads of a chunk group are adjacent items
    const int64_t n_in = a.in_count ? a.in_count[m] : a.in_count_const;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int K = a.keep / lc;
    // identity stages need no scores (the selection keeps every chunk)
    const bool run = item_ok && !(n_in <= a.keep || cc <= K) && static_cast<int64_t>(g) * 32 < cc;
    const int qh = m * hpm + hh;
    const int kvh = qh / (a.n_q_heads / a.keys.n_kv);
    const float* qrow = a.q + static_cast<int64_t>(qh) * kD;
    bool use_fma = false;  // set below, while the first rows are in flight
    unsigned char* wstage = smem + static_cast<size_t>(w) * 32 * G::stride;
    const unsigned char* myrow = wstage + lane * G::stride;
    const int swz = lane & (G::bytes / 16 - 1);
    const int64_t j = static_cast<int64_t>(g) * 32 + lane;
    const bool active = run && j < cc;
    const int64_t base = j * lc;
    const int len = active ? static_cast<int>(min64(lc, n_in - base)) : 0;
    int64_t t_first = 0;
    bool contiguous = true;
    if (active) {
        t_first = ref_token(a.in, m, base);
        if (len > 1) contiguous = ref_token(a.in, m, base + len - 1) - t_first == len - 1;
    }
    auto token = [&](int i) -> int64_t { return contiguous ? t_first + i : ref_token(a.in, m, base + i); };
    float* qrot = reinterpret_cast<float*>(smem + static_cast<size_t>(kWideWarps) * 32 * G::stride) + w * kD;
    const float* cs1 = nullptr; const float* sn1 = nullptr;
    const float* cs2 = nullptr; const float* sn2 = nullptr;
    bool same_rot = true, plain1 = false;
    if constexpr (EXT) {
        constexpr int half = kD / 2;
        const int64_t qp = rope_q_position(a.rope, a.query_position, a.stream_tokens, cc);
        for (int e = lane; e < half; e += 32) {
            const float x = __ldg(qrow + e), y = __ldg(qrow + e + half);
            const float c = a.rope.cos_tab[qp * half + e], sn = a.rope.sin_tab[qp * half + e];
            qrot[e] = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, sn));
            qrot[e + half] = __fadd_rn(__fmul_rn(x, sn), __fmul_rn(y, c));
        }
        __syncwarp();
        const int64_t p1 = rope_k_position(a.rope, 1, j), p2 = rope_k_position(a.rope, 2, j);
        cs1 = a.rope.cos_tab + p1 * half; sn1 = a.rope.sin_tab + p1 * half;
        cs2 = a.rope.cos_tab + p2 * half; sn2 = a.rope.sin_tab + p2 * half;
        same_rot = p1 == p2;
        plain1 = p1 == 0;
    }
    auto score = [&]() -> float {
        // q through L1: every lane reads the same address (one wavefront per load)
        const float4* q4 = reinterpret_cast<const float4*>(qrow);
        float acc = 0.0f;
        if constexpr (sizeof(T) == 2) {
#pragma unroll 4
            for (int c = 0; c < 16; ++c) {
                const uint4 wv = *reinterpret_cast<const uint4*>(myrow + ((c ^ swz) << 4));
                const float4 qa = __ldg(q4 + 2 * c), qb = __ldg(q4 + 2 * c + 1);
                if (use_fma) {
                    acc = __fmaf_rn(qa.x, bf16_lo(wv.x), acc); acc = __fmaf_rn(qa.y, bf16_hi(wv.x), acc);
                    acc = __fmaf_rn(qa.z, bf16_lo(wv.y), acc); acc = __fmaf_rn(qa.w, bf16_hi(wv.y), acc);
                    acc = __fmaf_rn(qb.x, bf16_lo(wv.z), acc); acc = __fmaf_rn(qb.y, bf16_hi(wv.z), acc);
                    acc = __fmaf_rn(qb.z, bf16_lo(wv.w), acc); acc = __fmaf_rn(qb.w, bf16_hi(wv.w), acc);
                } else {
                    acc = __fadd_rn(acc, __fmul_rn(qa.x, bf16_lo(wv.x))); acc = __fadd_rn(acc, __fmul_rn(qa.y, bf16_hi(wv.x)));
                    acc = __fadd_rn(acc, __fmul_rn(qa.z, bf16_lo(wv.y))); acc = __fadd_rn(acc, __fmul_rn(qa.w, bf16_hi(wv.y)));
                    acc = __fadd_rn(acc, __fmul_rn(qb.x, bf16_lo(wv.z))); acc = __fadd_rn(acc, __fmul_rn(qb.y, bf16_hi(wv.z)));
                    acc = __fadd_rn(acc, __fmul_rn(qb.z, bf16_lo(wv.w))); acc = __fadd_rn(acc, __fmul_rn(qb.w, bf16_hi(wv.w)));
                }
            }
        } else {
#pragma unroll 4
            for (int c = 0; c < 32; ++c) {
                const float4 wv = *reinterpret_cast<const float4*>(myrow + ((c ^ swz) << 4));
                const float4 qa = __ldg(q4 + c);
                acc = __fadd_rn(acc, __fmul_rn(qa.x, wv.x)); acc = __fadd_rn(acc, __fmul_rn(qa.y, wv.y));
                acc = __fadd_rn(acc, __fmul_rn(qa.z, wv.z)); acc = __fadd_rn(acc, __fmul_rn(qa.w, wv.w));
            }
        }
        return acc;
    };
    int first = 1, last = len, it = 0, iters = 0;
    while ((1 << iters) < len) ++iters;
    float s1 = 0.f, s2 = 0.f;
    stage_rows<T, false>(a.keys, kvh, active ? token(0) : -1, wstage, lane);
    if constexpr (!EXT) {
        // FFMA when every product is exact (bf16-exact q, keys certified), FMUL+FADD
        // otherwise — checked while the first gather is in flight
        bool q_safe = true;
#pragma unroll
        for (int i = 0; i < kD / 32; ++i) q_safe &= q_product_safe(__ldg(qrow + i * 32 + lane));
        use_fma = __all_sync(0xffffffffu, q_safe) && sizeof(T) == 2 && a.keys_exact != nullptr && *a.keys_exact != 0;
    }
    cp_async_wait_all();
    __syncwarp();
    // branch-1 / branch-2 scores of a staged row (identical without rotation)
    auto score2 = [&](float& b1, float& b2) {
        if constexpr (EXT && sizeof(T) == 2) {
            dot_row_rot2_bf16(myrow, swz, qrot, cs1, sn1, cs2, sn2, same_rot, b1, b2, plain1);
        } else if constexpr (EXT) {
            b1 = dot_row_rot<T>(myrow, swz, qrot, cs1, sn1);
            b2 = same_rot ? b1 : dot_row_rot<T>(myrow, swz, qrot, cs2, sn2);
        } else {
            b1 = b2 = score();
        }
    };
    if (active) score2(s1, s2);
    for (;;) {
        const bool go = active && it < iters && first < last;
        if (!__any_sync(0xffffffffu, go)) break;
        const int mid = (first + last + 1) >> 1;
        stage_rows<T>(a.keys, kvh, go ? token(mid - 1) : -1, wstage, lane);
        if (go) {
            float m1, m2;
            score2(m1, m2);
            if (m2 > s1) { first = mid; s1 = m1; s2 = m2; } else { last = mid - 1; }  // pruning.cpp:91
            ++it;
        }
    }
    // the representative's branch-2 score (pruning.cpp:181)
    if (active) hscores[(static_cast<int64_t>(m) * hpm + hh) * a.max_chunks + j] = s2;
}

// ------------------------------------------------- all-rows stage kernel (small l_c)
// For short chunks (l_c <= 32; the 3k preset's stage 3 has l_c = 8) a warp owns
// 32 / l_c whole chunks: lane i stages row i % l_c of chunk i / l_c (one gather for
// all the mask's heads, which share one kv head) and computes that row's sequential
// dot with every head's q (independent accumulators: q is a shared-memory broadcast,
// the row is read once). Each head's Alg. 3 descent is then replayed on those scores
// with shuffles inside the chunk's lane group — the same comparisons of the same fp32
// values, so representatives and scores are exactly the reference's — at one gather
// latency instead of ceil(log2 l_c) + 1 dependent ones. It reads every row of a chunk
// (8 here) where the descents touch ~5-7 distinct rows: ~1.2x the distinct bytes at
// 3k/1M for one dependent round trip instead of four.
constexpr int kAllRowsWarps = 8;
constexpr int kAllRowsHeads = 4;  // accumulators per lane (heads per pass)

// EXT: q rotated in shared memory once per CTA; each lane's row dotted rotated at its
// chunk's branch-1 and branch-2 key positions, and the replay compares branch-2 of the
// mid with branch-1 of the current first, as select_rep_rotated does.
template <typename T, bool EXT = false>
__global__ void __launch_bounds__(kAllRowsWarps * 32)
decode_stage_allrows_kernel(const hp_decode_stage_args a, float* scores) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(128) unsigned char smem[];
    const int cut = dev_cut_point(5);
    if (cut == 0) return;
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    const int lc = a.chunk_size;
    const int m = blockIdx.y;
    const int64_t n_in = a.in_count ? a.in_count[m] : a.in_count_const;
    const int64_t cc = (n_in + lc - 1) / lc;
    const int K = a.keep / lc;
    if (a.scores_out == nullptr && (n_in <= a.keep || cc <= K)) {  // identity (pruning.cpp:159-168)
        if (blockIdx.x == 0 && a.sel_out) {
            for (int64_t j = threadIdx.x; j < cc; j += blockDim.x) a.sel_out[static_cast<int64_t>(m) * a.sel_stride + j] = static_cast<int32_t>(j);
            if (threadIdx.x == 0) a.out_count[m] = static_cast<int32_t>(n_in);
        }
        return;
    }
    const int cpw = 32 / lc;  // chunks per warp
    const int lane = threadIdx.x & 31, w = warp_id();
    if (static_cast<int64_t>(blockIdx.x) * kAllRowsWarps * cpw >= cc) return;
    unsigned char* wstage = smem + static_cast<size_t>(w) * 32 * G::stride;
    float* qs = reinterpret_cast<float*>(smem + static_cast<size_t>(kAllRowsWarps) * 32 * G::stride);
    uint32_t* qb = reinterpret_cast<uint32_t*>(qs + hpm * kD);
    // the row gather goes out first; q staging and the exactness check overlap it
    const int cl = lane / lc, r = lane - cl * lc;  // lane -> (chunk of the warp, row)
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * kAllRowsWarps + w) * cpw + cl;
    const bool live = j < cc && cl < cpw;
    const int kvh = (m * hpm) / (a.n_q_heads / a.keys.n_kv);
    const int64_t base = j * lc;
    const int len = live ? static_cast<int>(min64(lc, n_in - base)) : 0;
    const int64_t tok = r < len ? ref_token(a.in, m, base + r) : -1;
    if (cut == 2 && tok == 123456789) scores[0] = 0.f;
    if (cut == 2) return;
    stage_rows<T, false>(a.keys, kvh, tok, wstage, lane);
    bool q_safe = true;
    for (int i = threadIdx.x; i < hpm * kD; i += blockDim.x) {
        const float x = a.q[static_cast<int64_t>(m * hpm) * kD + i];
        qs[i] = x;
        q_safe &= q_product_safe(x);
    }
    const bool use_fma = __syncthreads_and(q_safe) && !EXT && sizeof(T) == 2 && a.keys_exact != nullptr && *a.keys_exact != 0;
    if (use_fma) {
        for (int i = threadIdx.x; i < hpm * (kD / 2); i += blockDim.x)
            qb[i] = (__float_as_uint(qs[2 * i]) >> 16) | (__float_as_uint(qs[2 * i + 1]) & 0xffff0000u);
    }
    const float* cs1 = nullptr; const float* sn1 = nullptr;
    const float* cs2 = nullptr; const float* sn2 = nullptr;
    bool same_rot = true, plain1 = false;
    if constexpr (EXT) {
        constexpr int half = kD / 2;
        const int64_t qp = rope_q_position(a.rope, a.query_position, a.stream_tokens, cc);
        for (int i = threadIdx.x; i < hpm * half; i += blockDim.x) {
            const int hh = i / half, e = i - hh * half;
            float* qr = qs + hh * kD;
            const float c = a.rope.cos_tab[qp * half + e], sn = a.rope.sin_tab[qp * half + e];
            const float x = qr[e], y = qr[e + half];
            qr[e] = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, sn));
            qr[e + half] = __fadd_rn(__fmul_rn(x, sn), __fmul_rn(y, c));
        }
        const int64_t jj = live ? j : 0;
        const int64_t p1 = rope_k_position(a.rope, 1, jj), p2 = rope_k_position(a.rope, 2, jj);
        cs1 = a.rope.cos_tab + p1 * half; sn1 = a.rope.sin_tab + p1 * half;
        cs2 = a.rope.cos_tab + p2 * half; sn2 = a.rope.sin_tab + p2 * half;
        same_rot = p1 == p2;
        plain1 = p1 == 0;
    }
    __syncthreads();  // unconditional (see decode_stage_kernel)
    if (cut == 1) return;
    cp_async_wait_all();
    __syncwarp();
    if (cut == 3) return;
    const unsigned char* row = wstage + lane * G::stride;
    const int swz = lane & (G::bytes / 16 - 1);
    const int c0 = cl * lc;  // first lane of this chunk
    int iters = 0;
    while ((1 << iters) < lc) ++iters;
    float best = -INFINITY;
    for (int h0 = 0; h0 < hpm; h0 += kAllRowsHeads) {
        float acc[kAllRowsHeads], acc1[kAllRowsHeads];  // branch-2 / branch-1 row scores
#pragma unroll
        for (int u = 0; u < kAllRowsHeads; ++u) acc[u] = 0.0f;
        const int nh = min(kAllRowsHeads, hpm - h0);
        if constexpr (EXT) {
#pragma unroll
            for (int u = 0; u < kAllRowsHeads; ++u) {
                const float* qr = qs + (h0 + min(u, nh - 1)) * kD;
                if constexpr (sizeof(T) == 2) {
                    dot_row_rot2_bf16(row, swz, qr, cs1, sn1, cs2, sn2, same_rot, acc1[u], acc[u], plain1);
                } else {
                    acc1[u] = dot_row_rot<T>(row, swz, qr, cs1, sn1);
                    acc[u] = same_rot ? acc1[u] : dot_row_rot<T>(row, swz, qr, cs2, sn2);
                }
            }
        } else if (use_fma && nh == kAllRowsHeads) {  // full group of heads: constant q offsets, no index math
            const uint4* q4 = reinterpret_cast<const uint4*>(qb + h0 * (kD / 2));
            uint4 wv[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) wv[c] = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
#pragma unroll
            for (int c = 0; c < 16; ++c) {
#pragma unroll
                for (int u = 0; u < kAllRowsHeads; ++u) {
                    const uint4 q = q4[u * 16 + c];  // broadcast
                    acc[u] = fma_bf16(q.x, wv[c].x, acc[u], false);
                    acc[u] = fma_bf16(q.x, wv[c].x, acc[u], true);
                    acc[u] = fma_bf16(q.y, wv[c].y, acc[u], false);
                    acc[u] = fma_bf16(q.y, wv[c].y, acc[u], true);
                    acc[u] = fma_bf16(q.z, wv[c].z, acc[u], false);
                    acc[u] = fma_bf16(q.z, wv[c].z, acc[u], true);
                    acc[u] = fma_bf16(q.w, wv[c].w, acc[u], false);
                    acc[u] = fma_bf16(q.w, wv[c].w, acc[u], true);
                }
            }
        } else if (use_fma) {
            const uint4* q4 = reinterpret_cast<const uint4*>(qb + h0 * (kD / 2));
#pragma unroll 2
            for (int c = 0; c < 16; ++c) {
                const uint4 wv = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
#pragma unroll
                for (int u = 0; u < kAllRowsHeads; ++u) {
                    const uint4 q = q4[min(u, nh - 1) * 16 + c];  // broadcast; u >= nh redoes a head (discarded)
                    acc[u] = fma_bf16(q.x, wv.x, acc[u], false);
                    acc[u] = fma_bf16(q.x, wv.x, acc[u], true);
                    acc[u] = fma_bf16(q.y, wv.y, acc[u], false);
                    acc[u] = fma_bf16(q.y, wv.y, acc[u], true);
                    acc[u] = fma_bf16(q.z, wv.z, acc[u], false);
                    acc[u] = fma_bf16(q.z, wv.z, acc[u], true);
                    acc[u] = fma_bf16(q.w, wv.w, acc[u], false);
                    acc[u] = fma_bf16(q.w, wv.w, acc[u], true);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < kAllRowsHeads; ++u)
                acc[u] = dot_row<T>(row, swz, qs + (h0 + min(u, nh - 1)) * kD);
        }
        if (cut == 4 && acc[0] == 1.2345f) scores[0] = 0.f;
        // Alg. 3 per head on the chunk's row scores (pruning.cpp:69-98): right only on
        // strict s(mid) > s(first); sigma1 == sigma2 without rotation. ceil(log2 l_c)
        // rounds for every lane: a short chunk settles early and idles.
#pragma unroll
        for (int u = 0; u < kAllRowsHeads; ++u) {
            const float sc = r < len ? acc[u] : -INFINITY;  // branch-2 score of this lane's row
            if constexpr (EXT) {
                const float sc1 = r < len ? acc1[u] : -INFINITY;
                int first = 1, last = len;
                float s1 = __shfl_sync(0xffffffffu, sc1, c0), s2 = __shfl_sync(0xffffffffu, sc, c0);
                for (int it = 0; it < iters; ++it) {
                    const int mid = (first + last + 1) >> 1;
                    const bool go = first < last;
                    const int src = c0 + (go ? mid - 1 : 0);
                    const float m2 = __shfl_sync(0xffffffffu, sc, src), m1 = __shfl_sync(0xffffffffu, sc1, src);
                    if (go) {
                        if (m2 > s1) { first = mid; s1 = m1; s2 = m2; } else { last = mid - 1; }
                    }
                }
                if (u < nh) best = (best < s2) ? s2 : best;  // max over heads of branch 2 (pruning.cpp:181-182)
            } else {
                int first = 1, last = len;
                float s1 = __shfl_sync(0xffffffffu, sc, c0);
                for (int it = 0; it < iters; ++it) {
                    const int mid = (first + last + 1) >> 1;
                    const bool go = first < last;
                    const float s2 = __shfl_sync(0xffffffffu, sc, c0 + (go ? mid - 1 : 0));
                    if (go) {
                        if (s2 > s1) { first = mid; s1 = s2; } else { last = mid - 1; }
                    }
                }
                if (u < nh) best = (best < s1) ? s1 : best;  // max over heads (pruning.cpp:182)
            }
        }
    }
    if (cut == 4) return;
    if (live && r == 0) (a.scores_out ? a.scores_out : scores)[static_cast<int64_t>(m) * a.max_chunks + j] = best;
}

// ----------------------------------------------------------------- top-k kernel
// Exact top-(k/l_c) chunk selection for one mask by a 1024-thread CTA: the mask's
// chunk scores become order keys in shared memory and cta_topk_smem selects; the
// kept chunk ids land in sel_out in ascending order, and the stage's output count
// (pruning.cpp:194-199: K-1 full chunks plus the last kept chunk's length) in
// out_count. With list_out the stage's token list is materialised as well.
#ifndef HP_TOPK_THREADS
#define HP_TOPK_THREADS 1024
#endif
constexpr int kTopkThreads2 = HP_TOPK_THREADS;
constexpr int kTopkMaxKeys = 16384;

template <int HP>
__device__ __forceinline__ void load_head_max(const float* sc, int stride, int cc, uint32_t* keys, int hp = HP) {
    constexpr int kPer = 4;  // chunks per thread per round (4,096 chunks = one round at 1,024 threads)
    const int t = threadIdx.x, nt = blockDim.x;
    for (int j0 = 0; j0 < cc; j0 += kPer * nt) {
        float v[kPer][HP];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = j0 + k * nt + t;
#pragma unroll
            for (int h = 0; h < HP; ++h)
                v[k][h] = (j < cc && h < hp) ? __ldcg(sc + static_cast<int64_t>(h) * stride + j) : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = j0 + k * nt + t;
            float best = -INFINITY;
#pragma unroll
            for (int h = 0; h < HP; ++h) best = (best < v[k][h]) ? v[k][h] : best;
            if (j < cc) keys[j] = order_key(best);
        }
    }
}

__global__ void __launch_bounds__(kTopkThreads2)
decode_topk_kernel(const hp_decode_stage_args a, const float* scores, int head_planes) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ TopkShared sh;
    const int cut = dev_cut_point(3);
    if (cut == 0) return;
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
    uint32_t* keys = reinterpret_cast<uint32_t*>(tsm);              // [cc]
    int32_t* ssel = reinterpret_cast<int32_t*>(keys + ((a.max_chunks + 3) & ~3));  // [K] after keys[max_chunks]
    if (head_planes <= 1) {
        const float* sc = scores + static_cast<int64_t>(m) * a.max_chunks;
        constexpr int kPer = kTopkMaxKeys / kTopkThreads2;  // 16 independent loads per thread
        float v[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = k * nt + t;
            v[k] = j < cc ? __ldcg(sc + j) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = k * nt + t;
            if (j < cc) keys[j] = order_key(v[k]);
        }
    } else {
        // per-head representative scores [m][head][chunk]: chunk score = max over the
        // mask's heads in head order (pruning.cpp:176-184, std::max from -inf); every
        // load of the thread's chunks x heads is issued before the first use
        const float* sc = scores + static_cast<int64_t>(m) * head_planes * a.max_chunks;
        switch (head_planes) {
            case 2: load_head_max<2>(sc, a.max_chunks, cc, keys); break;
            case 3: load_head_max<3>(sc, a.max_chunks, cc, keys); break;
            case 4: load_head_max<4>(sc, a.max_chunks, cc, keys); break;
            default: load_head_max<8>(sc, a.max_chunks, cc, keys, head_planes); break;
        }
    }
    __syncthreads();
    trace(3, 1);
    if (cut == 1) return;
    cta_topk_smem(keys, cc, K, ssel, sh, cut);
    trace(3, 2);
    if (cut == 2 || cut >= 10) return;
    for (int i = t; i < K; i += nt) sel[i] = ssel[i];
    const int lastc = ssel[K - 1];
    const int n_out = (K - 1) * lc + min(lc, n_in - lastc * lc);
    if (t == 0) a.out_count[m] = n_out;
    if (cut == 3) return;
    if (a.list_out) {  // materialize: output position o -> chunk sel[o / lc] -> input list
        for (int o = t; o < n_out; o += nt) {
            const int r = o / lc;
            a.list_out[m * a.list_out_stride + o] =
                static_cast<int32_t>(ref_token(a.in, m, static_cast<int64_t>(ssel[r]) * lc + (o - r * lc)));
        }
    }
    trace(3, 4);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// -------------------------------------------------------------------- BSA kernel
// Split-K attention for one decode row per q-head over the selected set
// sinks ∪ mask ∪ stream (selected_indices + attention_row, sparse_attention.cpp:
// 33-60,95-112). grid = (splits, n_q_heads / HC): a CTA owns up to 128 consecutive
// selected positions for the HC q-heads that share one kv head (GQA), so every K/V
// row is gathered once for HC heads.
//   1. positions -> tokens (one list load), then ONE cp.async.bulk per K and V row
//      (256 B bf16) into shared memory, all completing on a single mbarrier;
//   2. QK: two threads per key (64 elements each, padded K stride -> conflict-free
//      LDS.128, q broadcast), one shuffle to combine;
//   3. softmax per head (warp h), PV with thread = (element pair, key quarter);
//   4. partial (m, l, o) per head to the workspace; the last CTA of the head group
//      (acq_rel ticket) merges all splits by log-sum-exp.
// The output matches attention_row within the stated fp32 tolerance (only the
// summation order differs from the reference's ascending loop).
constexpr int kBsaThreads = 256;
constexpr int kBsaRec = kD + 4;
#ifndef HP_BSA_CLUSTER
#define HP_BSA_CLUSTER 1
#endif
constexpr bool kBsaUseCluster = HP_BSA_CLUSTER != 0;  // partial record per (split, head): m, l, pad, pad, o[kD] (16 B aligned)
constexpr int kBsaMaxKeys = 128;
constexpr int kBsaMinKeys = 32;

template <typename T, int HC, int MK = kBsaMaxKeys, int NQ = kBsaThreads / 64>
struct BsaSmem {
    static constexpr int RB = kD * static_cast<int>(sizeof(T));
    static constexpr int KS = RB + 16;
    static constexpr size_t k_off = 0;
    static constexpr size_t v_off = k_off + static_cast<size_t>(MK) * KS;
    static constexpr size_t q_off = v_off + static_cast<size_t>(MK) * RB;
    static constexpr size_t p_off = q_off + HC * kD * 4;
    static constexpr size_t r_off = p_off + HC * MK * 4;
    static constexpr size_t ml_off = r_off + static_cast<size_t>(NQ) * HC * kD * 4;
    static constexpr size_t w_off = ml_off + ((2 * HC * 4 + 15) / 16) * 16;       // merge weights [HC][32]
    static constexpr size_t ml2_off = w_off + HC * 32 * 4;                          // merged (M, L) [HC][2]
    static constexpr size_t ptr_off = ml2_off + ((2 * HC * 4 + 15) / 16) * 16;
    static constexpr size_t bytes = ptr_off + 2 * static_cast<size_t>(MK) * 8;
};

// CLU: the splits of a head group are one thread-block cluster (<= 16 CTAs, 512
// threads, up to 256 keys each) and merge through distributed shared memory — no
// global partials, no ticket; otherwise the last CTA (ticket) merges from global.
template <typename T, int HC, bool EXT, int NT = kBsaThreads, int MK = kBsaMaxKeys, bool CLU = false>
__global__ void __launch_bounds__(NT, 1)
decode_bsa_kernel(const hp_decode_bsa_args a, float* part, int* tickets, int splits, int kpc) {
    pdl_trigger();
    constexpr int NQ = NT / 64;  // PV key groups of 32
    static_assert(MK / NQ == 32, "PV assumes 32 keys per group");
    using S = BsaSmem<T, HC, MK, NQ>;
    constexpr int RB = S::RB, KS = S::KS;
    constexpr int half = kD / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    const int cut = CLU ? -1 : dev_cut_point(2);  // a cut CTA would strand its cluster at the barrier
    if (cut == 0) return;
    unsigned char* Ks = smem + S::k_off;
    unsigned char* Vs = smem + S::v_off;
    float* qs = reinterpret_cast<float*>(smem + S::q_off);
    float* ps = reinterpret_cast<float*>(smem + S::p_off);
    float* red = reinterpret_cast<float*>(smem + S::r_off);
    float* ml = reinterpret_cast<float*>(smem + S::ml_off);
    float* ml2 = reinterpret_cast<float*>(smem + S::ml2_off);
    unsigned long long* kptr = reinterpret_cast<unsigned long long*>(smem + S::ptr_off);  // row addresses
    unsigned long long* vptr = kptr + MK;
    __shared__ int sh_last;

    const int t = threadIdx.x, lane = t & 31, w = warp_id();
    const int split = blockIdx.x, hg = blockIdx.y;
    const int h0 = hg * HC;
    const int mask = h0 / a.heads_per_mask;
    const int kvh = h0 / (a.n_q_heads / a.kv.n_kv);
    const int64_t pos = a.query_position;
    const int64_t sink_end = min64(a.sink_tokens, pos + 1);
    int64_t stream_begin = pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0;
    stream_begin = max64(stream_begin, sink_end);
    // PDL prologue: with a stable mask (resident KV) every row but the newest token's is
    // final before this launch, so CTAs without the newest row gather before the wait
    const bool early_ok = !EXT && a.mask_stable != 0 && a.kv.page_table == nullptr;
    if (!early_ok) pdl_wait();
    const int64_t n_mask = a.mask_count[mask];
    const int64_t n_sel = sink_end + n_mask + (pos + 1 - stream_begin);
    const int64_t p0 = static_cast<int64_t>(split) * kpc;
    const int nv = static_cast<int>(max64(0, min64(kpc, n_sel - p0)));
    const bool early = early_ok && p0 + nv < n_sel;  // the newest token (= last selected) is not here
    if (early_ok && !early) pdl_wait();
    const float scale = 1.0f / sqrtf(static_cast<float>(kD));

    trace(2, 0);
    // ---- 1. tokens, then the K/V rows with 16-byte cp.async: a warp moves one row pair
    //         (K row by lanes 0-15, V row by lanes 16-31 for bf16) per instruction
    if (t < nv) {
        const int64_t p = p0 + t;
        const int64_t tok = p < sink_end ? p
                            : p < sink_end + n_mask ? ref_token(a.mask, mask, p - sink_end)
                                                    : stream_begin + (p - sink_end - n_mask);
        kptr[t] = reinterpret_cast<unsigned long long>(kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kvh, tok, sizeof(T)));
        vptr[t] = reinterpret_cast<unsigned long long>(kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kvh, tok, sizeof(T)));
    }
    if (cut == 5) return;
    __syncthreads();
    if (cut == 6) return;
    {
        // K rows first (group 0), then V rows (group 1): QK starts while V is in flight.
        // bf16: a warp instruction moves two 256 B rows (16 lanes each); fp32: one.
        constexpr int CH = RB / 16;
        constexpr int RPI = 32 / CH;
        const int c = lane % CH, sub = lane / CH;
#pragma unroll
        for (int i = 0; i < MK / (NT / 32) / RPI; ++i) {
            const int r = (i * (NT / 32) + w) * RPI + sub;
            if (r < nv) cp_async16(Ks + r * KS + c * 16, reinterpret_cast<const char*>(kptr[r]) + c * 16);
        }
        cp_async_commit();
#pragma unroll
        for (int i = 0; i < MK / (NT / 32) / RPI; ++i) {
            const int r = (i * (NT / 32) + w) * RPI + sub;
            if (r < nv) cp_async16(Vs + r * RB + c * 16, reinterpret_cast<const char*>(vptr[r]) + c * 16);
        }
        cp_async_commit();
    }
    if (early) pdl_wait();  // q (and everything after) is the preceding launch's to write
    for (int i = t; i < HC * kD; i += NT) qs[i] = a.q[static_cast<int64_t>(h0) * kD + i];
    if constexpr (EXT) {  // q at its true position (sparse_attention.cpp:47)
        __syncthreads();
        const float* cs = a.rope.cos_tab + pos * half;
        const float* sn = a.rope.sin_tab + pos * half;
        for (int i = t; i < HC * half; i += NT) {
            const int hh = i / half, e = i - hh * half;
            float* row = qs + hh * kD;
            const float x = row[e], y = row[e + half], c = cs[e], s = sn[e];
            row[e] = x * c - y * s;
            row[e + half] = x * s + y * c;
        }
    }
    trace(2, 1);
    if (cut == 7) return;
    cp_async_wait_group<1>();  // K rows landed
    __syncthreads();
    trace(2, 2);
    if (cut == 1) return;

    // ---- 2. QK: key j = jb + w*16 + (lane & 15), elements [hf*64, hf*64 + 64)
    for (int jb = 0; jb < kpc; jb += (NT / 32) * 16) {
        const int j = jb + w * 16 + (lane & 15), hf = lane >> 4;
        float acc[HC];
#pragma unroll
        for (int hh = 0; hh < HC; ++hh) acc[hh] = 0.f;
        if (j < nv) {
            const unsigned char* kr = Ks + j * KS;
            if constexpr (!EXT) {
                constexpr int EPC = 16 / sizeof(T);
#pragma unroll
                for (int c = 0; c < RB / 32; ++c) {
                    const int cc = hf * (RB / 32) + c;
                    float kv8[EPC];
                    if constexpr (sizeof(T) == 2) {
                        const uint4 u = *reinterpret_cast<const uint4*>(kr + cc * 16);
                        kv8[0] = bf16_lo(u.x); kv8[1] = bf16_hi(u.x); kv8[2] = bf16_lo(u.y); kv8[3] = bf16_hi(u.y);
                        kv8[4] = bf16_lo(u.z); kv8[5] = bf16_hi(u.z); kv8[6] = bf16_lo(u.w); kv8[7] = bf16_hi(u.w);
                    } else {
                        const float4 f = *reinterpret_cast<const float4*>(kr + cc * 16);
                        kv8[0] = f.x; kv8[1] = f.y; kv8[2] = f.z; kv8[3] = f.w;
                    }
#pragma unroll
                    for (int hh = 0; hh < HC; ++hh) {
                        const float* qr = qs + hh * kD + cc * EPC;
#pragma unroll
                        for (int u = 0; u < EPC; u += 4) {
                            const float4 q4 = *reinterpret_cast<const float4*>(qr + u);
                            acc[hh] = fmaf(q4.x, kv8[u], acc[hh]);
                            acc[hh] = fmaf(q4.y, kv8[u + 1], acc[hh]);
                            acc[hh] = fmaf(q4.z, kv8[u + 2], acc[hh]);
                            acc[hh] = fmaf(q4.w, kv8[u + 3], acc[hh]);
                        }
                    }
                }
            } else {
                // streaming_positions (rope_policy.cpp:59-72): key at pos + 1 - n_sel + p
                const int64_t kpos = pos + 1 - n_sel + (p0 + j);
                const float* cs = a.rope.cos_tab + kpos * half;
                const float* sn = a.rope.sin_tab + kpos * half;
                const T* kt = reinterpret_cast<const T*>(kr);
                for (int e = 0; e < half; ++e) {
                    const float x = load_elem(kt, e), y = load_elem(kt, e + half);
                    const float c = __ldg(cs + e), s = __ldg(sn + e);
                    const float r = hf ? x * s + y * c : x * c - y * s;
#pragma unroll
                    for (int hh = 0; hh < HC; ++hh) acc[hh] = fmaf(qs[hh * kD + hf * half + e], r, acc[hh]);
                }
            }
        }
#pragma unroll
        for (int hh = 0; hh < HC; ++hh) acc[hh] += __shfl_xor_sync(0xffffffffu, acc[hh], 16);
        if (hf == 0 && j < MK) {
#pragma unroll
            for (int hh = 0; hh < HC; ++hh) ps[hh * MK + j] = j < nv ? acc[hh] * scale : -INFINITY;
        }
    }
    __syncthreads();
    trace(2, 3);
    if (cut == 2) return;
    // ---- 3. softmax pieces per head
    {  // every warp runs a head's reduction (warps >= HC redo head w % HC and discard it):
       // no warp-index branch around the shuffles
        const int hw = w % HC;
        const bool mine = w < HC;
        float* pr = ps + hw * MK;
        float mx = -INFINITY;
        for (int j = lane; j < nv; j += 32) mx = fmaxf(mx, pr[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float l = 0.f;
        float pv[MK / 32];
#pragma unroll
        for (int i = 0; i < MK / 32; ++i) {
            const int j = i * 32 + lane;
            pv[i] = (j < nv && mx != -INFINITY) ? expf(pr[j] - mx) : 0.f;
            l += pv[i];
        }
        l = warp_sum(l);
        __syncthreads();  // every warp has read its scores before the owners overwrite them
        if (mine) {
#pragma unroll
            for (int i = 0; i < MK / 32; ++i) pr[i * 32 + lane] = pv[i];
            if (lane == 0) { ml[2 * w] = mx; ml[2 * w + 1] = l; }
        }
    }
    cp_async_wait_all();  // V rows landed
    __syncthreads();
    // ---- PV: element pair d2, key quarter kq
    {
        const int d2 = t & 63, kq = t >> 6;
        float o0[HC], o1[HC];
#pragma unroll
        for (int hh = 0; hh < HC; ++hh) o0[hh] = o1[hh] = 0.f;
        const int j0 = kq * (MK / NQ), j1 = min(nv, j0 + MK / NQ);
        for (int j = j0; j < j1; ++j) {
            float vx, vy;
            if constexpr (sizeof(T) == 2) {
                const uint32_t u = *reinterpret_cast<const uint32_t*>(Vs + j * RB + d2 * 4);
                vx = bf16_lo(u); vy = bf16_hi(u);
            } else {
                const float2 f = *reinterpret_cast<const float2*>(Vs + j * RB + d2 * 8);
                vx = f.x; vy = f.y;
            }
#pragma unroll
            for (int hh = 0; hh < HC; ++hh) {
                const float p = ps[hh * MK + j];
                o0[hh] = fmaf(p, vx, o0[hh]);
                o1[hh] = fmaf(p, vy, o1[hh]);
            }
        }
#pragma unroll
        for (int hh = 0; hh < HC; ++hh) {
            red[(kq * HC + hh) * kD + 2 * d2] = o0[hh];
            red[(kq * HC + hh) * kD + 2 * d2 + 1] = o1[hh];
        }
    }
    __syncthreads();
    trace(2, 4);
    if (cut == 3) return;
    if constexpr (CLU) {
        // ---- 4'. merge across the cluster: this split's (m, l) and summed o stay in its
        //          shared memory; after one cluster barrier every CTA reads all splits'
        //          (m, l) and merges its slice of the outputs over DSMEM
        for (int idx = t; idx < HC * kD; idx += NT) {
            const int hh = idx / kD, e = idx - hh * kD;
            float o = red[hh * kD + e];
#pragma unroll
            for (int g = 1; g < NQ; ++g) o += red[(g * HC + hh) * kD + e];
            red[idx] = o;
        }
        cluster_sync_all();
        const unsigned rank = cluster_ctarank(), ncl = cluster_nctarank();
        float* wts = reinterpret_cast<float*>(smem + S::w_off);  // [HC][32]: weights, then M, L at [HC*32 + 2*hh]
        {
            const int hh = w % HC;
            const bool mine = w < HC;
            float mo = -INFINITY, lo = 0.f;
            if (static_cast<unsigned>(lane) < ncl) {
                const uint32_t r = dsmem_addr(ml, lane);
                mo = ld_dsmem(r + 8 * hh);
                lo = ld_dsmem(r + 8 * hh + 4);
            }
            float M = lo > 0.f ? mo : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            const float f = lo > 0.f ? expf(mo - M) : 0.f;
            const float L = warp_sum(lo * f);
            if (mine) wts[hh * 32 + lane] = f;
            if (mine && lane == 0) { ml2[2 * hh] = M; ml2[2 * hh + 1] = L; }
        }
        __syncthreads();
        const int chunk = (HC * kD + static_cast<int>(ncl) - 1) / static_cast<int>(ncl);
        const int i0 = static_cast<int>(rank) * chunk, i1 = min(HC * kD, i0 + chunk);
        for (int idx = i0 + t; idx < i1; idx += NT) {
            const int hh = idx / kD, e = idx - hh * kD;
            float o = 0.f;
            for (unsigned sr = 0; sr < ncl; ++sr) o = fmaf(ld_dsmem(dsmem_addr(red + idx, sr)), wts[hh * 32 + sr], o);
            const float M = ml2[2 * hh], L = ml2[2 * hh + 1];
            const int64_t h = h0 + hh;
            a.out[h * kD + e] = L > 0.f ? o / L : NAN;
            if (a.part_o) a.part_o[h * kD + e] = L > 0.f ? o / L : 0.f;
            if (e == 0 && a.part_m) { a.part_m[h] = M; a.part_l[h] = L; }
        }
        cluster_sync_all();  // no CTA leaves while its shared memory may still be read
        return;
    }
    float* pbase = part + static_cast<int64_t>(hg) * splits * HC * kBsaRec;
    for (int idx = t; idx < HC * kD; idx += NT) {
        const int hh = idx / kD, e = idx - hh * kD;
        float o = red[hh * kD + e];
#pragma unroll
        for (int g = 1; g < NQ; ++g) o += red[(g * HC + hh) * kD + e];
        float* pp = pbase + (static_cast<int64_t>(split) * HC + hh) * kBsaRec;
        if (e == 0) { pp[0] = ml[2 * hh]; pp[1] = ml[2 * hh + 1]; }
        pp[4 + e] = o;
    }
    if (cut == 4) return;
    const bool last_cta = cta_ticket_last(&tickets[hg], splits, &sh_last);
    trace(2, 6);
    if (!last_cta) return;
    // ---- 4. merge every split of this head group (log-sum-exp). One L2 round trip:
    //         the first records land in the K/V shared memory by cp.async while every
    //         split's (m, l) is read into the PV scratch.
    float* mlp = red;  // [splits][HC][2] (m, l) -> (weight, l); splits <= 2 * kD (host check)
    constexpr int kStaged = static_cast<int>(S::q_off / (HC * kBsaRec * 4));
    const int sb = min(splits, kStaged);
    {
        const char* src = reinterpret_cast<const char*>(pbase);
        const int n16 = sb * HC * kBsaRec / 4;
        for (int i = t; i < n16; i += NT) cp_async16(smem + i * 16, src + i * 16);
        cp_async_commit();
        for (int i = t; i < splits * HC; i += NT) {
            const float* pp = pbase + static_cast<int64_t>(i) * kBsaRec;
            mlp[2 * i] = __ldcg(pp);
            mlp[2 * i + 1] = __ldcg(pp + 1);
        }
        cp_async_wait_all();
    }
    __syncthreads();
    {  // head reductions on every warp (warps >= HC discard theirs), no warp-index branch
        const int hh = w % HC;
        const bool mine = w < HC;
        float M = -INFINITY;
        for (int s = lane; s < splits; s += 32)
            if (mlp[2 * (s * HC + hh) + 1] > 0.f) M = fmaxf(M, mlp[2 * (s * HC + hh)]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        float L = 0.f;
        for (int s = lane; s < splits; s += 32) {
            const float l = mlp[2 * (s * HC + hh) + 1];
            const float f = l > 0.f ? expf(mlp[2 * (s * HC + hh)] - M) : 0.f;
            L += l * f;
        }
        L = warp_sum(L);
        __syncthreads();
        if (mine) {
            for (int s = lane; s < splits; s += 32) {
                const float l = mlp[2 * (s * HC + hh) + 1];
                mlp[2 * (s * HC + hh)] = l > 0.f ? expf(mlp[2 * (s * HC + hh)] - M) : 0.f;  // weight replaces m
            }
            if (lane == 0) { ml[2 * hh] = M; ml[2 * hh + 1] = L; }
        }
    }
    __syncthreads();
    trace(2, 5);
    const float* staged = reinterpret_cast<const float*>(smem);
    for (int idx = t; idx < HC * kD; idx += NT) {
        const int hh = idx / kD, e = idx - hh * kD;
        float o = 0.f;
        for (int s = 0; s < sb; ++s) o = fmaf(staged[(s * HC + hh) * kBsaRec + 4 + e], mlp[2 * (s * HC + hh)], o);
        for (int s = sb; s < splits; ++s)  // records beyond the staging room (large selections)
            o = fmaf(__ldcg(pbase + static_cast<int64_t>(s * HC + hh) * kBsaRec + 4 + e), mlp[2 * (s * HC + hh)], o);
        const float M = ml[2 * hh], L = ml[2 * hh + 1];
        const int64_t h = h0 + hh;
        a.out[h * kD + e] = L > 0.f ? o / L : NAN;
        if (a.part_o) a.part_o[h * kD + e] = L > 0.f ? o / L : 0.f;
        if (e == 0 && a.part_m) { a.part_m[h] = M; a.part_l[h] = L; }
    }
    trace(2, 7);
}

// ------------------------------------------------------------------ materialize
struct MatArgs {
    hp_list_ref ref[4];
    const int32_t* count[4];
    int32_t* out[4];
    int64_t stride[4];
};

__global__ void materialize_kernel(const MatArgs a) {
    pdl_trigger();
    pdl_wait();
    const int l = blockIdx.z, m = blockIdx.y;
    const int64_t n = a.count[l][m];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        a.out[l][m * a.stride[l] + i] = static_cast<int32_t>(ref_token(a.ref[l], m, i));
}


int bsa_hc(int n_q_heads, int n_kv, int hpm) {
    const int g = n_q_heads / n_kv;
    int hc = std::__gcd(g, hpm);
    hc = std::__gcd(hc, kMaxHC);
    return std::max(1, hc);
}

// Which descent kernel a stage launch takes (hp_decode_stage_variant): the one-wave
// kernel for big stages, all-rows for short chunks, lookahead for latency-bound bf16
// descents, the classic kernel otherwise (and always with RoPE extension).
int stage_variant(const hp_decode_stage_args& a, size_t elem) {
    const bool ext = a.rope.extension != 0;
    const int hpm = a.heads_per_mask;
    const int groups = (a.max_chunks + 31) / 32;
    const int64_t wide_items = static_cast<int64_t>(a.n_masks) * groups * hpm;
    // from half a wave of descents up the stage is bandwidth-bound and the one-wave kernel
    // (1.0x bytes) beats the lookahead kernel (1.33x); below it the halved round count
    // wins (measured at 1M: 4 groups 32.6 vs 41.2 us; 2 groups 24.1 vs 21.7; 1 group 22.1 vs 18.2)
    if (a.scores_out == nullptr && a.chunk_size > 8 && hpm <= 8 &&
        align_up(static_cast<size_t>(a.n_masks) * 4, 256) + static_cast<size_t>(a.n_masks) * hpm * a.max_chunks * 4 <=
            a.workspace_bytes &&
        wide_items >= 2048)
        return HP_STAGE_WIDE;
    if (a.chunk_size <= 8 && 32 % a.chunk_size == 0 && (a.n_q_heads / a.keys.n_kv) % hpm == 0)
        return HP_STAGE_ALLROWS;
    if (!ext && elem == 2 && kLookahead) return HP_STAGE_LOOKAHEAD;
    return HP_STAGE_CLASSIC;
}

template <typename T, bool EXT>
cudaError_t launch_stage(const hp_decode_stage_args& a, float* scores, int* tickets, cudaStream_t s) {
    using G = RowGeom<T>;
    const int hpm = a.heads_per_mask;
    int cg = std::max(1, kStageWarps / hpm);
    const int warps = std::min(kStageWarps, std::max(hpm * cg, 1));
    const int threads = std::max(32, std::min(warps, hpm * cg) * 32);
    const int nw = threads / 32;
    const size_t smem = static_cast<size_t>(nw) * 32 * G::stride + static_cast<size_t>(hpm) * kD * 6 +
                        static_cast<size_t>(hpm) * 32 * cg * 4;
    cudaError_t e;
    int head_planes = 1;
    const int groups = (a.max_chunks + 31) / 32;
    const int64_t wide_items = static_cast<int64_t>(a.n_masks) * groups * hpm;
    const int variant = stage_variant(a, sizeof(T));
    if (variant == HP_STAGE_WIDE) {
        // big stage: one wave of 7-warp CTAs, per-head scores (decode_stage_wide_kernel)
        // + one rotated q per warp with RoPE extension (3 CTAs per SM then)
        const size_t smem3 = static_cast<size_t>(kWideWarps) * 32 * G::stride + (EXT ? kWideWarps * kD * 4 : 0);
        auto k3 = decode_stage_wide_kernel<T, EXT>;
        e = cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem3));
        if (e != cudaSuccess) return e;
        head_planes = hpm;
        e = launch_pdl(k3, dim3(static_cast<unsigned>((wide_items + kWideWarps - 1) / kWideWarps)), dim3(kWideWarps * 32),
                       smem3, s, a, scores, groups);
    } else if (variant == HP_STAGE_ALLROWS) {
        // short chunks: gather every row of a chunk at once (decode_stage_allrows_kernel)
        const size_t smem2 = static_cast<size_t>(kAllRowsWarps) * 32 * G::stride + static_cast<size_t>(hpm) * kD * 6;
        const int per_cta = kAllRowsWarps * (32 / a.chunk_size);
        auto k2 = decode_stage_allrows_kernel<T, EXT>;
        e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2));
        if (e != cudaSuccess) return e;
        e = launch_pdl(k2, dim3((a.max_chunks + per_cta - 1) / per_cta, a.n_masks), dim3(kAllRowsWarps * 32), smem2, s,
                       a, scores);
    } else if (variant == HP_STAGE_LOOKAHEAD) {
        // latency-bound descents: two comparisons per gather round (decode_stage_look_kernel)
        const size_t smem4 = static_cast<size_t>(nw) * kLookSlots * 32 * G::stride + static_cast<size_t>(nw) * kD * 6 +
                             static_cast<size_t>(hpm) * 32 * cg * 4;
        auto k4 = decode_stage_look_kernel;
        e = cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4));
        if (e != cudaSuccess) return e;
        dim3 grid((a.max_chunks + 32 * cg - 1) / (32 * cg), a.n_masks);
        const int64_t lanes = static_cast<int64_t>(a.n_masks) * a.max_chunks * hpm;
        e = launch_pdl(k4, grid, dim3(threads), smem4, s, a, scores, cg, lanes <= 65536 ? 1 : 0);
    } else {
        auto kern = decode_stage_kernel<T, EXT>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        dim3 grid((a.max_chunks + 32 * cg - 1) / (32 * cg), a.n_masks);
        // speculative next-row prefetch only where the stage is latency-bound (few descents)
        const int64_t lanes = static_cast<int64_t>(a.n_masks) * a.max_chunks * hpm;
        const int prefetch = lanes <= 65536 ? 1 : 0;
        e = launch_pdl(kern, grid, dim3(threads), smem, s, a, scores, tickets, cg, prefetch);
    }
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (a.sel_out == nullptr) return cudaSuccess;  // descent only: scores stay in the workspace
    // keys[max_chunks] + kept ids[K]: sized to the stage so the selection CTAs fit next to
    // the descent CTAs still draining (they launch early under PDL)
    const size_t tsmem = static_cast<size_t>((a.max_chunks + 3) & ~3) * 4 +
                         static_cast<size_t>(std::max(1, a.keep / a.chunk_size)) * 4;
    e = cudaFuncSetAttribute(decode_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem));
    if (e != cudaSuccess) return e;
    e = launch_pdl(decode_topk_kernel, dim3(a.n_masks), dim3(kTopkThreads2), tsmem, s, a,
                   static_cast<const float*>(a.scores_out ? a.scores_out : scores), head_planes);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int HC, bool EXT>
cudaError_t launch_bsa(const hp_decode_bsa_args& a, float* part, int* tickets, int splits, int kpc, cudaStream_t s) {
    using S = BsaSmem<T, HC>;
    if (splits > 2 * kD) return cudaErrorInvalidValue;  // (m, l) of every split fit the PV scratch
    auto kern = decode_bsa_kernel<T, HC, EXT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::bytes));
    if (e != cudaSuccess) return e;
    e = launch_pdl(kern, dim3(splits, a.n_q_heads / HC), dim3(kBsaThreads), S::bytes, s, a, part, tickets, splits, kpc);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// cluster variant: grid (splits, groups), cluster (splits, 1, 1), bf16 without RoPE
constexpr int kBsaCluThreads = 512, kBsaCluMaxKeys = 256, kBsaMaxCluster = 16;
template <int HC>
cudaError_t launch_bsa_cluster(const hp_decode_bsa_args& a, int splits, int kpc, cudaStream_t s,
                               bool query_only = false) {
    using S = BsaSmem<bf16_t, HC, kBsaCluMaxKeys, kBsaCluThreads / 64>;
    auto kern = decode_bsa_kernel<bf16_t, HC, false, kBsaCluThreads, kBsaCluMaxKeys, true>;
    static int checked_splits[kBsaMaxCluster + 1] = {};  // max active clusters, -1 = none
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::bytes));
    if (e != cudaSuccess) return e;
    if (splits > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(splits, a.n_q_heads / HC);
    cfg.blockDim = dim3(kBsaCluThreads);
    cfg.dynamicSmemBytes = S::bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = splits;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (checked_splits[splits] == 0) {  // how many clusters of this size fit at once (GPC-bound)
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        checked_splits[splits] = (e == cudaSuccess && n > 0) ? n : -1;
        cudaGetLastError();
    }
    // every head group's cluster resident in one wave, else the ticket path is faster
    // (B200, 162 KB CTAs: 7 clusters of 11-16 fit, 15 of 7-9)
    if (checked_splits[splits] < static_cast<int>(cfg.gridDim.y)) return cudaErrorNotSupported;
    if (query_only) return cudaSuccess;
    e = cudaLaunchKernelEx(&cfg, kern, a, static_cast<float*>(nullptr), static_cast<int*>(nullptr), splits, kpc);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, bool EXT>
cudaError_t dispatch_bsa_hc(const hp_decode_bsa_args& a, int hc, float* part, int* tickets, int splits, int kpc,
                            cudaStream_t s) {
    switch (hc) {
        case 1: return launch_bsa<T, 1, EXT>(a, part, tickets, splits, kpc, s);
        case 2: return launch_bsa<T, 2, EXT>(a, part, tickets, splits, kpc, s);
        case 4: return launch_bsa<T, 4, EXT>(a, part, tickets, splits, kpc, s);
        default: return launch_bsa<T, 8, EXT>(a, part, tickets, splits, kpc, s);
    }
}

// keys per CTA: enough CTAs to cover the SMs once, at most kBsaMaxKeys
int bsa_keys_per_cta(int64_t max_sel, int groups) {
    const int64_t want = (max_sel * groups + 147) / 148;
    int64_t k = (want + 15) / 16 * 16;
    k = std::max<int64_t>(kBsaMinKeys, std::min<int64_t>(kBsaMaxKeys, k));
    return static_cast<int>(k);
}

}  // namespace

// Developer instrumentation: record per-CTA phase stamps of kernel `kernel_id`
// (1 = decode stage, 2 = decode BSA) into buf [n_cta][8] (NULL disables).
#if defined(HP_TRACE) || defined(HP_DEV)  // developer hooks: dev builds only (include/hipprune_b200_dev.h)
extern "C" int hp_debug_cut(int kernel_id, int at) {
    if (int rc = hph::check_cuda(cudaMemcpyToSymbol(g_cut_kernel, &kernel_id, sizeof(int)), "hp_debug_cut")) return rc;
    return hph::check_cuda(cudaMemcpyToSymbol(g_cut_at, &at, sizeof(int)), "hp_debug_cut");
}

extern "C" int hp_trace_enable(unsigned long long* buf, int kernel_id) {
    if (int rc = hph::check_cuda(cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(buf)), "hp_trace_enable")) return rc;
    return hph::check_cuda(cudaMemcpyToSymbol(g_trace_kernel, &kernel_id, sizeof(int)), "hp_trace_enable");
}
#endif

// tickets, then chunk scores with room for up to kWideHeadPlanes per-head planes (the
// one-wave kernel keeps every head's representative score; the selection maxes them)
constexpr int kWideHeadPlanes = 8;
extern "C" size_t hp_decode_stage_workspace_bytes(int32_t n_masks, int32_t max_chunks) {
    return align_up(static_cast<size_t>(n_masks) * 4, 256) +
           align_up(static_cast<size_t>(n_masks) * kWideHeadPlanes * std::max(1, max_chunks) * 4, 256);
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
    if (a.sel_out && a.sel_stride < a.keep / a.chunk_size) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: sel_stride < k/l_c");
    if (a.max_chunks <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: max_chunks must be >= 1");
    if (a.max_chunks > kTopkMaxKeys)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: %d chunks per list exceed the fused selection limit %d",
                              a.max_chunks, kTopkMaxKeys);
    const size_t need = hp_decode_stage_workspace_bytes(a.n_masks, a.max_chunks);
    if (!a.workspace || a.workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage: workspace too small");
    // identity stages (pruning.cpp:159-168) never rotate, so the reference never range-checks
    // them: skip the check when the stage is provably the identity from host-known bounds
    const int64_t kk = a.keep / a.chunk_size;
    const bool identity = a.in_count ? a.max_chunks <= kk
                                     : (a.in_count_const <= a.keep || (a.in_count_const + a.chunk_size - 1) / a.chunk_size <= kk);
    if (a.rope.extension && !identity) {
        const int pol = a.rope.layer > a.rope.early_cutoff ? a.rope.late_policy : a.rope.early_policy;
        if (pol != HP_ROPE_CHUNK_INDEXED && pol != HP_ROPE_RELATIVE)
            return hph::set_error(HP_LOGIC_ERROR, "query_position: policy not applicable to pruning");
        const int64_t need_q = pol == HP_ROPE_RELATIVE ? a.stream_tokens + 1 : min64(a.query_position, a.max_chunks + a.stream_tokens);
        const int64_t need_k = pol == HP_ROPE_RELATIVE ? 1 : a.max_chunks - 1;
        if (std::max(need_q, need_k) >= a.rope.rope_max)
            return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                                  static_cast<long long>(std::max(need_q, need_k)), static_cast<long long>(a.rope.rope_max));
    }
    // tickets first (they stay zero between launches), then the chunk scores
    char* ws = static_cast<char*>(a.workspace);
    int* tickets = reinterpret_cast<int*>(ws);
    const size_t off = align_up(static_cast<size_t>(a.n_masks) * 4, 256);
    float* scores = reinterpret_cast<float*>(ws + off);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool ext = a.rope.extension != 0;
    cudaError_t e;
    if (a.keys.dtype == HP_BF16) e = ext ? launch_stage<bf16_t, true>(a, scores, tickets, s) : launch_stage<bf16_t, false>(a, scores, tickets, s);
    else e = ext ? launch_stage<float, true>(a, scores, tickets, s) : launch_stage<float, false>(a, scores, tickets, s);
    return hph::check_cuda(e, "decode_stage_kernel");
}

extern "C" int hp_select_topk(const float* scores, int64_t stride, int32_t n_masks, const int32_t* n_in,
                              int64_t n_in_const, int32_t chunk_size, int32_t keep, int32_t* sel_out,
                              int32_t sel_stride, int32_t* out_count, void* stream) {
    if (!scores || !sel_out || !out_count || n_masks <= 0 || stride <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk: bad arguments");
    if (chunk_size <= 0 || keep <= 0 || keep % chunk_size)
        return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: k must be a positive multiple of l_c");
    if (sel_stride < keep / chunk_size) return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk: sel_stride < k/l_c");
    if (stride > kTopkMaxKeys)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk: %lld chunks exceed the selection limit %d",
                              static_cast<long long>(stride), kTopkMaxKeys);
    hp_decode_stage_args a{};
    a.chunk_size = chunk_size;
    a.keep = keep;
    a.n_masks = n_masks;
    a.in_count = n_in;
    a.in_count_const = n_in_const;
    a.max_chunks = static_cast<int32_t>(stride);
    a.sel_stride = sel_stride;
    a.sel_out = sel_out;
    a.out_count = out_count;
    const size_t tsmem = static_cast<size_t>((stride + 3) & ~3) * 4 + static_cast<size_t>(keep / chunk_size) * 4;
    cudaError_t e = cudaFuncSetAttribute(decode_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem));
    if (e == cudaSuccess)
        e = launch_pdl(decode_topk_kernel, dim3(n_masks), dim3(kTopkThreads2), tsmem, static_cast<cudaStream_t>(stream), a,
                       scores, 1);
    return hph::check_cuda(e, "decode_topk_kernel");
}

// ------------------------------------------------------- sequence-sharded selection
// C5: every rank all-gathered every rank's chunk scores of the stage ([R][M][W], rank r's
// first counts[r][m] valid, ranks in global chunk order). One CTA per mask rebuilds the
// global score vector in shared memory, runs the same exact top-K as the unsharded stage
// (so every rank holds the same global selection), then cuts out this rank's part: the
// kept chunks inside its range as local ids and its output length (the globally last
// chunk may be short).
constexpr int kShardMaxRanks = 64;
__global__ void __launch_bounds__(kTopkThreads2)
select_sharded_kernel(const float* gathered, const int32_t* counts, int R, int W, int rank, const int32_t* n_in,
                      int64_t n_in_const, int lc, int keep, int32_t* sel_g, int sel_stride, int32_t* cnt_g,
                      int32_t* sel_l, int32_t* len_l) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ TopkShared sh;
    __shared__ int starts[kShardMaxRanks + 1];
    const int m = blockIdx.x, M = gridDim.x, t = threadIdx.x, nt = blockDim.x;
    if (t == 0) {
        int acc = 0;
        for (int r = 0; r < R; ++r) { starts[r] = acc; acc += counts[r * M + m]; }
        starts[R] = acc;
    }
    __syncthreads();
    const int64_t n = n_in ? n_in[m] : n_in_const;
    const int cc = static_cast<int>((n + lc - 1) / lc);
    const int K = keep / lc;
    uint32_t* keys = reinterpret_cast<uint32_t*>(tsm);
    int32_t* ssel = reinterpret_cast<int32_t*>(keys + ((R * W + 3) & ~3));
    int nsel;
    int64_t n_out;
    if (n <= keep || cc <= K) {  // identity (pruning.cpp:159-168)
        for (int j = t; j < cc; j += nt) ssel[j] = j;
        nsel = cc;
        n_out = n;
        __syncthreads();
    } else {
        for (int j = t; j < cc; j += nt) {
            int r = 0;
            while (r + 1 < R && starts[r + 1] <= j) ++r;
            keys[j] = order_key(__ldcg(gathered + (static_cast<int64_t>(r) * M + m) * W + (j - starts[r])));
        }
        __syncthreads();
        cta_topk_smem(keys, cc, K, ssel, sh);
        nsel = K;
        n_out = static_cast<int64_t>(K - 1) * lc + min64(lc, n - static_cast<int64_t>(ssel[K - 1]) * lc);
    }
    for (int j = t; j < nsel; j += nt) sel_g[static_cast<int64_t>(m) * sel_stride + j] = ssel[j];
    // this rank's part: the kept ids are ascending, so the ones in [lo, hi) are contiguous
    const int lo = starts[rank], hi = starts[rank + 1];
    int below = 0, inside = 0;
    for (int j = 0; j < nsel; ++j) {  // nsel <= a few thousand: every thread scans (no barrier)
        const int c = ssel[j];
        below += c < lo;
        inside += c >= lo && c < hi;
    }
    for (int j = t; j < inside; j += nt) sel_l[static_cast<int64_t>(m) * sel_stride + j] = ssel[below + j] - lo;
    if (t == 0) {
        cnt_g[m] = static_cast<int32_t>(n_out);
        const int last = cc - 1;
        const bool has_last = inside > 0 && ssel[below + inside - 1] == last && last >= lo && last < hi;
        const int64_t tail = n - static_cast<int64_t>(last) * lc;
        len_l[m] = static_cast<int32_t>(static_cast<int64_t>(inside) * lc - (has_last ? lc - tail : 0));
    }
}

extern "C" int hp_select_topk_sharded(const float* gathered, const int32_t* counts, int32_t n_ranks, int32_t width,
                                      int32_t rank, int32_t n_masks, const int32_t* n_in, int64_t n_in_const,
                                      int32_t chunk_size, int32_t keep, int32_t* sel_global, int32_t sel_stride,
                                      int32_t* count_global, int32_t* sel_local, int32_t* len_local, void* stream) {
    if (!gathered || !counts || !sel_global || !count_global || !sel_local || !len_local || n_masks <= 0 || width <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk_sharded: bad arguments");
    if (n_ranks <= 0 || n_ranks > kShardMaxRanks || rank < 0 || rank >= n_ranks)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk_sharded: rank %d of %d", rank, n_ranks);
    if (chunk_size <= 0 || keep <= 0 || keep % chunk_size)
        return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: k must be a positive multiple of l_c");
    if (sel_stride < keep / chunk_size) return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk_sharded: sel_stride < k/l_c");
    const int64_t total = static_cast<int64_t>(n_ranks) * width;
    if (total > kTopkMaxKeys)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_select_topk_sharded: %lld chunks exceed the selection limit %d",
                              static_cast<long long>(total), kTopkMaxKeys);
    const size_t tsmem = static_cast<size_t>((total + 3) & ~3) * 4 + static_cast<size_t>(std::max<int64_t>(keep / chunk_size, total)) * 4;
    cudaError_t e = cudaFuncSetAttribute(select_sharded_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem));
    if (e == cudaSuccess)
        e = launch_pdl(select_sharded_kernel, dim3(n_masks), dim3(kTopkThreads2), tsmem, static_cast<cudaStream_t>(stream),
                       gathered, counts, n_ranks, width, rank, n_in, n_in_const, chunk_size, keep, sel_global, sel_stride,
                       count_global, sel_local, len_local);
    if (e == cudaSuccess) e = cudaGetLastError();
    return hph::check_cuda(e, "select_sharded_kernel");
}

extern "C" size_t hp_decode_bsa_workspace_bytes(int32_t n_q_heads, int32_t max_sel) {
    const int splits = std::max(1, (max_sel + kBsaMinKeys - 1) / kBsaMinKeys);  // bound for any keys/CTA
    return align_up(static_cast<size_t>(n_q_heads) * splits * kBsaRec * 4, 256) + align_up(static_cast<size_t>(n_q_heads) * 4, 256);
}

// one cluster per head group when the selection fits 16 CTAs of <= 256 keys and every
// group's cluster is co-resident; false = the ticket-merge kernel
static bool try_bsa_cluster(const hp_decode_bsa_args& a, int64_t max_sel, int hc, cudaStream_t s, bool query_only) {
    if (a.kv.dtype != HP_BF16 || a.rope.extension || !kBsaUseCluster) return false;
    const int64_t kc = std::max<int64_t>(kBsaMaxKeys, ((max_sel + kBsaMaxCluster - 1) / kBsaMaxCluster + 15) / 16 * 16);
    const int sc = static_cast<int>((max_sel + kc - 1) / kc);
    if (!(kc <= kBsaCluMaxKeys && sc >= 2 && sc <= kBsaMaxCluster)) return false;
    cudaError_t e;
    switch (hc) {
        case 1: e = launch_bsa_cluster<1>(a, sc, static_cast<int>(kc), s, query_only); break;
        case 2: e = launch_bsa_cluster<2>(a, sc, static_cast<int>(kc), s, query_only); break;
        case 4: e = launch_bsa_cluster<4>(a, sc, static_cast<int>(kc), s, query_only); break;
        default: e = launch_bsa_cluster<8>(a, sc, static_cast<int>(kc), s, query_only); break;
    }
    if (e == cudaSuccess) return true;
    cudaGetLastError();  // not resident-able here: the ticket path
    return false;
}

static int decode_bsa_impl(const hp_decode_bsa_args* ap, void* stream, int* variant_out);

extern "C" int hp_decode_bsa(const hp_decode_bsa_args* ap, void* stream) { return decode_bsa_impl(ap, stream, nullptr); }

extern "C" int hp_decode_bsa_variant(const hp_decode_bsa_args* ap, int32_t* variant) {
    if (!variant) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa_variant: null output");
    int v = -1;
    const int rc = decode_bsa_impl(ap, nullptr, &v);
    *variant = v;
    return rc;
}

extern "C" int hp_decode_stage_variant(const hp_decode_stage_args* ap, int32_t* variant) {
    if (!ap || !variant) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_stage_variant: null pointer");
    *variant = stage_variant(*ap, ap->keys.dtype == HP_BF16 ? 2 : 4);
    return HP_OK;
}

static int decode_bsa_impl(const hp_decode_bsa_args* ap, void* stream, int* variant_out) {
    const bool query_only = variant_out != nullptr;
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: null args");
    const hp_decode_bsa_args& a = *ap;
    if (a.kv.d != kD) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: fused decode path needs head_dim 128");
    if (a.n_q_heads <= 0 || a.heads_per_mask <= 0 || a.kv.n_kv <= 0 || a.n_q_heads % a.kv.n_kv || a.n_q_heads % a.heads_per_mask)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: bad head geometry");
    if (!a.q || !a.out || !a.mask_count || !a.kv.k_pool || !a.kv.v_pool) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: null pointer");
    const int64_t pos = a.query_position;
    const int64_t sink_end = std::min<int64_t>(a.sink_tokens, pos + 1);
    const int64_t stream_begin = std::max<int64_t>(pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0, sink_end);
    // the selected set is a subset of [0, pos]: it never holds more than pos + 1 tokens,
    // so the grid is sized by the tighter of the two bounds (the reference's
    // streaming_positions check, sparse_attention.cpp:43-50, can then never fire)
    const int64_t max_sel = std::min<int64_t>(sink_end + a.max_mask + (pos + 1 - stream_begin), pos + 1);
    if (max_sel <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "attention_row: empty selected set");
    if (a.rope.extension && pos >= a.rope.rope_max)
        return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                              static_cast<long long>(pos), static_cast<long long>(a.rope.rope_max));
    const int hc = bsa_hc(a.n_q_heads, a.kv.n_kv, a.heads_per_mask);
    const int kpc = bsa_keys_per_cta(max_sel, a.n_q_heads / hc);
    const int splits = static_cast<int>((max_sel + kpc - 1) / kpc);
    const size_t need = hp_decode_bsa_workspace_bytes(a.n_q_heads, static_cast<int32_t>(max_sel));
    if (!a.workspace || a.workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_bsa: workspace too small");
    char* ws = static_cast<char*>(a.workspace);
    int* tickets = reinterpret_cast<int*>(ws);
    float* part = reinterpret_cast<float*>(ws + align_up(static_cast<size_t>(a.n_q_heads) * 4, 256));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool ext = a.rope.extension != 0;
    cudaError_t e;
    if (try_bsa_cluster(a, max_sel, hc, s, query_only)) {
        if (query_only) *variant_out = HP_BSA_CLUSTER;
        return HP_OK;
    }
    if (query_only) {
        *variant_out = HP_BSA_TICKET;
        return HP_OK;
    }
    if (a.kv.dtype == HP_BF16) e = ext ? dispatch_bsa_hc<bf16_t, true>(a, hc, part, tickets, splits, kpc, s) : dispatch_bsa_hc<bf16_t, false>(a, hc, part, tickets, splits, kpc, s);
    else e = ext ? dispatch_bsa_hc<float, true>(a, hc, part, tickets, splits, kpc, s) : dispatch_bsa_hc<float, false>(a, hc, part, tickets, splits, kpc, s);
    return hph::check_cuda(e, "decode_bsa_kernel");
}

__global__ void append_kernel(hp_kv_view kv, const unsigned char* k_rows,
                              const unsigned char* v_rows, int64_t token, int32_t* keys_exact) {
    pdl_trigger();
    pdl_wait();
    kv.touched = nullptr;  // the append is not a page access of any phase (decode.cpp:202-208)
    kv.row_bits = nullptr;
    const int eb = kv.dtype == HP_BF16 ? 2 : 4;
    const int row_bytes = kv.d * eb;
    const int h = blockIdx.x;
    // the row lands where the gathers will resolve it (slot or host tier); with a page
    // cache the host tier is written through, so an evicted page re-fetches it intact
    char* kd = const_cast<char*>(kv_row_ptr(kv, kv.k_pool, kv.k_host, h, token, eb));
    char* vd = kv.v_pool ? const_cast<char*>(kv_row_ptr(kv, kv.v_pool, kv.v_host, h, token, eb)) : nullptr;
    char* kh = nullptr;
    char* vh = nullptr;
    if (kv.page_table && kv.k_host) {
        const int64_t page = token / kv.page_size, off = token - page * kv.page_size;
        const int64_t o = (((page * kv.n_kv + h) * kv.page_size + off) * kv.d) * eb;
        if (kv.page_table[page] >= 0) {
            kh = const_cast<char*>(static_cast<const char*>(kv.k_host)) + o;
            if (kv.v_host) vh = const_cast<char*>(static_cast<const char*>(kv.v_host)) + o;
        }
    }
    bool ok = true;
    for (int i = threadIdx.x; i < row_bytes; i += blockDim.x) {
        kd[i] = k_rows[h * row_bytes + i];
        if (vd) vd[i] = v_rows[h * row_bytes + i];
        if (kh) kh[i] = k_rows[h * row_bytes + i];
        if (vh) vh[i] = v_rows[h * row_bytes + i];
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
    const cudaError_t e = launch_pdl(append_kernel, dim3(kv->n_kv), dim3(128), 0, static_cast<cudaStream_t>(stream), *kv,
                                     static_cast<const unsigned char*>(k_rows), static_cast<const unsigned char*>(v_rows),
                                     token, keys_exact);
    if (e != cudaSuccess) return hph::check_cuda(e, "append_kernel");
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
    // plain launch (no programmatic edge): the caches are usually refreshed on a side
    // branch of the step graph, off the layer's critical path (FusedDecodeLayer.run)
    materialize_kernel<<<dim3(blocks, n_masks, n_lists), dim3(256), 0, static_cast<cudaStream_t>(stream)>>>(m);
    return hph::check_cuda(cudaGetLastError(), "materialize_kernel");
}

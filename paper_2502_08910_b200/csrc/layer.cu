// Fused decode layer (d = 128, bf16 K/V, RoPE extension off): everything of the
// per-layer body of DecodeEngine::step after stage 0's descent in ONE kernel.
//
// Reference semantics (paths relative to /root/reference/proj):
//   stage chaining / caches        decode.cpp:225-249 (stage i consumes stage i-1)
//   identity, descent, top-K       pruning.cpp:69-98,153-200 (Alg. 3, stable top-K)
//   selected set, attention_row    sparse_attention.cpp:15-60,95-112
//
// B200 mapping. After stage 0 (131K independent descents at 1M: the one-wave kernel of
// decode.cu, HBM-bound), the rest of a layer step is a chain of small dependent pieces:
// stage-0 top-K, stage-1 descents (4K per KV group), top-K, stage-2 all-rows scoring,
// top-K, and a 3.3K-key attention with a split-K merge. As separate kernels every link
// pays a launch and a drain. Here a persistent grid owns the layer: n_SM / n_groups
// co-resident CTAs per KV group (one per SM: 18 per group for 8 groups, all 148 for one
// group — the 8-GPU KV-group split), and every link is a group barrier in L2:
//   * each CTA scores its slice of the stage's chunks — Alg. 3 descents (lane = chunk,
//     32 rows staged per warp with 16-byte cp.async), or all-rows scoring for l_c <= 8 —
//     and writes the chunk keys (max over the group's heads, order-mapped) to L2;
//   * one group barrier, every CTA copies the full key set and runs the same exact
//     radix top-K, so all hold the kept chunk ids and resolve the next stage's input
//     through shared memory (stage 0's keys need no exchange: every CTA forms them from
//     the descent kernel's L2-resident scores, so that selection has no barrier);
//   * the attention splits the selected positions over the CTAs (K/V gathered by
//     cp.async, QK^T and PV on mma.sync with bf16 hi/lo splits of q and p), the sink and
//     stream rows having been prefetched into L2 while the stages ran; partials (m, l, o)
//     go to L2 and the last CTA (acq_rel ticket) merges them.
// Measured and dropped: one thread-block cluster per group with DSMEM exchanges (8 CTAs
// per group: 107.8 vs 98.8 us per full-refresh layer — the phases are issue/latency
// bound on 8 SMs; 16-CTA clusters do not all fit).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "decode_dev.cuh"
#include "topk.cuh"

using namespace hpk;
using namespace hpk::dec;

namespace {

constexpr int kLT = 512;                              // threads per CTA
constexpr int kLW = kLT / 32;                         // warps per CTA
constexpr int kRow = kD * 2;                          // bf16 row bytes
constexpr int kSlot = 32 * kRow;                      // one 32-row staging slot (8 KB)
constexpr int kTile = 256;                            // attention keys per tile (K + V = 128 KB)
constexpr int kTileKV = 2 * kTile * kRow;             // 128 KB
// 140 KB: 16 warps x 8 KB of descent staging, or the attention tile + row pointers + p
constexpr int kPw = kTile + 8;                        // p row stride (floats): head rows 8 banks apart
constexpr int kStageBytes = kTileKV + 2 * kTile * 8 + 8 * kPw * 4;
constexpr int kMaxS = 4;
constexpr int kPart = kD + 2;                         // partial record: o[128], m, l
constexpr int kKeysMax = 16384;                       // chunk keys per stage selection
constexpr int kMaxGroupCtas = 160;                    // CTAs per KV group
constexpr int kBarInts = 4;                           // per mask: arrivals, generation, merge ticket, pad

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct LayerParams {
    hp_decode_layer_args a;
    uint32_t* gkeys;          // [2][n_masks][keys_cap] exchanged chunk keys (stage parity)
    float* gpart;             // [n_masks][CTAs][HP][kPart] attention partials
    int* gbar;                // [n_masks][kBarInts]
    const float* scores0;     // stage-0 chunk scores [m][planes0][max_chunks0]
    int32_t planes0;
    int32_t max_chunks0;
    int64_t n0;               // stage-0 input length
    int32_t keys_cap;         // order keys per buffer
    int32_t red_cap;          // per-head descent scores per CTA
    int32_t sel_off[kMaxS];   // offsets (ints) of each stage's kept ids in the shared sel area
    int32_t sel_total;
};

// Shared memory: the staging region is reused by phase — descents (a 32-row slot per
// warp), the selection's key copy (offset 0), the attention tile (K/V at 0, row pointers
// and probabilities behind it), the merge's staged partials; then the small arrays.
struct LayerSmem {
    size_t ptrs, pw, sel, qs, qb, qf, red, part, bytes;
    __host__ __device__ LayerSmem(int sel_total, int hp, int red_cap) {
        ptrs = kTileKV;                                      // K and V row pointers [2][kTile]
        pw = ptrs + 2 * kTile * 8;                           // [hp][kPw] scores / probabilities
        size_t o = kStageBytes;
        sel = o; o += align_up(static_cast<size_t>(sel_total) * 4, 16);
        qs = o; o += static_cast<size_t>(hp) * kD * 4;
        qb = o; o += static_cast<size_t>(hp) * kD * 2;
        qf = o; o += 8 * 2 * 2 * 32 * 4;                     // QK^T A fragments [k-step][half][hi, lo][lane]
        red = o; o += align_up(static_cast<size_t>(hp) * red_cap * 4, 16);
        part = o; o += align_up(static_cast<size_t>(hp) * kPart * 4, 16);
        bytes = o;
    }
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// D += A B, m16n8k16, bf16 inputs, fp32 accumulate (rows 8..15 of A unused here)
__device__ __forceinline__ void mma_bf16_16816(float& d0, float& d1, float& d2, float& d3, uint32_t a0, uint32_t a2,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t* r, const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

// Group barrier over the CTAs of one KV group: each CTA arrives with a fire-and-forget
// release add on a per-group counter and spins (acquire loads) until it reaches this
// barrier's target — n per barrier, the counter starting each launch at 0 (the last CTA
// to leave resets it). One L2 trip per arrival, no returned atomic on the critical path.
__device__ __forceinline__ void group_barrier(int* ctr, int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
        int v;
        do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

template <int HP>
__global__ void __launch_bounds__(kLT, 1) decode_layer_kernel(const LayerParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ TopkShared tsh;
    __shared__ float sh_m[HP], sh_l[HP], sh_alpha[HP];
    __shared__ int sh_last;
    const hp_decode_layer_args& a = P.a;
    const int m = blockIdx.y;
    const unsigned rank = blockIdx.x, CS = gridDim.x;
    const int t = threadIdx.x, lane = t & 31, w = warp_id();
    const LayerSmem L(P.sel_total, HP, P.red_cap);
    unsigned char* stage = smem;
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);  // the selection's copy (staging is idle then)
    const char** kptr = reinterpret_cast<const char**>(smem + L.ptrs);
    const char** vptr = kptr + kTile;
    float* pw = reinterpret_cast<float*>(smem + L.pw);
    int32_t* sel = reinterpret_cast<int32_t*>(smem + L.sel);
    float* qs = reinterpret_cast<float*>(smem + L.qs);
    uint32_t* qb = reinterpret_cast<uint32_t*>(smem + L.qb);
    uint32_t* qfr = reinterpret_cast<uint32_t*>(smem + L.qf);
    float* red = reinterpret_cast<float*>(smem + L.red);
    float* part = reinterpret_cast<float*>(smem + L.part);
    const int kvh = (m * HP) / (a.n_q_heads / a.kv.n_kv);  // the mask's heads share one kv head (host-checked)
    int* gbar = P.gbar + kBarInts * m;  // [0] barrier arrivals, [2] merge ticket, [3] exit ticket
    int n_bar = 0;

    trace(20, 0);
    pdl_wait();
    bool safe = true;
    for (int i = t; i < HP * kD; i += kLT) {
        const float x = a.q[static_cast<int64_t>(m * HP) * kD + i];
        qs[i] = x;
        safe &= q_product_safe(x);
    }
    // FFMA (FHFMA.BF16) dots only when every q*k product is exact (see decode.cu)
    const bool use_fma = __syncthreads_and(safe) && a.keys_exact != nullptr && *a.keys_exact != 0;
    for (int i = t; i < HP * kD / 2; i += kLT)
        qb[i] = (__float_as_uint(qs[2 * i]) >> 16) | (__float_as_uint(qs[2 * i + 1]) & 0xffff0000u);
    // the attention's QK^T A fragments (rows = heads, bf16 hi + lo parts of q), built once
    for (int i = t; i < 8 * 2 * 32; i += kLT) {
        const int ks = i >> 6, half = (i >> 5) & 1, ln = i & 31, gg = ln >> 2, tt = ln & 3;
        const int d = ks * 16 + half * 8 + 2 * tt;
        const float x0 = gg < HP ? qs[gg * kD + d] : 0.f, x1 = gg < HP ? qs[gg * kD + d + 1] : 0.f;
        const uint32_t h2 = pack_bf16(x0, x1);
        qfr[((ks * 2 + half) * 2) * 32 + ln] = h2;
        qfr[((ks * 2 + half) * 2 + 1) * 32 + ln] = pack_bf16(x0 - bf16_lo(h2), x1 - bf16_hi(h2));
    }

    // the attention's sink and stream rows are known now: warm them into L2 while the
    // stages run (the group's CTAs split them; K and V, two 128 B lines per row)
    const int64_t pos = a.query_position;
    const int64_t sink_end = min64(a.sink_tokens, pos + 1);
    const int64_t stream_begin = max64(pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0, sink_end);
    {
        const int64_t n_fixed = sink_end + (pos + 1 - stream_begin);
        for (int64_t x = static_cast<int64_t>(rank) * kLT + t; x < n_fixed; x += static_cast<int64_t>(CS) * kLT) {
            const int64_t tk = x < sink_end ? x : stream_begin + (x - sink_end);
            const char* kp = kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kvh, tk, 2);
            const char* vp = kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kvh, tk, 2);
            prefetch_l2(kp); prefetch_l2(kp + 128); prefetch_l2(vp); prefetch_l2(vp + 128);
        }
    }
    __syncthreads();
    trace(20, 1);

    // token at position p of stage i's output list (i = -1: stage 0's input range)
    auto resolve = [&](int i, int64_t p) -> int64_t {
#pragma unroll 1
        for (; i >= 0; --i) {
            if (!a.refresh[i]) return a.cache[i][static_cast<int64_t>(m) * a.cache_stride[i] + p];
            const int lc = a.chunk_size[i];
            const uint32_t p32 = static_cast<uint32_t>(p);
            const uint32_t r = p32 / static_cast<uint32_t>(lc);
            p = static_cast<int64_t>(sel[P.sel_off[i] + r]) * lc + (p32 - r * lc);
        }
        return a.sink_tokens + p;
    };
    int buf = 0;  // key buffer parity in L2: stage selections alternate between two buffers
    auto put_key = [&](int64_t c, uint32_t k) {
        P.gkeys[(static_cast<size_t>(buf) * a.n_masks + m) * P.keys_cap + c] = k;
    };

    const int S = a.n_stages;
    int64_t n_in = P.n0;
    const int swz = lane & 15;
    for (int i = 0; i < S; ++i) {
        if (!a.refresh[i]) {  // not due: the cached list stands (decode.cpp:241-249)
            n_in = a.count[i][m];
            continue;
        }
        const int lc = a.chunk_size[i], keep = a.keep[i], K = keep / lc;
        const int64_t cc = (n_in + lc - 1) / lc;
        int32_t* seli = sel + P.sel_off[i];
        int64_t n_out;
        int n_sel;
        if (n_in <= keep || cc <= K) {  // identity (pruning.cpp:159-168)
            for (int j = t; j < cc; j += kLT) seli[j] = j;
            n_out = n_in;
            n_sel = static_cast<int>(cc);
            __syncthreads();
        } else {
            if (i == 1) trace(22, 0);
            if (i == 0) {
                // stage 0's scores (decode.cu descent kernels, L2-resident): every CTA reads all
                // of them and forms the keys itself (max over heads) — no key exchange and no
                // group barrier for this selection
                for (int64_t c0 = 0; c0 < cc; c0 += 2 * kLT) {
                    float v[2][8];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int64_t c = c0 + u * kLT + t;
#pragma unroll
                        for (int h = 0; h < 8; ++h)  // every plane's load in flight before the first use
                            v[u][h] = (c < cc && h < P.planes0)
                                          ? __ldcg(P.scores0 + (static_cast<int64_t>(m) * P.planes0 + h) * P.max_chunks0 + c)
                                          : -INFINITY;
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int64_t c = c0 + u * kLT + t;
                        float best = -INFINITY;
#pragma unroll
                        for (int h = 0; h < 8; ++h) best = (best < v[u][h]) ? v[u][h] : best;  // std::max in head order (pruning.cpp:182)
                        if (c < cc) keys[c] = order_key(best);
                    }
                }
                __syncthreads();
            } else if (lc <= 8 && 32 % lc == 0) {
                // short chunks: a warp item = 32 / lc whole chunks, lane = row; one gather for
                // all heads, each head's Alg. 3 descent replayed on the row scores with shuffles
                const int cpw = 32 / lc;
                const int64_t n_items = (cc + cpw - 1) / cpw;
                const int64_t ipc = (n_items + CS - 1) / CS;
                const int64_t i0 = static_cast<int64_t>(rank) * ipc, i1 = min64(n_items, i0 + ipc);
                const int per_warp = static_cast<int>((max64(0, i1 - i0) + kLW - 1) / kLW);
                int iters = 0;
                while ((1 << iters) < lc) ++iters;
                const int cl = lane / lc, r = lane - cl * lc, c0l = cl * lc;
                unsigned char* wstage = stage + static_cast<size_t>(w) * kSlot;
                const unsigned char* myrow = wstage + lane * kRow;
                for (int k = 0; k < per_warp; ++k) {
                    const int64_t item = i0 + w + static_cast<int64_t>(k) * kLW;
                    const int64_t j = item * cpw + cl;
                    const bool live = item < i1 && j < cc;
                    const int len = live ? static_cast<int>(min64(lc, n_in - j * lc)) : 0;
                    const int64_t tk = r < len ? resolve(i - 1, j * lc + r) : -1;
                    __syncwarp();
                    stage_rows<bf16_t>(a.kv, kvh, tk, wstage, lane);
                    float acc[HP];
#pragma unroll
                    for (int h = 0; h < HP; ++h) acc[h] = 0.f;
                    if (use_fma) {
#pragma unroll 2
                        for (int c = 0; c < 16; ++c) {
                            const uint4 wv = *reinterpret_cast<const uint4*>(myrow + ((c ^ swz) << 4));
#pragma unroll
                            for (int h = 0; h < HP; ++h) {
                                const uint4 q = reinterpret_cast<const uint4*>(qb + h * (kD / 2))[c];
                                acc[h] = fma_bf16(q.x, wv.x, acc[h], false);
                                acc[h] = fma_bf16(q.x, wv.x, acc[h], true);
                                acc[h] = fma_bf16(q.y, wv.y, acc[h], false);
                                acc[h] = fma_bf16(q.y, wv.y, acc[h], true);
                                acc[h] = fma_bf16(q.z, wv.z, acc[h], false);
                                acc[h] = fma_bf16(q.z, wv.z, acc[h], true);
                                acc[h] = fma_bf16(q.w, wv.w, acc[h], false);
                                acc[h] = fma_bf16(q.w, wv.w, acc[h], true);
                            }
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < HP; ++h) acc[h] = dot_row<bf16_t>(myrow, swz, qs + h * kD);
                    }
                    float best = -INFINITY;
#pragma unroll
                    for (int h = 0; h < HP; ++h) {
                        const float sc = r < len ? acc[h] : -INFINITY;
                        int first = 1, last = len;
                        float s1 = __shfl_sync(0xffffffffu, sc, c0l);
                        for (int it = 0; it < iters; ++it) {
                            const int mid = (first + last + 1) >> 1;
                            const bool go = first < last;
                            const float s2 = __shfl_sync(0xffffffffu, sc, c0l + (go ? mid - 1 : 0));
                            if (go) {
                                if (s2 > s1) { first = mid; s1 = s2; } else { last = mid - 1; }
                            }
                        }
                        best = (best < s1) ? s1 : best;  // max over heads in head order
                    }
                    if (live && r == 0) put_key(j, order_key(best));
                }
            } else {
                // descents: a warp item = (32-chunk group, head), lane = chunk (Alg. 3, one
                // dependent row gather per comparison). (The two-comparison lookahead rounds of
                // decode_stage_look_kernel were measured slower here: 22.5 vs 17 us for stage 2
                // at 1M — 3x the rows per round on 8 warps per SM.)
                const int64_t n_groups = (cc + 31) / 32;
                const int64_t gpc = (n_groups + CS - 1) / CS;
                const int64_t g0 = static_cast<int64_t>(rank) * gpc;
                const int my_groups = static_cast<int>(max64(0, min64(n_groups, g0 + gpc) - g0));
                const int n_items = my_groups * HP;
                const int per_warp = (n_items + kLW - 1) / kLW;
                unsigned char* wstage = stage + static_cast<size_t>(w) * kSlot;
                const unsigned char* myrow = wstage + lane * kRow;
                for (int k = 0; k < per_warp; ++k) {
                    const int item_raw = w + k * kLW;
                    const bool item_ok = item_raw < n_items;
                    const int item = item_ok ? item_raw : n_items - 1;
                    const int gl = item / HP, hh = item - gl * HP;
                    const int64_t j = (g0 + gl) * 32 + lane;
                    const bool active = item_ok && j < cc;
                    const int64_t base = j * lc;
                    const int len = active ? static_cast<int>(min64(lc, n_in - base)) : 0;
                    int64_t t_first = 0;
                    bool contiguous = true;
                    if (active) {
                        t_first = resolve(i - 1, base);
                        if (len > 1) contiguous = resolve(i - 1, base + len - 1) - t_first == len - 1;
                    }
                    auto token = [&](int x) -> int64_t { return contiguous ? t_first + x : resolve(i - 1, base + x); };
                    const float* qrow = qs + hh * kD;
                    const uint32_t* qbrow = qb + hh * (kD / 2);
                    auto score = [&]() -> float {
                        return use_fma ? dot_row_bf16x(myrow, swz, qbrow) : dot_row<bf16_t>(myrow, swz, qrow);
                    };
                    int first = 1, last = len, it = 0, iters = 0;
                    while ((1 << iters) < len) ++iters;
                    float s1 = 0.f;
                    __syncwarp();
                    stage_rows<bf16_t>(a.kv, kvh, active ? token(0) : -1, wstage, lane);
                    if (active) s1 = score();
                    for (;;) {
                        const bool go = active && it < iters && first < last;
                        if (!__any_sync(0xffffffffu, go)) break;
                        const int mid = (first + last + 1) >> 1;
                        __syncwarp();
                        stage_rows<bf16_t>(a.kv, kvh, go ? token(mid - 1) : -1, wstage, lane);
                        if (go) {
                            const float m2 = score();
                            if (m2 > s1) { first = mid; s1 = m2; } else { last = mid - 1; }
                            ++it;
                        }
                    }
                    if (active) red[hh * P.red_cap + gl * 32 + lane] = s1;
                }
                __syncthreads();
                for (int c = t; c < my_groups * 32; c += kLT) {
                    const int64_t gc = g0 * 32 + c;
                    if (gc < cc) {
                        float best = -INFINITY;
#pragma unroll
                        for (int h = 0; h < HP; ++h) {
                            const float sv = red[h * P.red_cap + c];
                            best = (best < sv) ? sv : best;
                        }
                        put_key(gc, order_key(best));
                    }
                }
            }
            if (i != 0) {
                if (i == 1) trace(22, 1);
                group_barrier(gbar, static_cast<int>(++n_bar * CS));  // every CTA's keys are in L2
                if (i == 1) trace(22, 2);
                const uint32_t* gk = P.gkeys + (static_cast<size_t>(buf) * a.n_masks + m) * P.keys_cap;
                for (int64_t j0 = 0; j0 < cc; j0 += 8 * kLT) {  // 8 independent loads in flight per thread
                    uint32_t v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t j = j0 + u * kLT + t;
                        v[u] = j < cc ? __ldcg(gk + j) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t j = j0 + u * kLT + t;
                        if (j < cc) keys[j] = v[u];
                    }
                }
                __syncthreads();
            }
            if (i == 1) trace(22, 3);
            cta_topk_smem(keys, static_cast<int>(cc), K, seli, tsh);
            if (i == 1) trace(22, 4);
            n_out = static_cast<int64_t>(K - 1) * lc + min64(lc, n_in - static_cast<int64_t>(seli[K - 1]) * lc);
            n_sel = K;
            if (i != 0) buf ^= 1;  // a fast CTA's next keys never land in a buffer a slow CTA still copies
        }
        if (rank == 0) {  // the stage's kept chunk ids and output length (the caches' source)
            for (int j = t; j < n_sel; j += kLT) a.sel[i][static_cast<int64_t>(m) * a.sel_stride[i] + j] = seli[j];
            if (t == 0) a.count[i][m] = static_cast<int32_t>(n_out);
        }
        n_in = n_out;
        trace(20, 2 + i);
    }

    // ---- block-sparse attention over sinks ∪ last list ∪ stream (selected_indices +
    // attention_row, sparse_attention.cpp:15-60,95-112), the selected positions split
    // over the group's CTAs
    const int64_t mc = n_in;
    const int64_t nsel = sink_end + mc + (pos + 1 - stream_begin);
    const int64_t per = (nsel + CS - 1) / CS;
    const int64_t p0 = min64(nsel, static_cast<int64_t>(rank) * per), p1 = min64(nsel, p0 + per);
    const float scale = 1.0f / sqrtf(static_cast<float>(kD));
    unsigned char* Ks = stage;
    unsigned char* Vs = stage + kTile * kRow;
    if (t < HP) { sh_m[t] = -INFINITY; sh_l[t] = 0.f; }
    // Tensor-core tiles (mma.sync m16n8k16, bf16 in, fp32 accumulate): rows = the group's
    // heads (HP <= 8 of 16), q and p split into bf16 hi + lo parts so the products carry
    // ~16 mantissa bits (fp32-grade vs the 1e-3 tolerance; K and V are bf16 exactly).
    const int g = lane >> 2, tq = lane & 3;
    // P.V split: warp -> 16 output dims (two n-tiles) x one half of the tile's keys
    const int pv_n0 = (w & 7) * 16, pv_half = w >> 3;
    float oacc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};  // rows g (< HP): dims pv_n0 + {0, 8} + 2tq + {0,1}
    const int last = S - 1;
    trace(21, 0);
    for (int64_t pt = p0; pt < p1; pt += kTile) {
        const int nk = static_cast<int>(min64(kTile, p1 - pt));
        const int nk16 = (nk + 15) & ~15;
        for (int j = t; j < nk; j += kLT) {
            const int64_t p = pt + j;
            int64_t tk;
            if (p < sink_end) tk = p;
            else if (p < sink_end + mc) tk = resolve(last, p - sink_end);
            else tk = stream_begin + (p - sink_end - mc);
            kptr[j] = kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kvh, tk, 2);  // resolved once per key
            vptr[j] = kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kvh, tk, 2);
        }
        __syncthreads();
        if (pt == p0) trace(21, 1);
        // K and V rows, 16-byte chunk c of row j at slot c ^ (j & 15) (conflict-free fragment
        // loads and ldmatrix); padded rows of V are zeroed (p = 0 must not meet a NaN)
        for (int x = t; x < nk16 * 16; x += kLT) {
            const int j = x >> 4, c = x & 15;
            const int so = j * kRow + ((c ^ (j & 15)) << 4);
            if (j < nk) {
                cp_async16(Ks + so, kptr[j] + (c << 4));
                cp_async16(Vs + so, vptr[j] + (c << 4));
            } else {
                *reinterpret_cast<uint4*>(Vs + so) = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        if (pt == p0) trace(21, 2);
        // S = q K^T: warp w takes key tiles of 8 (n = key), 8 k-steps, hi and lo q
        for (int kt = w; kt < nk16 / 8; kt += kLW) {
            float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;  // hi parts of q
            float e0 = 0.f, e1 = 0.f, e2 = 0.f, e3 = 0.f;  // lo parts: an independent MMA chain
            const int j = kt * 8 + g;  // this thread's key for the B fragment
            const unsigned char* kr = Ks + j * kRow;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint32_t ah0 = qfr[((ks * 2 + 0) * 2) * 32 + lane], al0 = qfr[((ks * 2 + 0) * 2 + 1) * 32 + lane];
                const uint32_t ah1 = qfr[((ks * 2 + 1) * 2) * 32 + lane], al1 = qfr[((ks * 2 + 1) * 2 + 1) * 32 + lane];
                const int d0 = ks * 16 + 2 * tq, d1 = d0 + 8;
                const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + (((d0 >> 3) ^ (j & 15)) << 4) + (d0 & 7) * 2);
                const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + (((d1 >> 3) ^ (j & 15)) << 4) + (d1 & 7) * 2);
                mma_bf16_16816(c0, c1, c2, c3, ah0, ah1, b0, b1);
                mma_bf16_16816(e0, e1, e2, e3, al0, al1, b0, b1);
            }
            c0 += e0;
            c1 += e1;
            if (g < HP) {
                const int jj = kt * 8 + 2 * tq;
                pw[g * kPw + jj] = jj < nk ? c0 * scale : -INFINITY;
                pw[g * kPw + jj + 1] = jj + 1 < nk ? c1 * scale : -INFINITY;
            }
        }
        __syncthreads();
        if (pt == p0) trace(21, 3);
        // online softmax per head: warp h reduces head h's tile
        if (w < HP) {
            float mt = -INFINITY;
            for (int j = lane; j < nk; j += 32) mt = fmaxf(mt, pw[w * kPw + j]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
            const float m_old = sh_m[w];
            const float m_new = fmaxf(m_old, mt);
            float ls = 0.f;
            for (int j = lane; j < nk16; j += 32) {
                const float p = j < nk ? expf(pw[w * kPw + j] - m_new) : 0.f;
                pw[w * kPw + j] = p;
                ls += p;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
            if (lane == 0) {
                const float al = m_old == -INFINITY ? 0.f : expf(m_old - m_new);
                sh_alpha[w] = al;
                sh_m[w] = m_new;
                sh_l[w] = sh_l[w] * al + ls;
            }
        }
        __syncthreads();
        if (pt == p0) trace(21, 4);
        // O += P V: A = P (rows = heads, k = keys, hi + lo), B = V via ldmatrix.trans
        {
            const float al = g < HP ? sh_alpha[g] : 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) { oacc[nt][0] *= al; oacc[nt][1] *= al; }
            const int nsteps = nk16 / 16;
            const int s_begin = pv_half * ((nsteps + 1) / 2), s_end = min(nsteps, s_begin + (nsteps + 1) / 2);
            for (int st = s_begin; st < s_end; ++st) {
                const int k0 = st * 16;
                uint32_t ah[2], alo[2];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int kk = k0 + half * 8 + 2 * tq;
                    const float p0_ = g < HP ? pw[g * kPw + kk] : 0.f, p1_ = g < HP ? pw[g * kPw + kk + 1] : 0.f;
                    const uint32_t h2 = pack_bf16(p0_, p1_);
                    ah[half] = h2;
                    alo[half] = pack_bf16(p0_ - bf16_lo(h2), p1_ - bf16_hi(h2));
                }
                // ldmatrix.x4.trans: matrices (keys k0..+7 | k0+8..+15) x (dims n0 | n0+8)
                const int r = lane & 15, nsl = lane >> 4;
                const int jrow = k0 + r, cch = (pv_n0 >> 3) + nsl;
                uint32_t b[4];
                ldmatrix_x4_trans(b, Vs + jrow * kRow + ((cch ^ (jrow & 15)) << 4));
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    float d0 = oacc[nt][0], d1 = oacc[nt][1], d2 = 0.f, d3 = 0.f;
                    mma_bf16_16816(d0, d1, d2, d3, ah[0], ah[1], b[2 * nt], b[2 * nt + 1]);
                    mma_bf16_16816(d0, d1, d2, d3, alo[0], alo[1], b[2 * nt], b[2 * nt + 1]);
                    oacc[nt][0] = d0;
                    oacc[nt][1] = d1;
                }
            }
        }
        __syncthreads();  // the next tile's gathers overwrite K/V/P
        if (pt == p0) trace(21, 5);
    }
    trace(20, 5);
    // partial (o, m, l) per head; the two key halves are summed first
    float* pt2 = reinterpret_cast<float*>(stage);  // [2][HP][kD] scratch (tiles are done)
    if (g < HP) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int e = pv_n0 + nt * 8 + 2 * tq;
            pt2[(pv_half * HP + g) * kD + e] = oacc[nt][0];
            pt2[(pv_half * HP + g) * kD + e + 1] = oacc[nt][1];
        }
    }
    __syncthreads();
    for (int x = t; x < HP * kD; x += kLT) {
        const int h = x / kD, e = x - h * kD;
        part[h * kPart + e] = pt2[h * kD + e] + pt2[(HP + h) * kD + e];
    }
    if (t < HP) { part[t * kPart + kD] = sh_m[t]; part[t * kPart + kD + 1] = sh_l[t]; }
    __syncthreads();
    float* gp = P.gpart + static_cast<size_t>(m) * CS * HP * kPart;
    for (int x = t; x < HP * kPart; x += kLT) gp[static_cast<size_t>(rank) * HP * kPart + x] = part[x];
    float* allp = reinterpret_cast<float*>(stage);  // staged partials
    if (static_cast<int>(CS) * HP * kPart * 4 <= kStageBytes) {
        // the last CTA to finish (acq_rel ticket) merges every head: no CTA waits
        __syncthreads();
        if (t == 0) {
            int prev;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(gbar + 2) : "memory");
            sh_last = prev == static_cast<int>(CS) - 1;
            if (sh_last) {  // every CTA is past every barrier: reset for the next launch
                gbar[0] = 0;
                gbar[2] = 0;
            }
        }
        __syncthreads();
        pdl_trigger();  // every CTA of the grid is past its last barrier
        if (!sh_last) return;
        {
            const int n = static_cast<int>(CS) * HP * kPart;
            for (int x0 = 0; x0 < n; x0 += 8 * kLT) {  // 8 independent L2 loads in flight per thread
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int x = x0 + u * kLT + t;
                    v[u] = x < n ? __ldcg(gp + x) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int x = x0 + u * kLT + t;
                    if (x < n) allp[x] = v[u];
                }
            }
        }
        __syncthreads();
        for (int x = t; x < HP * kD; x += kLT) {
            const int h = x / kD, e = x - h * kD;
            float M = -INFINITY;
            for (unsigned c = 0; c < CS; ++c) M = fmaxf(M, allp[(c * HP + h) * kPart + kD]);
            float Lsum = 0.f, O = 0.f;
            for (unsigned c = 0; c < CS; ++c) {
                const float* pc = allp + (c * HP + h) * kPart;
                if (pc[kD] == -INFINITY) continue;
                const float wgt = expf(pc[kD] - M);
                Lsum += wgt * pc[kD + 1];
                O += wgt * pc[e];
            }
            a.out[static_cast<int64_t>(m * HP + h) * kD + e] = O / Lsum;
        }
    } else {
        // many CTAs per group: a barrier, then CTA r merges heads r, r + CS, ... with every
        // CTA's partials of those heads staged ([local head][CS][kPart])
        group_barrier(gbar, static_cast<int>(++n_bar * CS));
        pdl_trigger();
        for (int h = rank, hl = 0; h < HP; h += CS, ++hl)
            for (int x = t; x < static_cast<int>(CS) * kPart; x += kLT) {
                const int c = x / kPart, o = x - c * kPart;
                allp[(hl * CS + c) * kPart + o] = __ldcg(gp + (static_cast<size_t>(c) * HP + h) * kPart + o);
            }
        __syncthreads();
        for (int h = rank, hl = 0; h < HP; h += CS, ++hl) {
            if (t < kD) {
                float M = -INFINITY;
                for (unsigned c = 0; c < CS; ++c) M = fmaxf(M, allp[(hl * CS + c) * kPart + kD]);
                float Lsum = 0.f, O = 0.f;
                for (unsigned c = 0; c < CS; ++c) {
                    const float* pc = allp + (hl * CS + c) * kPart;
                    if (pc[kD] == -INFINITY) continue;
                    const float wgt = expf(pc[kD] - M);
                    Lsum += wgt * pc[kD + 1];
                    O += wgt * pc[t];
                }
                a.out[static_cast<int64_t>(m * HP + h) * kD + t] = O / Lsum;
            }
        }
        __syncthreads();
        if (t == 0) {  // exit ticket: the last CTA out resets the counters for the next launch
            int prev;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(gbar + 3) : "memory");
            if (prev == static_cast<int>(CS) - 1) {
                gbar[0] = 0;
                gbar[3] = 0;
            }
        }
    }
    trace(20, 6);
}

template <int HP>
cudaError_t launch_layer(const LayerParams& p, int ctas, size_t smem, cudaStream_t s) {
    auto kern = decode_layer_kernel<HP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas, p.a.n_masks);
    cfg.blockDim = dim3(kLT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t dispatch(int hp, const LayerParams& p, int ctas, size_t smem, cudaStream_t s) {
    switch (hp) {
        case 1: return launch_layer<1>(p, ctas, smem, s);
        case 2: return launch_layer<2>(p, ctas, smem, s);
        case 4: return launch_layer<4>(p, ctas, smem, s);
        default: return launch_layer<8>(p, ctas, smem, s);
    }
}

size_t ws_stage_bytes(int32_t n_masks, int32_t max_chunks0) { return align_up(hp_decode_stage_workspace_bytes(n_masks, max_chunks0), 256); }
size_t ws_keys_bytes(int32_t n_masks) { return align_up(static_cast<size_t>(2) * n_masks * kKeysMax * 4, 256); }
size_t ws_part_bytes(int32_t n_masks) { return align_up(static_cast<size_t>(n_masks) * kMaxGroupCtas * 8 * kPart * 4, 256); }

// host validation shared by _supported and the launch; returns HP_OK or sets the error
int check_args(const hp_decode_layer_args& a) {
    if (a.n_stages < 1 || a.n_stages > kMaxS) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: 1..4 stages");
    for (int i = 0; i < a.n_stages; ++i) {
        if (a.chunk_size[i] <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: b_q and l_c must be >= 1");
        if (a.keep[i] <= 0 || a.keep[i] % a.chunk_size[i]) return hph::set_error(HP_INVALID_ARGUMENT, "StageConfig: k must be a positive multiple of l_c");
        if (a.sel_stride[i] < a.keep[i] / a.chunk_size[i]) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: sel_stride < k/l_c");
        if (!a.sel[i] || !a.count[i]) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: null sel/count");
        if (i > 0 && a.keep[i] > a.keep[i - 1]) return hph::set_error(HP_INVALID_ARGUMENT, "PruningPlan: k must be non-increasing across stages");
    }
    const int hp = a.heads_per_mask;
    if (a.kv.d != kD || a.kv.dtype != HP_BF16) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: bf16 K/V with head_dim 128 only");
    if (!(hp == 1 || hp == 2 || hp == 4 || hp == 8) || a.n_masks <= 0 || a.n_q_heads != a.n_masks * hp || a.kv.n_kv <= 0 ||
        a.n_q_heads % a.kv.n_kv || (a.n_q_heads / a.kv.n_kv) % hp)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: bad head geometry");
    if (!a.q || !a.out || !a.kv.k_pool || !a.kv.v_pool) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: null pointer");
    return HP_OK;
}

}  // namespace

// stage-0 scores (hp_decode_stage's workspace), then the exchanged keys, the attention
// partials and per-group barrier counters (which must start at zero: the workspace must
// be zeroed once before first use; every launch leaves them consistent for the next)
extern "C" size_t hp_decode_layer_workspace_bytes(int32_t n_masks, int32_t max_chunks0) {
    return ws_stage_bytes(n_masks, max_chunks0) + ws_keys_bytes(n_masks) + ws_part_bytes(n_masks) +
           align_up(static_cast<size_t>(n_masks) * kBarInts * 4, 256);
}

extern "C" int hp_decode_layer_supported(const hp_decode_layer_args* ap) {
    if (!ap) return 0;
    return check_args(*ap) == HP_OK ? 1 : 0;
}

#if defined(HP_TRACE) || defined(HP_DEV)  // developer hooks: dev builds only (include/hipprune_b200_dev.h)
// per-CTA phase stamps of the layer kernel (trace ids 20-22) into buf
extern "C" int hp_layer_trace_enable(unsigned long long* buf, int kernel_id) {
    if (int rc = hph::check_cuda(cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(buf)), "hp_layer_trace_enable")) return rc;
    return hph::check_cuda(cudaMemcpyToSymbol(g_trace_kernel, &kernel_id, sizeof(int)), "hp_layer_trace_enable");
}
#endif

extern "C" int hp_decode_layer(const hp_decode_layer_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: null args");
    const hp_decode_layer_args& a = *ap;
    if (int rc = check_args(a)) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t pos = a.query_position;
    const int64_t t = pos + 1;
    const int64_t upper = t > a.stream_tokens ? t - a.stream_tokens : 0;
    const int64_t n0 = std::max<int64_t>(0, upper - a.sink_tokens);
    const int lc0 = a.chunk_size[0];
    const int32_t mc0 = static_cast<int32_t>(std::max<int64_t>(1, (n0 + lc0 - 1) / lc0));
    if (mc0 > kKeysMax) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: %d stage-0 chunks exceed %d", mc0, kKeysMax);
    const size_t need = hp_decode_layer_workspace_bytes(a.n_masks, mc0);
    if (!a.workspace || a.workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: workspace too small");
    if (a.n_masks > 4096) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: at most 4096 masks");
    LayerParams p{};
    p.a = a;
    p.n0 = n0;
    p.max_chunks0 = mc0;
    p.planes0 = 1;
    p.scores0 = reinterpret_cast<const float*>(static_cast<const char*>(a.workspace) + align_up(static_cast<size_t>(a.n_masks) * 4, 256));
    const bool sel0 = a.refresh[0] && !(n0 <= a.keep[0] || mc0 <= a.keep[0] / lc0);
    if (sel0) {
        // stage 0's descent on its own kernel (decode.cu): scores only, selected in the layer kernel
        hp_decode_stage_args sa{};
        sa.chunk_size = lc0;
        sa.keep = a.keep[0];
        sa.n_masks = a.n_masks;
        sa.heads_per_mask = a.heads_per_mask;
        sa.n_q_heads = a.n_q_heads;
        sa.stream_tokens = a.stream_tokens;
        sa.q = a.q;
        sa.query_position = pos;
        sa.in.depth = 0;
        sa.in.range_start = a.sink_tokens;
        sa.in_count = nullptr;
        sa.in_count_const = n0;
        sa.max_chunks = mc0;
        sa.sel_stride = a.sel_stride[0];
        sa.sel_out = nullptr;
        sa.out_count = a.count[0];
        sa.workspace = a.workspace;
        sa.workspace_bytes = a.workspace_bytes;
        sa.keys = a.kv;
        sa.keys_exact = a.keys_exact;
        int32_t variant = 0;
        hp_decode_stage_variant(&sa, &variant);
        p.planes0 = variant == HP_STAGE_WIDE ? a.heads_per_mask : 1;
        if (int rc = hp_decode_stage(&sa, stream)) return rc;
    }
    // one co-resident CTA per SM, n_SM / n_masks CTAs per KV group
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int ctas = std::max(1, std::min(kMaxGroupCtas, n_sm / std::max(1, a.n_masks)));
    // per-stage input bounds -> shared-memory sizing
    int64_t bound = n0;
    int keys_cap = 1, red_cap = 32, sel_total = 0;
    for (int i = 0; i < a.n_stages; ++i) {
        if (i > 0) bound = a.refresh[i - 1] ? std::min<int64_t>(bound, a.keep[i - 1]) : a.keep[i - 1];
        const int lc = a.chunk_size[i];
        const int64_t cc = (bound + lc - 1) / lc;
        p.sel_off[i] = sel_total;
        sel_total += std::max(1, a.keep[i] / lc);
        if (a.refresh[i]) {
            keys_cap = static_cast<int>(std::max<int64_t>(keys_cap, cc));
            const int64_t gpc = ((cc + 31) / 32 + ctas - 1) / ctas;
            red_cap = static_cast<int>(std::max<int64_t>(red_cap, gpc * 32));
        }
    }
    if (keys_cap > kKeysMax) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: %d chunks per stage exceed %d", keys_cap, kKeysMax);
    p.keys_cap = (keys_cap + 3) & ~3;
    p.red_cap = red_cap;
    p.sel_total = sel_total;
    char* ws = static_cast<char*>(a.workspace);
    size_t off = ws_stage_bytes(a.n_masks, mc0);
    p.gkeys = reinterpret_cast<uint32_t*>(ws + off);
    off += ws_keys_bytes(a.n_masks);
    p.gpart = reinterpret_cast<float*>(ws + off);
    off += ws_part_bytes(a.n_masks);
    p.gbar = reinterpret_cast<int*>(ws + off);
    const LayerSmem L(sel_total, a.heads_per_mask, red_cap);
    if (L.bytes + 8 * 1024 > 227 * 1024) return hph::set_error(HP_INVALID_ARGUMENT, "hp_decode_layer: stage lists too long for shared memory");
    const cudaError_t e = dispatch(a.heads_per_mask, p, ctas, L.bytes, s);
    if (e != cudaSuccess) return hph::check_cuda(e, "decode_layer_kernel");
    return hph::check_cuda(cudaGetLastError(), "decode_layer_kernel");
}

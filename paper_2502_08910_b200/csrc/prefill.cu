// Prefill block-sparse attention on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Replaces block_sparse_attention (reference proj/src/sparse_attention.cpp:114-145):
// every query row r attends to its selected set — sinks [0, min(n_sink, pos+1)), the
// mask of its query block inside [sink_end, stream_begin), and the stream window
// [stream_begin, pos] — with scale 1/sqrt(d) and a softmax over that set.
//
// A CTA owns one query block (b_q rows) for the 128 / b_q q-heads of one KV group that
// fill a 128-row MMA tile, so every key tile is shared by those heads (GQA). The
// block's union key list (sinks ∪ mask ∪ the block's stream span, each token once,
// flagged with mask membership) is built in shared memory; per row, key u counts iff
//   u <= pos  &&  (u < n_sink  ||  u in mask  ||  u >= stream_begin(pos))
// which is exactly selected_indices (sparse_attention.cpp:95-112) for that row.
// Per 128-key tile:
//   1. gather the K and V rows (16-byte cp.async through the page table) into the
//      canonical no-swizzle UMMA layouts (K K-major, V MN-major), bf16;
//   2. one thread issues S = Q K^T as 8 x tcgen05.mma (M=128, N=128, K=16) into TMEM;
//   3. four threads own a row (32 columns each): tcgen05.ld of their S columns, causal/selection mask,
//      online-softmax update, P (bf16) to shared memory, O rescaled in TMEM
//      (tcgen05.ld / tcgen05.st);
//   4. O += P V as 8 x tcgen05.mma into the TMEM accumulator.
// MMA completion is tracked with tcgen05.commit -> mbarrier. The tile contraction is
// bf16 x bf16 -> fp32 (Q and P rounded to bf16): the stated bf16 tolerance applies.
#include <cstdint>

#include "common.cuh"
#include "umma.cuh"

using namespace hpk;
using namespace hpk::um;

namespace {

constexpr int kTM = 128;       // query rows per MMA tile (TMEM lanes)
constexpr int kTN = 128;       // keys per tile
constexpr int kHD = 128;       // head dim
constexpr int kThreads = 512;  // four threads per query row (32 score / output columns each)
constexpr int kQ = kThreads / kTM;  // threads per row
constexpr int kCols = kTN / kQ;     // score (and output) columns per thread
constexpr uint32_t kTmemCols = 256;  // S [0,128) + O [128,256)

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// dev builds: progress codes written by thread 0 to a (mapped host) word, to locate a
// stall; compiled out of the product kernel
#if defined(HP_TRACE) || defined(HP_DEV)
__device__ volatile int* g_pf_progress = nullptr;
__device__ __forceinline__ void progress(int code) {
    if (threadIdx.x == 0 && g_pf_progress) {
        *g_pf_progress = code;
        __threadfence_system();
    }
}
#else
__device__ __forceinline__ void progress(int) {}
#endif

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct PrefillSmem {
    static constexpr uint32_t tile_bytes = kTN * kHD * 2;  // 32 KB
    static constexpr uint32_t q_off = 0;
    static constexpr uint32_t k_off = q_off + kTM * kHD * 2;  // K[2] (double buffered)
    static constexpr uint32_t v_off = k_off + 2 * tile_bytes;  // V[2]
    static constexpr uint32_t p_off = v_off + 2 * tile_bytes;
    static constexpr uint32_t u_off = p_off + kTM * kTN * 2;   // union list (int32, bit 31 = in mask)
};

__global__ void __launch_bounds__(kThreads, 1) bsa_prefill_tc_kernel(const hp_bsa_prefill_args a, int max_union) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar_s, bar_o;
    __shared__ uint32_t tmem_base_sh;
    __shared__ int sh_counts[4];
    static_assert(kCols == 32 && kTN == kHD, "a thread's S and O columns are one 32-column TMEM load each");
    using S = PrefillSmem;
    const int t = threadIdx.x, lane = t & 31, w = warp_id();
    const int bs = a.block_size;
    const int hpt = kTM / bs;  // heads per tile
    const int b = blockIdx.x, m = blockIdx.y, hp = blockIdx.z;
    const int hpm = a.heads_per_mask;
    const int kvh = (m * hpm) / (a.n_q_heads / a.kv.n_kv);
    const int row0 = b * bs;
    const int rows_here = min(bs, a.n_rows - row0);
    const int64_t pos_first = a.query_offset + row0;
    const int64_t pos_last = pos_first + rows_here - 1;
    const int64_t sink = a.sink_tokens;
    auto stream_begin = [&](int64_t pos) {
        const int64_t se = min64(sink, pos + 1);
        const int64_t sb = pos + 1 > a.stream_tokens ? pos + 1 - a.stream_tokens : 0;
        return max64(sb, se);
    };
    const int64_t sbf = stream_begin(pos_first);
    const int64_t s0 = min64(sink, pos_last + 1);  // sinks of the union
    const int32_t* mlist = a.mask_list + (static_cast<int64_t>(m) * a.n_mask_blocks + b) * a.mask_stride;
    const int mcount = a.mask_count[static_cast<int64_t>(m) * a.n_mask_blocks + b];

    progress(1);
    // ---- TMEM + barriers
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        mbar_init(&bar_s, 1);
        mbar_init(&bar_o, 1);
    }
    // ---- union key list: sinks, mask entries below sbf, then the stream span [max(sbf, s0), pos_last]
    int32_t* uni = reinterpret_cast<int32_t*>(smem + S::u_off);
    if (t == 0) {
        int lo = 0, hi = mcount;  // first mask entry >= sbf
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (mlist[mid] < sbf) lo = mid + 1; else hi = mid;
        }
        int msink = 0;  // mask entries < s0 are sinks already (middle lists start at n_sink)
        while (msink < lo && mlist[msink] < s0) ++msink;
        sh_counts[0] = msink;
        sh_counts[1] = lo;
        sh_counts[2] = static_cast<int>(max64(0, pos_last + 1 - max64(sbf, s0)));
    }
    progress(2);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    progress(3);
    const int msink = sh_counts[0], mmid = sh_counts[1], nstream = sh_counts[2];
    const int nmid = mmid - msink;
    const int64_t st0 = max64(sbf, s0);
    const int U = static_cast<int>(s0) + nmid + nstream;
    for (int i = t; i < U; i += kThreads) {
        int32_t v;
        if (i < s0) v = i;
        else if (i < s0 + nmid) v = mlist[msink + i - s0] | static_cast<int32_t>(0x80000000u);
        else v = static_cast<int32_t>(st0 + (i - s0 - nmid));
        uni[i] = v;
    }
    __syncthreads();
    // mask entries inside the stream span: flag them (a row whose own stream window starts
    // later still selects them through its mask)
    for (int i = mmid + t; i < mcount; i += kThreads) {
        const int64_t u = mlist[i];
        if (u >= st0 && u <= pos_last) uni[s0 + nmid + (u - st0)] |= static_cast<int32_t>(0x80000000u);
    }
    // ---- Q tile (bf16, K-major): tile row i = head (i / bs) of the pair, block row (i % bs)
    const int my_i = t & (kTM - 1), half = t >> 7;  // row, column quarter
    {
        const int i = my_i;
        const int hh = hp * hpt + i / bs, r = i % bs;
        const bool ok = r < rows_here;
        const float* qr = a.q + (static_cast<int64_t>(m * hpm + hh) * a.n_rows + row0 + r) * kHD;
        unsigned char* qs = smem + S::q_off;
        for (int c = half * (16 / kQ); c < (half + 1) * (16 / kQ); ++c) {
            uint4 pk = make_uint4(0, 0, 0, 0);
            if (ok) {
                const float4 x0 = reinterpret_cast<const float4*>(qr)[2 * c];
                const float4 x1 = reinterpret_cast<const float4*>(qr)[2 * c + 1];
                pk = make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
            }
            *reinterpret_cast<uint4*>(qs + kmajor_off(i, c * 8)) = pk;
        }
    }
    const int my_r = my_i % bs;
    const bool my_ok = my_r < rows_here;
    const int64_t my_pos = pos_first + (my_ok ? my_r : rows_here - 1);
    const int64_t my_sb = stream_begin(my_pos);
    // the block's first row is past every sink of the union (a block overlapping the sink
    // region, e.g. a prompt prefilled from position 0, keeps the causal test per entry)
    const bool all_see_low = pos_first + 1 >= s0;
    // softmax in base 2: scores scaled by log2(e)/sqrt(d), exponentials on MUFU.EX2
    const float scale = 1.4426950408889634f / sqrtf(static_cast<float>(kHD));
    float run_m = -INFINITY, run_l = 0.f;  // run_l: this thread's quarter of the row sum
    const uint32_t lane_base = static_cast<uint32_t>((w & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + half * kCols;        // this quarter's S columns
    const uint32_t tO = tmem + lane_base + 128 + half * kCols;  // this quarter's O columns
    const uint32_t idesc_qk = instr_desc(kTM, kTN, 0, 0);
    const uint32_t idesc_pv = instr_desc(kTM, kHD, 0, 1);
    const uint32_t sbase = smem_u32(smem);
    const int n_tiles = (U + kTN - 1) / kTN;
    __shared__ float sh_max[kQ][kTM];
    // resident KV with power-of-two pages: a row is pool + 256 B x (page*n_kv + kvh)*ps + off,
    // 32-bit index math (rows < 2^32) instead of the general page-table walk
    const uint32_t ps = static_cast<uint32_t>(a.kv.page_size);
    const bool fast_rows = a.kv.page_table == nullptr && a.kv.touched == nullptr && a.kv.row_bits == nullptr &&
                           (ps & (ps - 1)) == 0 &&
                           static_cast<uint64_t>(a.kv.num_pages) * a.kv.n_kv * ps < (1ull << 32);
    const uint32_t ps_shift = static_cast<uint32_t>(__ffs(static_cast<int>(ps)) - 1);
    const uint32_t nkv = static_cast<uint32_t>(a.kv.n_kv);
    // coalesced gather: 16 threads per 256 B row (one 16 B chunk each), 16 rows per pass
    auto gather = [&](int tile, int buf) {
        unsigned char* ks = smem + S::k_off + buf * S::tile_bytes;
        unsigned char* vs = smem + S::v_off + buf * S::tile_bytes;
        const int c = t & 15;
#pragma unroll 2
        for (int j0 = 0; j0 < kTN; j0 += kThreads / 16) {
            const int j = j0 + (t >> 4);
            const int ui = tile * kTN + j;
            if (ui < U) {
                const uint32_t tk = static_cast<uint32_t>(uni[ui]) & 0x7fffffffu;
                const char* kp;
                const char* vp;
                if (fast_rows) {
                    const uint32_t idx = (((tk >> ps_shift) * nkv + static_cast<uint32_t>(kvh)) << ps_shift) + (tk & (ps - 1));
                    kp = static_cast<const char*>(a.kv.k_pool) + static_cast<size_t>(idx) * (kHD * 2);
                    vp = static_cast<const char*>(a.kv.v_pool) + static_cast<size_t>(idx) * (kHD * 2);
                } else {
                    kp = kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kvh, tk, 2);
                    vp = kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kvh, tk, 2);
                }
                cp_async16(ks + kmajor_off(j, c * 8), kp + c * 16);
                cp_async16(vs + mnmajor_off(j, c * 8), vp + c * 16);
            } else {
                *reinterpret_cast<uint4*>(ks + kmajor_off(j, c * 8)) = make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(vs + mnmajor_off(j, c * 8)) = make_uint4(0, 0, 0, 0);
            }
        }
    };
    if (n_tiles > 0) gather(0, 0);
    for (int tile = 0; tile < n_tiles; ++tile) {
        const int buf = tile & 1;
        // 1. this tile's K/V have landed
        cp_async_wait_all();
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        progress(10 + tile * 10);
        // 2. S = Q K^T (queued behind the previous P.V on the tensor core)
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kHD / 16; ++k) {
                const uint64_t da = smem_desc(sbase + S::q_off + k * 256, 128, 2048);
                const uint64_t db = smem_desc(sbase + S::k_off + buf * S::tile_bytes + k * 256, 128, 2048);
                mma_bf16(tmem, da, db, idesc_qk, k > 0);
            }
            mma_commit(&bar_s);
        }
        // 3. the previous P.V is done: its P, V buffer and O are free -> prefetch the next tile
        if (tile > 0) {
            mbar_wait_bounded(&bar_o, (tile - 1) & 1);
            tc_fence_after();
        }
        if (tile + 1 < n_tiles) gather(tile + 1, buf ^ 1);
        progress(11 + tile * 10);
        mbar_wait_bounded(&bar_s, tile & 1);
        progress(12 + tile * 10);
        tc_fence_after();
        // 4. masked online softmax over this thread's 64 columns; row max shared by the two halves
        float sv[kCols];
        tmem_ld32(tS, sv);
        // selection test, branch-free (union entries past U read as 0x7fffffff = never
        // selected); four independent max chains
        float tm4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        const int ub = tile * kTN + half * kCols;
        const int32_t pos32 = my_ok ? static_cast<int32_t>(my_pos) : -1;
        const int32_t sb32 = static_cast<int32_t>(my_sb), sink32 = static_cast<int32_t>(min64(sink, 0x7fffffff));
        if (my_ok && all_see_low && ub + kCols <= s0 + nmid) {
            // sinks and mask entries (union index < s0 + nmid) precede every row of the
            // block (< stream_begin(first row), and the first row already sees every
            // sink): all selected, no per-entry test
#pragma unroll
            for (int jj = 0; jj < kCols; ++jj) tm4[jj & 3] = fmaxf(tm4[jj & 3], sv[jj]);
        } else {
#pragma unroll
        for (int j4 = 0; j4 < kCols; j4 += 4) {  // four union entries per 16-byte load
            const int4 e4 = *reinterpret_cast<const int4*>(uni + ub + j4);
            const int32_t ev[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int jj = j4 + q;
                const int32_t e = (ub + jj < U) ? ev[q] : 0x7fffffff;
                const int32_t u = e & 0x7fffffff;
                const bool ok = u <= pos32 && (u < sink32 || e < 0 || u >= sb32);
                sv[jj] = ok ? sv[jj] : -INFINITY;  // raw scores; the scale is folded into the exponent
                tm4[q] = fmaxf(tm4[q], sv[jj]);
            }
        }
        }
        const float tmax = fmaxf(fmaxf(tm4[0], tm4[1]), fmaxf(tm4[2], tm4[3])) * scale;
        sh_max[half][my_i] = tmax;
        __syncthreads();
        // lazy rescale (base 2): keep a stale running max unless the tile's max exceeds it
        // by more than 2^8 — P (bf16) and the fp32 sums stay in range, O and l share the
        // same reference, so the final O / l is unchanged; most tiles skip the TMEM rescale
        const float tile_m = fmaxf(fmaxf(sh_max[0][my_i], sh_max[1][my_i]), fmaxf(sh_max[2][my_i], sh_max[3][my_i]));
        const float new_m = (run_m != -INFINITY && tile_m <= run_m + 8.0f) ? run_m : fmaxf(run_m, tile_m);
        const float alpha = (run_m == -INFINITY) ? 0.f : ex2_approx(run_m - new_m);
        float ps4[4] = {0.f, 0.f, 0.f, 0.f};
        const float mref = new_m == -INFINITY ? 0.f : new_m;  // rows with nothing selected yet: all p = 0
        unsigned char* ps = smem + S::p_off;
#pragma unroll
        for (int c = 0; c < kCols / 8; ++c) {
            float p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float x = sv[c * 8 + u];
                p[u] = ex2_approx(fmaf(x, scale, -mref));  // masked: ex2(-inf) = 0
                ps4[u & 3] += p[u];
            }
            *reinterpret_cast<uint4*>(ps + kmajor_off(my_i, half * kCols + c * 8)) =
                make_uint4(pack_bf16(p[0], p[1]), pack_bf16(p[2], p[3]), pack_bf16(p[4], p[5]), pack_bf16(p[6], p[7]));
        }
        const float psum = (ps4[0] + ps4[1]) + (ps4[2] + ps4[3]);
        run_l = run_l * alpha + psum;
        run_m = new_m;
        // tcgen05.ld/st are .sync.aligned: the whole warp rescales if any row needs it
        if (tile > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
            float ov[32];
            tmem_ld32(tO, ov);
#pragma unroll
            for (int u = 0; u < 32; ++u) ov[u] *= alpha;
            tmem_st32(tO, ov);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        // 5. O += P V
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kTN / 16; ++k) {
                const uint64_t da = smem_desc(sbase + S::p_off + k * 256, 128, 2048);
                const uint64_t db = smem_desc(sbase + S::v_off + buf * S::tile_bytes + k * 4096, 2048, 128);
                mma_bf16(tmem + 128, da, db, idesc_pv, (tile > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&bar_o);
        }
        progress(13 + tile * 10);
    }
    // ---- epilogue: O / l for this thread's row and column half
    if (n_tiles > 0) {
        mbar_wait_bounded(&bar_o, (n_tiles - 1) & 1);
        tc_fence_after();
    }
    sh_max[half][my_i] = run_l;
    __syncthreads();
    const float row_l = (sh_max[0][my_i] + sh_max[1][my_i]) + (sh_max[2][my_i] + sh_max[3][my_i]);
    {
        const int hh = hp * hpt + my_i / bs;
        float* orow = a.out + (static_cast<int64_t>(m * hpm + hh) * a.n_rows + row0 + my_r) * kHD + half * kCols;
        float ov[32];
        if (n_tiles > 0) tmem_ld32(tO, ov);
        if (my_ok) {
            const float inv = row_l > 0.f ? 1.0f / row_l : NAN;
#pragma unroll
            for (int u = 0; u < 32; u += 4)
                *reinterpret_cast<float4*>(orow + u) = make_float4(ov[u] * inv, ov[u + 1] * inv, ov[u + 2] * inv, ov[u + 3] * inv);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace

#if defined(HP_TRACE) || defined(HP_DEV)  // developer hook: dev builds only (include/hipprune_b200_dev.h)
extern "C" int hp_debug_prefill_progress(int* mapped_word) {
    return hph::check_cuda(cudaMemcpyToSymbol(g_pf_progress, &mapped_word, sizeof(mapped_word)), "hp_debug_prefill_progress");
}
#endif

extern "C" size_t hp_bsa_prefill_smem_bytes(int32_t max_union) {
    // union list padded to whole 128-key tiles: the selection test reads it 16 bytes at a time
    return PrefillSmem::u_off + static_cast<size_t>((max_union + kTN - 1) / kTN * kTN) * 4;
}

extern "C" int hp_bsa_prefill(const hp_bsa_prefill_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa_prefill: null args");
    const hp_bsa_prefill_args& a = *ap;
    if (a.kv.d != kHD || a.kv.dtype != HP_BF16)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa_prefill: the tensor-core path needs bf16 K/V with head_dim 128");
    if (a.block_size <= 0 || kTM % a.block_size || a.heads_per_mask % (kTM / a.block_size) ||
        a.n_q_heads % a.heads_per_mask || a.n_q_heads % a.kv.n_kv || (a.n_q_heads / a.kv.n_kv) % a.heads_per_mask)
        return hph::set_error(HP_INVALID_ARGUMENT,
                              "hp_bsa_prefill: block_size must divide 128 and 128/block_size heads must share a kv head");
    if (!a.q || !a.out || !a.mask_list || !a.mask_count || !a.kv.k_pool || !a.kv.v_pool)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa_prefill: null pointer");
    const int n_blocks = (a.n_rows + a.block_size - 1) / a.block_size;
    if (a.n_mask_blocks < n_blocks) return hph::set_error(HP_INVALID_ARGUMENT, "block_sparse_attention: mask does not cover the queries");
    const int max_union = a.sink_tokens + a.max_mask + a.stream_tokens + a.block_size;
    const size_t smem = hp_bsa_prefill_smem_bytes(max_union);
    if (smem > 227 * 1024) return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa_prefill: selected set too large (%d keys)", max_union);
    cudaError_t e = cudaFuncSetAttribute(bsa_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return hph::check_cuda(e, "bsa_prefill_tc_kernel");
    const int n_masks = a.n_q_heads / a.heads_per_mask;
    dim3 grid(n_blocks, n_masks, a.heads_per_mask / (kTM / a.block_size));
    bsa_prefill_tc_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(a, max_union);
    return hph::check_cuda(cudaGetLastError(), "bsa_prefill_tc_kernel");
}

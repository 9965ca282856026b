/*
 * hipprune_b200 — C ABI of the B200-native InfiniteHiP attention hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types). All device pointers
 * are caller-owned; no entry point allocates on the hot path. Every call is
 * asynchronous on the given cudaStream_t (passed as void*) and re-entrant per
 * stream. Status codes map 1:1 onto the reference's exception types
 * (SURVEY.md §8(b)); hp_last_error() returns the thread's last message.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Layouts
 *   q        fp32 [n_q_heads][q_rows][d]          (decode: q_rows == 1)
 *   K/V pool [num_slots][n_kv][page_size][d]      of HP_F32 or HP_BF16
 *   page     covers page_size consecutive tokens of all kv heads of one layer
 *            (kv_store.cpp:50-56); page_table maps page -> slot, -1 = not
 *            resident (read from the host tier instead, a cache miss).
 *   lists    int32 token indices, [n_masks][n_blocks][stride] + int32 counts.
 *   GQA      q-head h reads kv-head h / (n_q_heads / n_kv); mask m pools the
 *            q-heads [m*hpm, (m+1)*hpm) (one reference call per KV group).
 */
#ifndef HIPPRUNE_B200_H
#define HIPPRUNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes == reference exception types */
enum hp_status {
    HP_OK = 0,
    HP_CONTRACT_VIOLATION = 1, /* hipprune::ContractViolation (errors.hpp:8-10)  */
    HP_INVALID_ARGUMENT = 2,   /* std::invalid_argument                         */
    HP_OUT_OF_RANGE = 3,       /* std::out_of_range                             */
    HP_LOGIC_ERROR = 4,        /* std::logic_error                              */
    HP_RUNTIME_ERROR = 5,      /* std::runtime_error / CUDA failure             */
    HP_PARTIAL_COMMIT = 6      /* hipprune::PartialCommitError (kv_store.hpp:41) */
};

enum hp_dtype { HP_F32 = 0, HP_BF16 = 1 };

/* RoPE policy ids (rope_policy.hpp:11) */
enum hp_rope_policy { HP_ROPE_CHUNK_INDEXED = 0, HP_ROPE_RELATIVE = 1, HP_ROPE_STREAMING = 2 };

const char* hp_last_error(void);
int hp_version(void);
/* 1 when a CUDA device is usable; product calls fail with HP_RUNTIME_ERROR otherwise. */
int hp_device_available(void);

/* Device-resident paged KV of one layer (replaces KeySource / KvView,
 * key_source.hpp:13-18, kv_store.cpp:160-200). */
typedef struct hp_kv_view {
    const void* k_pool;          /* [num_slots][n_kv][page_size][d]                    */
    const void* v_pool;          /* same layout; may be NULL for key-only (Mask bank)  */
    const void* k_host;          /* optional device-mapped host tier [num_pages][...]  */
    const void* v_host;
    const int32_t* page_table;   /* [num_pages] page -> slot (-1 miss); NULL = identity */
    uint8_t* touched;            /* optional [num_pages] flags: 1 hit, 2 miss (phase)  */
    int32_t num_pages;
    int32_t page_size;
    int32_t n_kv;
    int32_t d;
    int32_t dtype;               /* hp_dtype */
    int32_t t_kv;                /* valid tokens (bounds) */
    /* optional instrumentation: bit (kv * row_bits_stride + token) is set for every
     * key row read (distinct-row / algorithmic-byte accounting; NULL = off) */
    uint32_t* row_bits;
    int64_t row_bits_stride;
} hp_kv_view;

/* RoPE context (StageContext, pruning.hpp:55-63 + RopePolicySet, rope_policy.hpp:24-34).
 * cos/sin: device fp32 [rope_max][d/2], built by hp_build_rope_table (bit-identical
 * to build_rope_table, tensor.cpp:30-59). */
typedef struct hp_rope_ctx {
    const float* cos_tab;
    const float* sin_tab;
    int64_t rope_max;
    int32_t extension;           /* RopePolicySet::extension_enabled                  */
    int32_t early_cutoff;        /* early_layer_cutoff (layers are 1-based)            */
    int32_t early_policy;        /* hp_rope_policy for layers <= cutoff                */
    int32_t late_policy;         /* hp_rope_policy for layers > cutoff                 */
    int32_t layer;               /* 1-based layer (StageContext::layer)                */
    int32_t pad_;
} hp_rope_ctx;

/* Host helper: the reference's double-precision table, cast to float. */
int hp_build_rope_table(int64_t max_pos, int32_t d, float theta, float* cos_out, float* sin_out);

/* ------------------------------------------------------------------------ *
 * One pruning stage over a batch of (mask, query-block) index lists.
 * Replaces run_pruning_stage + select_rep + block_scores
 * (pruning.cpp:69-98,153-200; tensor.cpp:88-114) with index-exact results.
 * ------------------------------------------------------------------------ */
typedef struct hp_stage_args {
    /* stage S = (b_q, l_c, k)  (StageConfig, pruning.hpp:15-21) */
    int32_t query_block;
    int32_t chunk_size;
    int32_t keep;
    /* batch geometry */
    int32_t n_masks;             /* independent pooled masks (KV groups)               */
    int32_t heads_per_mask;      /* q-heads pooled into one chunk score                */
    int32_t n_q_heads;
    int32_t n_blocks;            /* query blocks per mask                              */
    int32_t q_rows;              /* rows of q per head (T_q)                           */
    const float* q;              /* [n_q_heads][q_rows][d]                             */
    int64_t query_offset;        /* absolute position of q row 0 (T_kv - T_q)          */
    int32_t stream_tokens;       /* StageContext::stream_tokens                        */
    int32_t max_chunks;          /* upper bound on chunks per list (grid sizing)       */
    /* input: range mode (in_list == NULL): list(m,b) = [in_start[mb], in_start[mb]+in_count[mb])
     *        list mode: in_list[mb*in_stride + i], i < in_count[mb] (sorted, unique) */
    const int32_t* in_list;
    const int32_t* in_start;
    const int32_t* in_count;
    int64_t in_stride;
    /* output: out_list[mb*out_stride + i], out_count[mb]; out_stride >= keep (or >= in for identity) */
    int32_t* out_list;
    int32_t* out_count;
    int64_t out_stride;
    /* workspace: >= hp_stage_workspace_bytes() bytes of device memory */
    void* workspace;
    size_t workspace_bytes;
    hp_kv_view keys;
    hp_rope_ctx rope;
    /* optional device flag (NULL = unknown): nonzero when every bf16 key is 0 or has
     * |k| in [2^-63, 2^63], so bf16 q*k products are exact in fp32 and the sequential
     * dot may run as one fused multiply-add per element (same result, fewer instructions) */
    const int32_t* keys_exact;
    /* optional (NULL = off): each descent's branch decisions, bit `it` set when
     * iteration `it` went right — path_out[(list * max_chunks + chunk) * heads_per_mask + head].
     * With the chunk lists this reproduces the reference's exact key-read sequence
     * (select_rep_rotated, pruning.cpp:69-98) for KeySource instrumentation. */
    uint32_t* path_out;
    /* 1: run the descents even when the stage is the identity (select_rep on one chunk) */
    int32_t descend_always;
    int32_t pad2_;
} hp_stage_args;

size_t hp_stage_workspace_bytes(int32_t n_lists, int32_t max_chunks, int32_t keep, int32_t chunk_size);
int hp_prune_stage(const hp_stage_args* args, void* stream);

/* Which descent hp_prune_stage launches (host-only query, no launch): query-block stages
 * (16..64 q rows, <= 8 heads per mask) over bf16 keys with the keys_exact flag, d = 128, RoPE off,
 * score rows on the tensor cores with a certified error bound and settle every undecided
 * comparison and the top-K boundary with exact dots; everything else runs the CUDA-core
 * descent. Both give the reference's indices. */
enum hp_prune_variant { HP_PRUNE_CUDA_CORE = 0, HP_PRUNE_TENSOR_CORE = 1 };
int hp_prune_stage_variant(const hp_stage_args* args, int32_t* variant);

/* Sub-block remap between stages with different b_q (pruning.cpp:285-303):
 * next(m2) = { idx in parent(min(m2/ratio, nb-1)) : idx < middle_upper(bq_next, m2) }. */
int hp_remap_blocks(const int32_t* in_list, const int32_t* in_count, int64_t in_stride,
                    int32_t n_masks, int32_t n_blocks, int32_t bq, int32_t bq_next, int32_t t_q,
                    int64_t query_offset, int32_t stream_tokens, int32_t* out_list,
                    int32_t* out_count, int64_t out_stride, void* stream);

/* Per-row selected index list (selected_indices, sparse_attention.cpp:95-112):
 * sinks [0,min(n_sink,pos+1)) ++ mask∩[sink_end,stream_begin) ++ [stream_begin,pos]. */
int hp_selected_indices(const int32_t* mask_list, const int32_t* mask_count, int64_t mask_stride,
                        int32_t n_masks, int32_t n_rows, int32_t block_size, int64_t query_offset,
                        int32_t sink_tokens, int32_t stream_tokens, int32_t* sel_list,
                        int32_t* sel_count, int64_t sel_stride, void* stream);

/* ------------------------------------------------------------------------ *
 * Block-sparse attention over explicit per-row selected lists: split-K with
 * online softmax + log-sum-exp combine. Replaces attention_row +
 * softmax_weighted_sum (sparse_attention.cpp:15-60) for decode and for
 * block_sparse_attention (sparse_attention.cpp:114-145) row by row.
 * ------------------------------------------------------------------------ */
typedef struct hp_bsa_args {
    int32_t n_q_heads;
    int32_t heads_per_mask;      /* q-head h uses the lists of mask h / heads_per_mask  */
    int32_t n_rows;              /* query rows per head                                  */
    const float* q;              /* [n_q_heads][n_rows][d]                              */
    int64_t query_offset;        /* position of row r = query_offset + r                 */
    const int32_t* sel_list;     /* [n_masks][n_rows][sel_stride]                       */
    const int32_t* sel_count;    /* [n_masks][n_rows]                                   */
    int64_t sel_stride;
    int32_t max_sel;             /* upper bound on counts (grid sizing)                 */
    float* out;                  /* [n_q_heads][n_rows][d] fp32                          */
    /* optional per-split partials for a cross-shard merge (NULL = combine in place):
     * m, l [n_q_heads][n_rows], o [n_q_heads][n_rows][d] — the shard's LSE triple */
    float* part_m;
    float* part_l;
    float* part_o;
    void* workspace;
    size_t workspace_bytes;
    hp_kv_view kv;
    hp_rope_ctx rope;            /* extension on => streaming positions (BSA policy)    */
} hp_bsa_args;

size_t hp_bsa_workspace_bytes(int32_t n_q_heads, int32_t n_rows, int32_t max_sel, int32_t d);
int hp_bsa(const hp_bsa_args* args, void* stream);

/* ------------------------------------------------------------------------ *
 * Prefill block-sparse attention on the tensor cores (tcgen05 + TMEM): each
 * query block's rows x its union of selected keys as 128 x 128 MMA tiles, the
 * per-row selection (selected_indices, sparse_attention.cpp:95-112) applied as a
 * mask on the scores, online softmax, O accumulated in TMEM. Replaces
 * block_sparse_attention (sparse_attention.cpp:114-145) for bf16 K/V, d = 128,
 * extension off; Q and P enter the tensor cores as bf16 (bf16 tolerance).
 * ------------------------------------------------------------------------ */
typedef struct hp_bsa_prefill_args {
    int32_t n_q_heads;
    int32_t heads_per_mask;      /* q-heads pooled into one mask (one KV group)          */
    int32_t n_rows;              /* T_q                                                 */
    int32_t block_size;          /* mask block size b_q (divides 128)                   */
    const float* q;              /* [n_q_heads][n_rows][128] fp32                       */
    int64_t query_offset;        /* T_kv - T_q                                          */
    const int32_t* mask_list;    /* [n_masks][n_mask_blocks][mask_stride] middle indices */
    const int32_t* mask_count;   /* [n_masks][n_mask_blocks]                            */
    int64_t mask_stride;
    int32_t n_mask_blocks;
    int32_t max_mask;            /* upper bound on mask_count                           */
    int32_t sink_tokens;
    int32_t stream_tokens;
    float* out;                  /* [n_q_heads][n_rows][128] fp32                       */
    hp_kv_view kv;               /* bf16, d = 128                                       */
} hp_bsa_prefill_args;

size_t hp_bsa_prefill_smem_bytes(int32_t max_union);
int hp_bsa_prefill(const hp_bsa_prefill_args* args, void* stream);

/* ------------------------------------------------------------------------ *
 * Fused decode path (one query row per q-head, d = 128): the per-layer body of
 * DecodeEngine::step (decode.cpp:225-273) as 1 kernel per stage + 1 BSA kernel.
 * Stage outputs stay implicit between kernels: a stage emits only its kept
 * chunk ids (sel) and the next stage resolves list positions through them
 * (hp_list_ref); hp_decode_materialize expands any stage's list on demand
 * (the DecodeEngine stage caches, decode.hpp:85-90).
 * ------------------------------------------------------------------------ */
typedef struct hp_list_ref {
    int32_t depth;               /* number of chunk-selection hops (<= 4)               */
    int32_t pad_;
    const int32_t* sel[4];       /* hop i: kept chunk ids [n_masks][sel_stride[i]]       */
    int32_t sel_stride[4];
    int32_t lc[4];               /* chunk size of hop i                                 */
    const int32_t* base_list;    /* NULL => base is the range [range_start, ...)        */
    int64_t base_stride;
    int64_t range_start;
} hp_list_ref;

typedef struct hp_decode_stage_args {
    int32_t chunk_size;
    int32_t keep;
    int32_t n_masks;
    int32_t heads_per_mask;
    int32_t n_q_heads;
    int32_t stream_tokens;
    const float* q;              /* [n_q_heads][d] fp32                                 */
    int64_t query_position;      /* T - 1                                               */
    hp_list_ref in;              /* input list per mask                                 */
    const int32_t* in_count;     /* [n_masks] device counts, or NULL => in_count_const  */
    int64_t in_count_const;
    int32_t max_chunks;          /* >= ceil(in_count / chunk_size)                      */
    int32_t sel_stride;          /* >= keep / chunk_size                                */
    int32_t* sel_out;            /* [n_masks][sel_stride] kept chunk ids, ascending; NULL =
                                    descent only (chunk scores left in the workspace)      */
    int32_t* out_count;          /* [n_masks] output list length                        */
    void* workspace;             /* >= hp_decode_stage_workspace_bytes()                */
    size_t workspace_bytes;
    hp_kv_view keys;
    hp_rope_ctx rope;
    /* optional device int: nonzero when every key element is bf16 with |k| in
     * [2^-63, 2^63] or 0. With bf16-exact q (checked in-kernel) every q*k product
     * is then exact in fp32, so fma(q,k,acc) == acc + q*k bit for bit and the
     * sequential dot issues one FFMA per element instead of FMUL + FADD. */
    const int32_t* keys_exact;
    /* optional: also write the stage's output token list, list_out[m*stride + i] for
     * i < out_count[m] (resolved through `in`), so a consumer needs no chain hops */
    int32_t* list_out;
    int64_t list_out_stride;
    /* optional: chunk scores (max over the mask's heads) land here, [n_masks][max_chunks],
     * instead of the workspace — with sel_out == NULL this is the descent of one shard of
     * a sequence-sharded stage, selected globally by hp_select_topk */
    float* scores_out;
} hp_decode_stage_args;

size_t hp_decode_stage_workspace_bytes(int32_t n_masks, int32_t max_chunks);
int hp_decode_stage(const hp_decode_stage_args* args, void* stream);

/* Which descent kernel hp_decode_stage launches for these arguments (host-only query,
 * no launch): the one-wave kernel for big stages (>= ~2K warps of descents), all-rows
 * for l_c <= 8, the two-comparison lookahead kernel for other bf16 stages, the classic
 * one-row-per-round kernel otherwise (and whenever RoPE extension is on). */
enum hp_stage_variant { HP_STAGE_CLASSIC = 0, HP_STAGE_LOOKAHEAD = 1, HP_STAGE_WIDE = 2, HP_STAGE_ALLROWS = 3 };
int hp_decode_stage_variant(const hp_decode_stage_args* args, int32_t* variant);

/* The stage's chunk selection on its own (run_pruning_stage's stable top-K,
 * pruning.cpp:187-192): per mask, keep the keep/chunk_size best of ceil(n_in/chunk_size)
 * scores (score desc, chunk asc), kept chunk ids ascending in sel_out, the stage output
 * length in out_count (identity when n_in <= keep). scores [n_masks][stride];
 * n_in: device counts [n_masks] or NULL => n_in_const. For sequence sharding: the
 * all-gathered scores of every shard give every rank the same global selection. */
int hp_select_topk(const float* scores, int64_t stride, int32_t n_masks, const int32_t* n_in,
                   int64_t n_in_const, int32_t chunk_size, int32_t keep, int32_t* sel_out,
                   int32_t sel_stride, int32_t* out_count, void* stream);

/* Sequence-sharded stage selection (C5): `gathered` [n_ranks][n_masks][width] holds every
 * rank's chunk scores of the stage (rank r's first counts[r][m] valid; ranks in global
 * chunk order), as an all-gather leaves them. Per mask: the global stable top-K (same
 * as hp_select_topk on the concatenated scores) -> sel_global / count_global, and this
 * rank's part of it -> sel_local (kept chunk ids inside the rank's range, local, ascending)
 * and len_local (the rank's share of the stage output). Identical on every rank. */
int hp_select_topk_sharded(const float* gathered, const int32_t* counts, int32_t n_ranks, int32_t width,
                           int32_t rank, int32_t n_masks, const int32_t* n_in, int64_t n_in_const,
                           int32_t chunk_size, int32_t keep, int32_t* sel_global, int32_t sel_stride,
                           int32_t* count_global, int32_t* sel_local, int32_t* len_local, void* stream);

typedef struct hp_decode_bsa_args {
    int32_t n_q_heads;
    int32_t heads_per_mask;
    int32_t sink_tokens;
    int32_t stream_tokens;
    const float* q;              /* [n_q_heads][d] fp32                                 */
    int64_t query_position;
    hp_list_ref mask;            /* middle indices per mask (all in [sink_end, stream_begin)) */
    const int32_t* mask_count;   /* [n_masks] */
    int32_t max_mask;            /* upper bound on mask counts                          */
    float* out;                  /* [n_q_heads][d] fp32                                 */
    float* part_m;               /* optional shard LSE triple (m, l [n_q_heads], o [n_q_heads][d]) */
    float* part_l;
    float* part_o;
    void* workspace;
    size_t workspace_bytes;
    hp_kv_view kv;
    hp_rope_ctx rope;
    /* 1 = the mask lists/counts and every K/V row except the newest token's (position
     * query_position) are already final when the launch is enqueued — no launch still in
     * flight writes them (e.g. a step that reuses the cached last stage). The kernel then
     * gathers those rows in its PDL prologue, overlapping the previous kernel's tail.
     * Ignored with a page table (cached KV). 0 = wait first (always safe). */
    int32_t mask_stable;
} hp_decode_bsa_args;

/* The workspace starts with per-head-group last-CTA ticket counters: zero it once before
 * first use (cudaMemset); every launch leaves the counters at zero for the next one. */
size_t hp_decode_bsa_workspace_bytes(int32_t n_q_heads, int32_t max_sel);
int hp_decode_bsa(const hp_decode_bsa_args* args, void* stream);

/* Which BSA kernel hp_decode_bsa launches for these arguments (validates them, no launch;
 * queries the device's cluster occupancy): the thread-block-cluster kernel merging over
 * distributed shared memory, or the split-K kernel whose last CTA merges (ticket). */
enum hp_bsa_variant { HP_BSA_TICKET = 0, HP_BSA_CLUSTER = 1 };
int hp_decode_bsa_variant(const hp_decode_bsa_args* args, int32_t* variant);

/* ------------------------------------------------------------------------ *
 * The whole per-layer decode body in two launches (d = 128, bf16 K/V, RoPE
 * extension off): stage 0's descent (hp_decode_stage's kernels, scores only),
 * then ONE kernel per layer in which a thread-block cluster per KV group runs
 * stage 0's selection, every later due stage (descent + exact top-K), and the
 * block-sparse attention with its log-sum-exp combine — the selections and the
 * merge exchange data through distributed shared memory, so nothing between the
 * stages is a kernel boundary. Same results as hp_decode_stage + hp_decode_bsa
 * (selections index-exact; output within the fp32 tolerance).
 * Replaces DecodeEngine::step's per-layer body (decode.cpp:225-273): stages due
 * this step (refresh[i]) chain through each other (stage i reads stage i-1's list
 * when i-1 also ran, else the cached list cache[i-1] with count[i-1]); the BSA
 * reads the last stage's list. Stage i's kept chunk ids land in sel[i] and its
 * output length in count[i] (the stage caches are then expanded on demand with
 * hp_decode_materialize, e.g. on a side stream).
 * ------------------------------------------------------------------------ */
typedef struct hp_decode_layer_args {
    int32_t n_stages;            /* 1..4                                                  */
    int32_t chunk_size[4];
    int32_t keep[4];
    int32_t refresh[4];          /* 1 = stage due this step (refresh_due, decode.cpp:212-224) */
    int32_t n_masks;             /* KV groups, one pooled mask each                       */
    int32_t heads_per_mask;      /* 1, 2, 4 or 8; a mask's heads share one kv head        */
    int32_t n_q_heads;
    int32_t sink_tokens;
    int32_t stream_tokens;
    int32_t pad_;
    const float* q;              /* [n_q_heads][128] fp32                                 */
    int64_t query_position;      /* T - 1; stage 0 reads [n_sink, T - n_stream)           */
    int32_t* sel[4];             /* [n_masks][sel_stride[i]] kept chunk ids (written if due) */
    int32_t sel_stride[4];       /* >= keep[i] / chunk_size[i]                            */
    int32_t* count[4];           /* [n_masks] stage output lengths (written if due)       */
    const int32_t* cache[4];     /* [n_masks][cache_stride[i]] materialized stage lists   */
    int64_t cache_stride[4];
    float* out;                  /* [n_q_heads][128] fp32                                 */
    void* workspace;             /* >= hp_decode_layer_workspace_bytes()                  */
    size_t workspace_bytes;
    hp_kv_view kv;               /* bf16, d = 128                                         */
    const int32_t* keys_exact;   /* as in hp_decode_stage_args                            */
} hp_decode_layer_args;

size_t hp_decode_layer_workspace_bytes(int32_t n_masks, int32_t max_chunks0);
/* 1 when hp_decode_layer takes this configuration, 0 otherwise (then use the
 * per-stage entry points); no launch. */
int hp_decode_layer_supported(const hp_decode_layer_args* args);
/* The layer kernel is a persistent grid (one CTA per SM, the CTAs of a KV group meeting at
 * barriers in L2): do not run two hp_decode_layer launches concurrently on one device
 * (different streams of one context) — each could hold SMs the other's barriers wait for.
 * Stream-ordered launches (one stream, or graphs) and other kernels alongside are fine. */
int hp_decode_layer(const hp_decode_layer_args* args, void* stream);

/* Append one token's K/V rows (DecodeEngine::step, decode.cpp:202-208): rows
 * [n_kv][d] (same dtype as the pools) land at `token` of the paged pools; keys_exact
 * (optional device int) is cleared if a new key breaks the exact-product range. */
int hp_decode_append(const hp_kv_view* kv, const void* k_rows, const void* v_rows, int64_t token,
                     int32_t* keys_exact, void* stream);

/* Expand lists: out[m][i] = ref(m, i) for i < count[m] (n_lists refs at once). */
int hp_decode_materialize(const hp_list_ref* refs, const int32_t* const* counts,
                          int32_t* const* outs, const int64_t* out_strides, int32_t n_lists,
                          int32_t n_masks, int32_t max_count, void* stream);


/* ------------------------------------------------------------------------ *
 * On-GPU LRU page cache over a pinned host tier (replaces TieredKvStore::
 * access_pages / commit and KvView::account, kv_store.cpp:58-120,188-200).
 * Point an hp_kv_view at it (k_pool = k_slots, k_host = k_host, page_table,
 * touched): every gather then reads resident pages from their slot and missing
 * pages from the mapped host tier in the same kernel, flagging touched[page]
 * (1 hit, 2 miss). hp_cache_commit is the step-end commit: hits take `stamp`,
 * misses are installed into the least-recently-used slots (host -> slot copies
 * on the device), stats[0..2] += hits, misses, evictions, touched is cleared.
 * stamp 0 = use (and advance) a step clock kept in the workspace, so a captured
 * CUDA graph can replay the commit; explicit stamps must be > 1 (1 = warm start).
 * The workspace must be zeroed before first use.
 * ------------------------------------------------------------------------ */
typedef struct hp_page_cache {
    void* k_slots;               /* [num_slots][n_kv][page_size][d] device             */
    void* v_slots;               /* same, or NULL (key-only cache)                      */
    const void* k_host;          /* [num_pages][n_kv][page_size][d] pinned, device-mapped */
    const void* v_host;
    int32_t* page_table;         /* [num_pages] page -> slot, -1 = host only            */
    int32_t* slot_page;          /* [num_slots] slot -> page, -1 = free                 */
    uint32_t* slot_stamp;        /* [num_slots] logical time of last use (0 = free)     */
    uint8_t* touched;            /* [num_pages] per-step access flags                   */
    int32_t num_pages;
    int32_t num_slots;           /* <= 16384 */
    int32_t page_size;
    int32_t n_kv;
    int32_t d;
    int32_t dtype;               /* hp_dtype */
} hp_page_cache;

size_t hp_cache_workspace_bytes(int32_t num_pages, int32_t num_slots);
int hp_cache_commit(const hp_page_cache* cache, uint32_t stamp, int32_t* stats, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Log-sum-exp merge of per-shard (m, l, o) partials (C5 sequence sharding):
 * m, l [n_shards][n]; o [n_shards][n][d] -> out [n][d]. */
int hp_lse_merge(const float* m, const float* l, const float* o, int32_t n_shards, int32_t n,
                 int32_t d, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HIPPRUNE_B200_H */

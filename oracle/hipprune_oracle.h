/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference hipprune hot path (the "port" oracle).
 * Each function cites the reference file:line it follows (paths relative to
 * /root/reference/proj). Parity is PINNED: tests/test_oracle_pin.py checks this
 * port bit-for-bit against the unmodified reference (oracle/_ref/libhipref.so,
 * built from the reference sources) and against the committed golden vectors
 * in tests/golden/ that the reference produced (tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as the checker. The product path never calls into it.
 *
 * Conventions shared with oracle/ref_shim.cpp and the CUDA C-ABI:
 *   q : [n_heads][rows][d] fp32,  k/v : [n_kv][t_kv][d] fp32,
 *   q-head h reads kv-head h / (n_heads / n_kv);  index lists are int64.
 *   Return codes: 0 ok, 1 ContractViolation, 2 invalid_argument, 3 out_of_range,
 *   4 logic_error, 5 runtime_error, 6 PartialCommitError.
 */
#ifndef HIPPRUNE_ORACLE_H
#define HIPPRUNE_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_last_error_code(void);

/* list-set handles (vector<vector<size_t>>) */
size_t orc_lists_count(void* h);
size_t orc_lists_len(void* h, size_t i);
void orc_lists_get(void* h, size_t i, int64_t* out);
void orc_lists_free(void* h);
void* orc_lists_from(const int64_t* flat, const size_t* lens, size_t n);

int orc_build_rope_table(size_t max_pos, size_t d, float theta, float* cos_out, float* sin_out);

void* orc_run_pruning_stage(size_t bq, size_t lc, size_t keep, const int64_t* idx, size_t n,
                            const float* q, size_t n_heads, size_t rows, const float* k,
                            size_t n_kv, size_t t_kv, size_t d, size_t layer1, size_t stream,
                            size_t qstart, int ext, size_t cutoff, size_t rope_max,
                            uint64_t* reads_total, uint64_t* reads_distinct);

int orc_select_rep(const float* q, size_t rows, const int64_t* chunk, size_t n, const float* k,
                   size_t t_kv, size_t d, size_t layer1, size_t stream, size_t qstart, int ext,
                   size_t cutoff, size_t chunk_index, size_t chunk_count, size_t rope_max,
                   int64_t* rep_out, int64_t* reads_out, size_t* n_reads);

void* orc_build_mask(const float* q, const float* k, size_t n_heads, size_t n_kv, size_t t_q,
                     size_t t_kv, size_t d, size_t layer0, const size_t* stages, size_t n_stages,
                     size_t sink, size_t stream, int ext, size_t cutoff, size_t threads,
                     void** trace_out, size_t* block_size_out, size_t* query_offset_out);

void* orc_selected_indices(void* lists, size_t block_size, size_t sink, size_t stream,
                           size_t offset, size_t row);

int orc_attention_row(const float* q, const int64_t* sel, size_t n, size_t pos, int ext,
                      const float* k, const float* v, size_t t_kv, size_t d, size_t rope_max,
                      float* out);

int orc_block_sparse_attention(const float* q, const float* k, const float* v, size_t n_heads,
                               size_t n_kv, size_t t_q, size_t t_kv, size_t d, void* lists,
                               size_t block_size, size_t sink, size_t stream, size_t offset,
                               int ext, float* out);

int orc_dense_attention(const float* q, const float* k, const float* v, size_t n_heads,
                        size_t t_q, size_t t_kv, size_t d, float* out);

void* orc_exact_topk(const float* q, const float* keys, size_t rows, size_t d, size_t k);
double orc_attention_recall(const int64_t* sel, size_t n, const float* q, const float* keys,
                            size_t rows, size_t d);

int orc_decode_layer_step(const float* q, const float* k, const float* v, size_t groups,
                          size_t hpm, size_t t, size_t d, const size_t* stages, size_t n_stages,
                          size_t sink, size_t stream, int ext, size_t layer1, size_t cutoff,
                          size_t threads, int kv_shared, int64_t* mask_out, size_t cap,
                          size_t* mask_len, float* out, double* seconds);

/* paged two-bank LRU store (kv_store.cpp) */
void* orc_store_new(size_t num_layers, size_t page_size, size_t mask_cap, size_t sa_cap);
void orc_store_free(void* h);
int orc_store_page_of(void* h, size_t layer, size_t token, uint64_t* out);
int orc_store_access(void* h, int bank, const uint64_t* pages, size_t n, uint64_t* missing,
                     size_t* n_missing);
int orc_store_commit(void* h, int bank, const uint64_t* pages, size_t n, uint64_t* evicted,
                     size_t* n_evicted);
size_t orc_store_recency(void* h, int bank, uint64_t* out, size_t cap);
void orc_store_stats(void* h, int bank, uint64_t* out3);
int orc_store_check(void* h);

#ifdef __cplusplus
}
#endif
#endif

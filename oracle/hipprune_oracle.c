/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See hipprune_oracle.h.
 *
 * A sequential, single-precision restatement of the reference hot path. Every
 * float operation is separately rounded (built with -ffp-contract=off) and
 * performed in the reference's order, so results are bit-identical to the
 * reference library (pinned by tests/test_oracle_pin.py).
 */
#define _GNU_SOURCE
#include "hipprune_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];
static __thread int g_err_code;

enum { OK = 0, E_CONTRACT = 1, E_INVALID = 2, E_RANGE = 3, E_LOGIC = 4, E_RUNTIME = 5, E_PARTIAL = 6 };

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_err_code = code;
    return code;
}
static int ok(void) { g_err[0] = 0; g_err_code = OK; return OK; }
const char* orc_last_error(void) { return g_err; }
int orc_last_error_code(void) { return g_err_code; }

/* ------------------------------------------------------------- list sets */
typedef struct { int64_t* v; size_t n, cap; } List;
typedef struct { List* l; size_t n; } Lists;

static void list_push(List* l, int64_t x) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 16;
        l->v = (int64_t*)realloc(l->v, l->cap * sizeof(int64_t));
    }
    l->v[l->n++] = x;
}
static void list_free(List* l) { free(l->v); l->v = NULL; l->n = l->cap = 0; }
static Lists* lists_new(size_t n) {
    Lists* s = (Lists*)calloc(1, sizeof(Lists));
    s->n = n;
    s->l = (List*)calloc(n ? n : 1, sizeof(List));
    return s;
}
size_t orc_lists_count(void* h) { return ((Lists*)h)->n; }
size_t orc_lists_len(void* h, size_t i) { return ((Lists*)h)->l[i].n; }
void orc_lists_get(void* h, size_t i, int64_t* out) {
    List* l = &((Lists*)h)->l[i];
    if (l->n) memcpy(out, l->v, l->n * sizeof(int64_t));
}
void orc_lists_free(void* h) {
    Lists* s = (Lists*)h;
    if (!s) return;
    for (size_t i = 0; i < s->n; ++i) list_free(&s->l[i]);
    free(s->l);
    free(s);
}
void* orc_lists_from(const int64_t* flat, const size_t* lens, size_t n) {
    Lists* s = lists_new(n);
    size_t off = 0;
    for (size_t i = 0; i < n; ++i) {
        for (size_t j = 0; j < lens[i]; ++j) list_push(&s->l[i], flat[off + j]);
        off += lens[i];
    }
    return s;
}

/* ------------------------------------------------------------------ rope
 * build_rope_table (tensor.cpp:30-59): freq_i = theta^(-2i/d) in double,
 * angle = p * freq_i in double, cos/sin in double, cast to float. The port
 * evaluates the same expression on demand (memoised per position). */
typedef struct { size_t pos; size_t d; float theta; float* cs; } RopeRow; /* cs: [d/2 cos | d/2 sin] */
#define ROPE_SLOTS 4096
static __thread RopeRow g_rope[ROPE_SLOTS];

static const float* rope_row(size_t pos, size_t d, float theta) {
    RopeRow* r = &g_rope[pos % ROPE_SLOTS];
    if (r->cs && r->pos == pos && r->d == d && r->theta == theta) return r->cs;
    const size_t half = d / 2;
    free(r->cs);
    r->cs = (float*)malloc(d * sizeof(float));
    for (size_t i = 0; i < half; ++i) {
        const double freq = pow((double)theta, -2.0 * (double)i / (double)d);
        const double angle = (double)pos * freq;
        r->cs[i] = (float)cos(angle);
        r->cs[half + i] = (float)sin(angle);
    }
    r->pos = pos;
    r->d = d;
    r->theta = theta;
    return r->cs;
}

int orc_build_rope_table(size_t max_pos, size_t d, float theta, float* cos_out, float* sin_out) {
    if (d == 0 || d % 2) return fail(E_INVALID, "build_rope_table: head_dim must be even and positive");
    if (max_pos == 0) return fail(E_INVALID, "build_rope_table: max_position must be >= 1");
    if (!(theta > 0.0f)) return fail(E_INVALID, "build_rope_table: theta_base must be positive");
    const size_t half = d / 2;
    for (size_t p = 0; p < max_pos; ++p) {
        const float* cs = rope_row(p, d, theta);
        memcpy(cos_out + p * half, cs, half * sizeof(float));
        memcpy(sin_out + p * half, cs + half, half * sizeof(float));
    }
    return ok();
}

/* apply_rope_inplace (tensor.cpp:61-79): half-split pairs, x*c - y*s, x*s + y*c. */
static int apply_rope(float* vec, size_t d, size_t pos, size_t rope_max) {
    if (pos >= rope_max) return fail(E_RANGE, "apply_rope: position %zu >= max_position %zu", pos, rope_max);
    const size_t half = d / 2;
    const float* cs = rope_row(pos, d, 10000.0f);
    for (size_t i = 0; i < half; ++i) {
        const float x = vec[i], y = vec[i + half];
        const float c = cs[i], s = cs[half + i];
        vec[i] = x * c - y * s;
        vec[i + half] = x * s + y * c;
    }
    return OK;
}

/* dot_f32 (tensor.cpp:88-98): sequential left-to-right fp32. */
static float dot_f32(const float* a, const float* b, size_t d) {
    float acc = 0.0f;
    for (size_t i = 0; i < d; ++i) acc += a[i] * b[i];
    return acc;
}

/* block_scores (tensor.cpp:100-114): max over rows, strict '>' update. */
static float block_scores(const float* qb, size_t rows, const float* key, size_t d) {
    float best = dot_f32(qb, key, d);
    for (size_t t = 1; t < rows; ++t) {
        const float s = dot_f32(qb + t * d, key, d);
        if (s > best) best = s;
    }
    return best;
}

/* ---------------------------------------------------------- rope policy
 * query_position / key_position (rope_policy.cpp:18-57). Default policy set:
 * ChunkIndexed for layers <= cutoff, Relative above (rope_policy.hpp:24-34). */
static size_t q_position(size_t layer1, size_t cutoff, size_t qpos, size_t stream, size_t chunk_count) {
    if (layer1 > cutoff) return stream + 1;                         /* Relative */
    const size_t cap = chunk_count + stream;                          /* ChunkIndexed */
    return qpos < cap ? qpos : cap;
}
static size_t k_position(size_t layer1, size_t cutoff, int branch, size_t chunk_index) {
    if (layer1 > cutoff) return (size_t)(branch - 1);
    return chunk_index;
}

typedef struct {
    const float* k; size_t t_kv, d; size_t group;   /* kv = head / group */
    size_t layer1, cutoff, stream, qstart, rope_max; int ext;
    /* read logging */
    int log; uint64_t reads; int64_t* trace; size_t trace_n, trace_cap;
    uint8_t* seen; size_t seen_n; uint64_t distinct; size_t n_kv;
} Ctx;

static const float* key_row(Ctx* c, size_t head, int64_t token, int* err) {
    if (token < 0 || (size_t)token >= c->t_kv) { *err = fail(E_RANGE, "key_row: token out of range"); return NULL; }
    const size_t kv = head / c->group;
    if (c->log) {
        c->reads++;
        if (c->trace && c->trace_n < c->trace_cap) c->trace[c->trace_n++] = token;
        if (c->seen) {
            const size_t bit = kv * c->t_kv + (size_t)token;
            if (!(c->seen[bit >> 3] & (1u << (bit & 7)))) { c->seen[bit >> 3] |= (uint8_t)(1u << (bit & 7)); c->distinct++; }
        }
    }
    return c->k + (kv * c->t_kv + (size_t)token) * c->d;
}

/* rotate_queries (pruning.cpp:39-52): rows rotated at query_position. */
static int rotate_queries(Ctx* c, const float* qb, size_t rows, size_t chunk_count, float* out) {
    memcpy(out, qb, rows * c->d * sizeof(float));
    if (!c->ext) return OK;
    for (size_t t = 0; t < rows; ++t) {
        const size_t pos = q_position(c->layer1, c->cutoff, c->qstart + t, c->stream, chunk_count);
        int e = apply_rope(out + t * c->d, c->d, pos, c->rope_max);
        if (e) return e;
    }
    return OK;
}

/* rotate_key (pruning.cpp:54-67). */
static int rotate_key(Ctx* c, const float* key, int branch, size_t chunk_index, float* out) {
    memcpy(out, key, c->d * sizeof(float));
    if (!c->ext) return OK;
    return apply_rope(out, c->d, k_position(c->layer1, c->cutoff, branch, chunk_index), c->rope_max);
}

static size_t ceil_log2(size_t n) {
    size_t bits = 0, v = 1;
    while (v < n) { v <<= 1; ++bits; }
    return bits;
}

/* select_rep_rotated (pruning.cpp:69-98): Alg. 3 descent, 1-based [first,last],
 * mid rounds half up, right only on strict sigma2 > sigma1. */
static int select_rep_rotated(Ctx* c, const float* rq, size_t rows, const int64_t* chunk, size_t n,
                              size_t head, size_t chunk_index, int64_t* rep) {
    if (n == 0) return fail(E_CONTRACT, "select_rep: empty chunk");
    if (n == 1) { *rep = chunk[0]; return OK; }
    size_t first = 1, last = n;
    const size_t iters = ceil_log2(n);
    float key[1024];
    for (size_t it = 0; it < iters && first < last; ++it) {
        const size_t mid = (first + last + 1) / 2;
        float sigma[2];
        const int64_t reps[2] = {chunk[first - 1], chunk[mid - 1]};
        for (int j = 0; j < 2; ++j) {
            int e = 0;
            const float* row = key_row(c, head, reps[j], &e);
            if (e) return e;
            if ((e = rotate_key(c, row, j + 1, chunk_index, key))) return e;
            sigma[j] = block_scores(rq, rows, key, c->d);
        }
        if (sigma[1] > sigma[0]) first = mid; else last = mid - 1;
    }
    *rep = chunk[first - 1];
    return OK;
}

static int check_sorted_unique(const int64_t* idx, size_t n) {
    for (size_t i = 1; i < n; ++i)
        if (idx[i] <= idx[i - 1]) return fail(E_CONTRACT, "run_pruning_stage: indices must be sorted and duplicate-free");
    return OK;
}

static int stage_validate(size_t bq, size_t lc, size_t keep) {
    if (bq == 0 || lc == 0) return fail(E_INVALID, "StageConfig: b_q and l_c must be >= 1");
    if (keep == 0 || keep % lc) return fail(E_INVALID, "StageConfig: k must be a positive multiple of l_c");
    return OK;
}

typedef struct { const float* s; } SortCtx;
static __thread const float* g_sort_scores;
/* stable descending order == descending score, ties to the lower chunk index */
static int cmp_desc(const void* a, const void* b) {
    const size_t ia = *(const size_t*)a, ib = *(const size_t*)b;
    const float sa = g_sort_scores[ia], sb = g_sort_scores[ib];
    if (sa > sb) return -1;
    if (sb > sa) return 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}
static int cmp_size(const void* a, const void* b) {
    const size_t ia = *(const size_t*)a, ib = *(const size_t*)b;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

/* run_pruning_stage (pruning.cpp:153-200). qb: [n_heads][rows][d]. */
static int pruning_stage(Ctx* c, size_t bq, size_t lc, size_t keep, const int64_t* idx, size_t n,
                         const float* qb, size_t n_heads, size_t rows, List* out) {
    int e;
    if ((e = stage_validate(bq, lc, keep))) return e;
    if ((e = check_sorted_unique(idx, n))) return e;
    out->n = 0;
    if (n <= keep) { for (size_t i = 0; i < n; ++i) list_push(out, idx[i]); return OK; }
    const size_t chunk_count = (n + lc - 1) / lc;
    const size_t keep_chunks = keep / lc;
    if (chunk_count <= keep_chunks) { for (size_t i = 0; i < n; ++i) list_push(out, idx[i]); return OK; }
    const size_t d = c->d;
    float* rq = (float*)malloc(n_heads * rows * d * sizeof(float));
    for (size_t h = 0; h < n_heads; ++h)
        if ((e = rotate_queries(c, qb + h * rows * d, rows, chunk_count, rq + h * rows * d))) { free(rq); return e; }
    float* scores = (float*)malloc(chunk_count * sizeof(float));
    float key[1024];
    for (size_t j = 0; j < chunk_count; ++j) {
        const int64_t* chunk = idx + j * lc;
        const size_t len = (j + 1) * lc <= n ? lc : n - j * lc;
        float best = -INFINITY;
        for (size_t h = 0; h < n_heads; ++h) {
            int64_t rep;
            if ((e = select_rep_rotated(c, rq + h * rows * d, rows, chunk, len, h, j, &rep))) goto done;
            const float* row = key_row(c, h, rep, &e);
            if (e) goto done;
            if ((e = rotate_key(c, row, 2, j, key))) goto done;
            const float s = block_scores(rq + h * rows * d, rows, key, d);
            best = (best < s) ? s : best; /* std::max */
        }
        scores[j] = best;
    }
    {
        size_t* order = (size_t*)malloc(chunk_count * sizeof(size_t));
        for (size_t j = 0; j < chunk_count; ++j) order[j] = j;
        g_sort_scores = scores;
        qsort(order, chunk_count, sizeof(size_t), cmp_desc);
        qsort(order, keep_chunks, sizeof(size_t), cmp_size);
        for (size_t r = 0; r < keep_chunks; ++r) {
            const size_t j = order[r];
            const size_t end = (j + 1) * lc <= n ? (j + 1) * lc : n;
            for (size_t i = j * lc; i < end; ++i) list_push(out, idx[i]);
        }
        free(order);
    }
    e = OK;
done:
    free(scores);
    free(rq);
    return e;
}

static void ctx_init(Ctx* c, const float* k, size_t n_heads, size_t n_kv, size_t t_kv, size_t d,
                     size_t layer1, size_t stream, size_t qstart, int ext, size_t cutoff, size_t rope_max) {
    memset(c, 0, sizeof *c);
    c->k = k; c->t_kv = t_kv; c->d = d; c->n_kv = n_kv;
    c->group = n_kv ? n_heads / n_kv : 1;
    if (!c->group) c->group = 1;
    c->layer1 = layer1; c->stream = stream; c->qstart = qstart; c->ext = ext; c->cutoff = cutoff;
    c->rope_max = rope_max ? rope_max : t_kv + 2;
}

void* orc_run_pruning_stage(size_t bq, size_t lc, size_t keep, const int64_t* idx, size_t n,
                            const float* q, size_t n_heads, size_t rows, const float* k,
                            size_t n_kv, size_t t_kv, size_t d, size_t layer1, size_t stream,
                            size_t qstart, int ext, size_t cutoff, size_t rope_max,
                            uint64_t* reads_total, uint64_t* reads_distinct) {
    Ctx c;
    ctx_init(&c, k, n_heads, n_kv, t_kv, d, layer1, stream, qstart, ext, cutoff, rope_max);
    if (reads_total) {
        c.log = 1;
        c.seen = (uint8_t*)calloc((n_kv * t_kv + 7) / 8 + 1, 1);
    }
    Lists* out = lists_new(1);
    int e = pruning_stage(&c, bq, lc, keep, idx, n, q, n_heads, rows, &out->l[0]);
    if (reads_total) { *reads_total = c.reads; *reads_distinct = c.distinct; free(c.seen); }
    if (e) { orc_lists_free(out); return NULL; }
    ok();
    return out;
}

int orc_select_rep(const float* q, size_t rows, const int64_t* chunk, size_t n, const float* k,
                   size_t t_kv, size_t d, size_t layer1, size_t stream, size_t qstart, int ext,
                   size_t cutoff, size_t chunk_index, size_t chunk_count, size_t rope_max,
                   int64_t* rep_out, int64_t* reads_out, size_t* n_reads) {
    Ctx c;
    ctx_init(&c, k, 1, 1, t_kv, d, layer1, stream, qstart, ext, cutoff, rope_max);
    c.log = 1; c.trace = reads_out; c.trace_cap = 1 << 20;
    float* rq = (float*)malloc(rows * d * sizeof(float));
    int e = rotate_queries(&c, q, rows, chunk_count, rq);
    if (!e) e = select_rep_rotated(&c, rq, rows, chunk, n, 0, chunk_index, rep_out);
    free(rq);
    *n_reads = c.trace_n;
    return e ? e : ok();
}

/* ------------------------------------------------------------ build_mask
 * pruning.cpp:202-313 (Alg. 1): initial lists [n_sink, causal_end - n_stream),
 * stages over query blocks (ctx.layer = layer0 + 1, query_start = offset + row0),
 * trace of the last block per stage, sub-block remap with causal re-clamp. */
typedef struct {
    Ctx base; const float* q; size_t n_heads, t_q, bq, lc, keep, offset, d;
    List* lists; size_t num_blocks; size_t next; pthread_mutex_t mu; int err; char msg[512];
} MaskJob;

static int process_block(MaskJob* J, size_t m) {
    const size_t row_begin = m * J->bq;
    const size_t row_end = row_begin + J->bq < J->t_q ? row_begin + J->bq : J->t_q;
    const size_t rows = row_end - row_begin, d = J->d;
    float* qb = (float*)malloc(J->n_heads * rows * d * sizeof(float));
    for (size_t h = 0; h < J->n_heads; ++h)
        memcpy(qb + h * rows * d, J->q + (h * J->t_q + row_begin) * d, rows * d * sizeof(float));
    Ctx c = J->base;
    c.qstart = J->offset + row_begin;
    List out = {0};
    int e = pruning_stage(&c, J->bq, J->lc, J->keep, J->lists[m].v, J->lists[m].n, qb, J->n_heads, rows, &out);
    free(qb);
    if (e) { list_free(&out); return e; }
    list_free(&J->lists[m]);
    J->lists[m] = out;
    return OK;
}

static void* mask_worker(void* arg) {
    MaskJob* J = (MaskJob*)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const size_t m = J->next++;
        const int stop = J->err != 0 || m >= J->num_blocks;
        pthread_mutex_unlock(&J->mu);
        if (stop) break;
        int e = process_block(J, m);
        if (e) {
            pthread_mutex_lock(&J->mu);
            if (!J->err) { J->err = e; snprintf(J->msg, sizeof J->msg, "%s", g_err); }
            pthread_mutex_unlock(&J->mu);
        }
    }
    return NULL;
}

void* orc_build_mask(const float* q, const float* k, size_t n_heads, size_t n_kv, size_t t_q,
                     size_t t_kv, size_t d, size_t layer0, const size_t* stages, size_t n_stages,
                     size_t sink, size_t stream, int ext, size_t cutoff, size_t threads,
                     void** trace_out, size_t* block_size_out, size_t* query_offset_out) {
    int e;
    /* PruningPlan::validate (pruning.cpp:111-132) */
    if (n_stages == 0) { fail(E_INVALID, "PruningPlan: no stages"); return NULL; }
    for (size_t i = 0; i < n_stages; ++i)
        if ((e = stage_validate(stages[3 * i], stages[3 * i + 1], stages[3 * i + 2]))) return NULL;
    for (size_t i = 1; i < n_stages; ++i) {
        if (stages[3 * i] > stages[3 * (i - 1)] || stages[3 * (i - 1)] % stages[3 * i]) {
            fail(E_INVALID, "PruningPlan: successive b_q must be non-increasing and divisible");
            return NULL;
        }
        if (stages[3 * i + 2] > stages[3 * (i - 1) + 2]) { fail(E_INVALID, "PruningPlan: k must be non-increasing across stages"); return NULL; }
    }
    if (t_q == 0 || t_q > t_kv) { fail(E_INVALID, "build_mask: workload query length inconsistent"); return NULL; }
    const size_t offset = t_kv - t_q;
    size_t bq = stages[0];
    size_t num_blocks = (t_q + bq - 1) / bq;
    List* lists = (List*)calloc(num_blocks, sizeof(List));
    for (size_t m = 0; m < num_blocks; ++m) {
        const size_t end = offset + ((m + 1) * bq < t_q ? (m + 1) * bq : t_q);
        const size_t upper = end > stream ? end - stream : 0;
        for (size_t i = sink; i < upper; ++i) list_push(&lists[m], (int64_t)i);
    }
    Lists* trace = lists_new(n_stages);
    MaskJob J;
    memset(&J, 0, sizeof J);
    ctx_init(&J.base, k, n_heads, n_kv, t_kv, d, layer0 + 1, stream, 0, ext, cutoff, t_kv + 2);
    J.q = q; J.n_heads = n_heads; J.t_q = t_q; J.offset = offset; J.d = d;
    pthread_mutex_init(&J.mu, NULL);
    for (size_t si = 0; si < n_stages; ++si) {
        bq = stages[3 * si];
        J.bq = bq; J.lc = stages[3 * si + 1]; J.keep = stages[3 * si + 2];
        J.lists = lists; J.num_blocks = num_blocks; J.next = 0; J.err = 0;
        size_t workers = threads < num_blocks ? threads : num_blocks;
        if (workers <= 1) {
            for (size_t m = 0; m < num_blocks; ++m) if ((e = process_block(&J, m))) goto fail_out;
        } else {
            pthread_t* th = (pthread_t*)malloc(workers * sizeof(pthread_t));
            for (size_t w = 0; w < workers; ++w) pthread_create(&th[w], NULL, mask_worker, &J);
            for (size_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
            free(th);
            if (J.err) { e = fail(J.err, "%s", J.msg); goto fail_out; }
        }
        for (size_t i = 0; i < lists[num_blocks - 1].n; ++i) list_push(&trace->l[si], lists[num_blocks - 1].v[i]);
        if (si + 1 < n_stages) {
            const size_t bq_next = stages[3 * (si + 1)];
            if (bq_next != bq) {
                const size_t ratio = bq / bq_next;
                const size_t next_blocks = (t_q + bq_next - 1) / bq_next;
                List* next = (List*)calloc(next_blocks, sizeof(List));
                for (size_t m2 = 0; m2 < next_blocks; ++m2) {
                    const size_t p = m2 / ratio < num_blocks - 1 ? m2 / ratio : num_blocks - 1;
                    const size_t end = offset + ((m2 + 1) * bq_next < t_q ? (m2 + 1) * bq_next : t_q);
                    const size_t upper = end > stream ? end - stream : 0;
                    for (size_t i = 0; i < lists[p].n; ++i)
                        if ((size_t)lists[p].v[i] < upper) list_push(&next[m2], lists[p].v[i]);
                }
                for (size_t m = 0; m < num_blocks; ++m) list_free(&lists[m]);
                free(lists);
                lists = next;
                num_blocks = next_blocks;
            }
        }
    }
    pthread_mutex_destroy(&J.mu);
    {
        Lists* out = lists_new(0);
        free(out->l);
        out->l = lists; out->n = num_blocks;
        if (trace_out) *trace_out = trace; else orc_lists_free(trace);
        if (block_size_out) *block_size_out = stages[3 * (n_stages - 1)];
        if (query_offset_out) *query_offset_out = offset;
        ok();
        return out;
    }
fail_out:
    pthread_mutex_destroy(&J.mu);
    for (size_t m = 0; m < num_blocks; ++m) list_free(&lists[m]);
    free(lists);
    orc_lists_free(trace);
    return NULL;
}

/* ------------------------------------------------------- sparse attention */
/* selected_indices (sparse_attention.cpp:95-112) */
static int selected(const Lists* mask, size_t block_size, size_t sink, size_t stream, size_t offset,
                    size_t row, List* out) {
    const size_t block = row / block_size;
    if (block >= mask->n) return fail(E_RANGE, "selected_indices: row outside the mask");
    const size_t pos = offset + row;
    const size_t sink_end = sink < pos + 1 ? sink : pos + 1;
    size_t stream_begin = pos + 1 > stream ? pos + 1 - stream : 0;
    if (stream_begin < sink_end) stream_begin = sink_end;
    out->n = 0;
    for (size_t j = 0; j < sink_end; ++j) list_push(out, (int64_t)j);
    const List* l = &mask->l[block];
    for (size_t i = 0; i < l->n; ++i)
        if ((size_t)l->v[i] >= sink_end && (size_t)l->v[i] < stream_begin) list_push(out, l->v[i]);
    for (size_t j = stream_begin; j <= pos; ++j) list_push(out, (int64_t)j);
    return OK;
}

void* orc_selected_indices(void* lists, size_t block_size, size_t sink, size_t stream,
                           size_t offset, size_t row) {
    Lists* out = lists_new(1);
    if (selected((Lists*)lists, block_size, sink, stream, offset, row, &out->l[0])) { orc_lists_free(out); return NULL; }
    ok();
    return out;
}

/* softmax_weighted_sum (sparse_attention.cpp:15-29) */
static void softmax_weighted_sum(float* scores, const int64_t* sel, size_t n, const float* v,
                                 size_t d, float* out) {
    float mx = scores[0];
    for (size_t j = 0; j < n; ++j) mx = (mx < scores[j]) ? scores[j] : mx;
    float denom = 0.0f;
    for (size_t j = 0; j < n; ++j) { scores[j] = expf(scores[j] - mx); denom += scores[j]; }
    for (size_t j = 0; j < n; ++j) {
        const float w = scores[j] / denom;
        const float* vr = v + (size_t)sel[j] * d;
        for (size_t c = 0; c < d; ++c) out[c] += w * vr[c];
    }
}

/* attention_row (sparse_attention.cpp:33-60); k/v: one head [t_kv][d]. */
static int attention_row(const float* q, const int64_t* sel, size_t n, size_t pos, int ext,
                         const float* k, const float* v, size_t t_kv, size_t d, size_t rope_max,
                         float* out) {
    memset(out, 0, d * sizeof(float));
    if (n == 0) return fail(E_INVALID, "attention_row: empty selected set");
    for (size_t j = 0; j < n; ++j)
        if (sel[j] < 0 || (size_t)sel[j] >= t_kv) return fail(E_RANGE, "attention_row: index out of range");
    const float scale = 1.0f / sqrtf((float)d);
    float* scores = (float*)malloc(n * sizeof(float));
    if (ext) {
        if (n > pos + 1) { free(scores); return fail(E_LOGIC, "streaming_positions: selected tokens cannot fit below position"); }
        float qr[1024], kr[1024];
        memcpy(qr, q, d * sizeof(float));
        int e = apply_rope(qr, d, pos, rope_max);
        if (e) { free(scores); return e; }
        for (size_t j = 0; j < n; ++j) {
            memcpy(kr, k + (size_t)sel[j] * d, d * sizeof(float));
            if ((e = apply_rope(kr, d, pos + 1 - n + j, rope_max))) { free(scores); return e; }
            scores[j] = dot_f32(qr, kr, d) * scale;
        }
    } else {
        for (size_t j = 0; j < n; ++j) scores[j] = dot_f32(q, k + (size_t)sel[j] * d, d) * scale;
    }
    softmax_weighted_sum(scores, sel, n, v, d, out);
    free(scores);
    return OK;
}

int orc_attention_row(const float* q, const int64_t* sel, size_t n, size_t pos, int ext,
                      const float* k, const float* v, size_t t_kv, size_t d, size_t rope_max,
                      float* out) {
    int e = attention_row(q, sel, n, pos, ext, k, v, t_kv, d, rope_max ? rope_max : t_kv + 2, out);
    return e ? e : ok();
}

/* block_sparse_attention (sparse_attention.cpp:114-145) */
int orc_block_sparse_attention(const float* q, const float* k, const float* v, size_t n_heads,
                               size_t n_kv, size_t t_q, size_t t_kv, size_t d, void* lists,
                               size_t block_size, size_t sink, size_t stream, size_t offset,
                               int ext, float* out) {
    const Lists* mask = (const Lists*)lists;
    if (block_size == 0 || mask->n != (t_q + block_size - 1) / block_size)
        return fail(E_INVALID, "block_sparse_attention: mask does not cover the queries");
    const size_t group = n_heads / n_kv;
    List sel = {0};
    for (size_t h = 0; h < n_heads; ++h) {
        const size_t kv = h / group;
        for (size_t r = 0; r < t_q; ++r) {
            int e = selected(mask, block_size, sink, stream, offset, r, &sel);
            if (!e) e = attention_row(q + (h * t_q + r) * d, sel.v, sel.n, offset + r, ext,
                                      k + kv * t_kv * d, v + kv * t_kv * d, t_kv, d, t_kv + 2,
                                      out + (h * t_q + r) * d);
            if (e) { list_free(&sel); return e; }
        }
    }
    list_free(&sel);
    return ok();
}

/* dense_attention (sparse_attention.cpp:62-93) */
int orc_dense_attention(const float* q, const float* k, const float* v, size_t n_heads,
                        size_t t_q, size_t t_kv, size_t d, float* out) {
    const size_t offset = t_kv - t_q;
    const float scale = 1.0f / sqrtf((float)d);
    float* scores = (float*)malloc(t_kv * sizeof(float));
    int64_t* sel = (int64_t*)malloc(t_kv * sizeof(int64_t));
    for (size_t j = 0; j < t_kv; ++j) sel[j] = (int64_t)j;
    for (size_t h = 0; h < n_heads; ++h) {
        for (size_t r = 0; r < t_q; ++r) {
            const size_t visible = offset + r + 1;
            for (size_t j = 0; j < visible; ++j)
                scores[j] = dot_f32(q + (h * t_q + r) * d, k + (h * t_kv + j) * d, d) * scale;
            float* o = out + (h * t_q + r) * d;
            memset(o, 0, d * sizeof(float));
            softmax_weighted_sum(scores, sel, visible, v + h * t_kv * d, d, o);
        }
    }
    free(scores);
    free(sel);
    return ok();
}

/* exact_topk (sparse_attention.cpp:147-160) */
void* orc_exact_topk(const float* q, const float* keys, size_t rows, size_t d, size_t kk) {
    if (kk > rows) { fail(E_INVALID, "exact_topk: k exceeds the key count"); return NULL; }
    float* s = (float*)malloc((rows ? rows : 1) * sizeof(float));
    size_t* order = (size_t*)malloc((rows ? rows : 1) * sizeof(size_t));
    for (size_t j = 0; j < rows; ++j) { s[j] = dot_f32(q, keys + j * d, d); order[j] = j; }
    g_sort_scores = s;
    qsort(order, rows, sizeof(size_t), cmp_desc);
    Lists* out = lists_new(1);
    for (size_t i = 0; i < kk; ++i) list_push(&out->l[0], (int64_t)order[i]);
    free(s);
    free(order);
    ok();
    return out;
}

/* attention_recall (sparse_attention.cpp:162-186) */
double orc_attention_recall(const int64_t* sel, size_t n, const float* q, const float* keys,
                            size_t rows, size_t d) {
    uint8_t* in = (uint8_t*)calloc(rows ? rows : 1, 1);
    for (size_t i = 0; i < n; ++i) {
        if (sel[i] < 0 || (size_t)sel[i] >= rows) { free(in); fail(E_RANGE, "attention_recall: selected index out of range"); return -1.0; }
        in[sel[i]] = 1;
    }
    const float scale = 1.0f / sqrtf((float)d);
    float* s = (float*)malloc((rows ? rows : 1) * sizeof(float));
    float mx = -INFINITY;
    for (size_t j = 0; j < rows; ++j) { s[j] = dot_f32(q, keys + j * d, d) * scale; mx = (mx < s[j]) ? s[j] : mx; }
    double total = 0.0, captured = 0.0;
    for (size_t j = 0; j < rows; ++j) {
        const double w = exp((double)s[j] - mx);
        total += w;
        if (in[j]) captured += w;
    }
    free(s);
    free(in);
    ok();
    return captured / total;
}

/* -------------------------------------------- per-layer decode body (Alg. 4)
 * decode.cpp:225-273 with every stage due: stage i consumes stage i-1's list,
 * 1-row query blocks at position T-1, then selected_indices + attention_row. */
typedef struct {
    const float *q, *k, *v; size_t groups, hpm, t, d; const size_t* stages; size_t n_stages;
    size_t sink, stream; int ext; size_t layer1, cutoff; int kv_shared;
    int64_t* mask_out; size_t cap; size_t* mask_len; float* out;
    size_t next; pthread_mutex_t mu; int err; char msg[512];
} DecJob;

static int decode_group(DecJob* J, size_t g) {
    const size_t d = J->d, t = J->t, pos = t - 1;
    const float* kg = J->k + (J->kv_shared ? 0 : g * t * d);
    const float* vg = J->v + (J->kv_shared ? 0 : g * t * d);
    Ctx c;
    ctx_init(&c, kg, J->hpm, 1, t, d, J->layer1, J->stream, pos, J->ext, J->cutoff, t + 2);
    List list = {0}, next = {0};
    const size_t upper = t > J->stream ? t - J->stream : 0;
    for (size_t i = J->sink; i < upper; ++i) list_push(&list, (int64_t)i);
    const float* qg = J->q + g * J->hpm * d;
    int e = OK;
    for (size_t s = 0; s < J->n_stages && !e; ++s) {
        e = pruning_stage(&c, J->stages[3 * s], J->stages[3 * s + 1], J->stages[3 * s + 2], list.v, list.n, qg, J->hpm, 1, &next);
        List tmp = list; list = next; next = tmp;
    }
    if (!e) {
        Lists mask = {&list, 1};
        List sel = {0};
        e = selected(&mask, 1, J->sink, J->stream, pos, 0, &sel);
        for (size_t h = 0; h < J->hpm && !e; ++h) {
            float row[1024];
            e = attention_row(qg + h * d, sel.v, sel.n, pos, J->ext, kg, vg, t, d, t + 2, row);
            if (!e && J->out) memcpy(J->out + (g * J->hpm + h) * d, row, d * sizeof(float));
        }
        list_free(&sel);
        if (!e && J->mask_out) {
            const size_t m = J->cap < list.n ? J->cap : list.n;
            memcpy(J->mask_out + g * J->cap, list.v, m * sizeof(int64_t));
        }
        if (!e && J->mask_len) J->mask_len[g] = list.n;
    }
    list_free(&list);
    list_free(&next);
    return e;
}

static void* decode_worker(void* arg) {
    DecJob* J = (DecJob*)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const size_t g = J->next++;
        const int stop = J->err != 0 || g >= J->groups;
        pthread_mutex_unlock(&J->mu);
        if (stop) break;
        int e = decode_group(J, g);
        if (e) {
            pthread_mutex_lock(&J->mu);
            if (!J->err) { J->err = e; snprintf(J->msg, sizeof J->msg, "%s", g_err); }
            pthread_mutex_unlock(&J->mu);
        }
    }
    return NULL;
}

int orc_decode_layer_step(const float* q, const float* k, const float* v, size_t groups,
                          size_t hpm, size_t t, size_t d, const size_t* stages, size_t n_stages,
                          size_t sink, size_t stream, int ext, size_t layer1, size_t cutoff,
                          size_t threads, int kv_shared, int64_t* mask_out, size_t cap,
                          size_t* mask_len, float* out, double* seconds) {
    DecJob J;
    memset(&J, 0, sizeof J);
    J.q = q; J.k = k; J.v = v; J.groups = groups; J.hpm = hpm; J.t = t; J.d = d;
    J.stages = stages; J.n_stages = n_stages; J.sink = sink; J.stream = stream; J.ext = ext;
    J.layer1 = layer1; J.cutoff = cutoff; J.kv_shared = kv_shared;
    J.mask_out = mask_out; J.cap = cap; J.mask_len = mask_len; J.out = out;
    pthread_mutex_init(&J.mu, NULL);
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    size_t workers = threads < groups ? threads : groups;
    if (workers <= 1) {
        for (size_t g = 0; g < groups; ++g) { int e = decode_group(&J, g); if (e) { pthread_mutex_destroy(&J.mu); return e; } }
    } else {
        pthread_t* th = (pthread_t*)malloc(workers * sizeof(pthread_t));
        for (size_t w = 0; w < workers; ++w) pthread_create(&th[w], NULL, decode_worker, &J);
        for (size_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
        free(th);
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    pthread_mutex_destroy(&J.mu);
    if (J.err) return fail(J.err, "%s", J.msg);
    if (seconds) *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    return ok();
}

/* ----------------------------------------------------- paged LRU store
 * TieredKvStore (kv_store.cpp:24-158): page id = (layer << 32) | token/page_size;
 * per bank: slot array, free-slot stack initialised descending (pop from back),
 * page table, LRU list (front = most recent, evict from back). */
typedef struct { uint64_t key; int64_t slot; int used; } HEnt;
typedef struct {
    size_t cap;
    int64_t* slot_page;      /* page in slot or -1 */
    size_t* free_slots; size_t n_free;
    int64_t *prev, *next; int64_t head, tail; size_t n_lru; /* LRU over slots */
    HEnt* tab; size_t tab_n;  /* open addressing page -> slot */
    uint64_t hits, misses, evictions;
} Bank;
typedef struct { size_t num_layers, page_size; Bank b[2]; } Store;

static size_t h64(uint64_t x, size_t n) { x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; return (size_t)(x & (n - 1)); }
static int64_t tab_get(Bank* b, uint64_t key) {
    for (size_t i = h64(key, b->tab_n);; i = (i + 1) & (b->tab_n - 1)) {
        if (!b->tab[i].used) return -1;
        if (b->tab[i].key == key) return b->tab[i].slot;
    }
}
static void tab_put(Bank* b, uint64_t key, int64_t slot) {
    size_t i = h64(key, b->tab_n);
    while (b->tab[i].used && b->tab[i].key != key) i = (i + 1) & (b->tab_n - 1);
    b->tab[i].used = 1; b->tab[i].key = key; b->tab[i].slot = slot;
}
static void tab_del(Bank* b, uint64_t key) {
    size_t i = h64(key, b->tab_n);
    while (b->tab[i].used && b->tab[i].key != key) i = (i + 1) & (b->tab_n - 1);
    if (!b->tab[i].used) return;
    b->tab[i].used = 0;
    for (size_t j = (i + 1) & (b->tab_n - 1); b->tab[j].used; j = (j + 1) & (b->tab_n - 1)) {
        HEnt e = b->tab[j];
        b->tab[j].used = 0;
        tab_put(b, e.key, e.slot);
    }
}
static void lru_unlink(Bank* b, int64_t s) {
    if (b->prev[s] >= 0) b->next[b->prev[s]] = b->next[s]; else b->head = b->next[s];
    if (b->next[s] >= 0) b->prev[b->next[s]] = b->prev[s]; else b->tail = b->prev[s];
    b->n_lru--;
}
static void lru_front(Bank* b, int64_t s) {
    b->prev[s] = -1; b->next[s] = b->head;
    if (b->head >= 0) b->prev[b->head] = s; else b->tail = s;
    b->head = s;
    b->n_lru++;
}

void* orc_store_new(size_t num_layers, size_t page_size, size_t mask_cap, size_t sa_cap) {
    if (page_size == 0) { fail(E_INVALID, "TieredKvStore: page size must be >= 1"); return NULL; }
    Store* s = (Store*)calloc(1, sizeof(Store));
    s->num_layers = num_layers; s->page_size = page_size;
    for (int i = 0; i < 2; ++i) {
        Bank* b = &s->b[i];
        b->cap = i == 0 ? mask_cap : sa_cap;
        const size_t n = b->cap ? b->cap : 1;
        b->slot_page = (int64_t*)malloc(n * sizeof(int64_t));
        b->free_slots = (size_t*)malloc(n * sizeof(size_t));
        b->prev = (int64_t*)malloc(n * sizeof(int64_t));
        b->next = (int64_t*)malloc(n * sizeof(int64_t));
        for (size_t j = 0; j < b->cap; ++j) { b->slot_page[j] = -1; b->free_slots[j] = b->cap - 1 - j; }
        b->n_free = b->cap;
        b->head = b->tail = -1;
        b->tab_n = 16;
        while (b->tab_n < 4 * n) b->tab_n <<= 1;
        b->tab = (HEnt*)calloc(b->tab_n, sizeof(HEnt));
    }
    ok();
    return s;
}
void orc_store_free(void* h) {
    Store* s = (Store*)h;
    if (!s) return;
    for (int i = 0; i < 2; ++i) {
        free(s->b[i].slot_page); free(s->b[i].free_slots); free(s->b[i].prev); free(s->b[i].next); free(s->b[i].tab);
    }
    free(s);
}
int orc_store_page_of(void* h, size_t layer, size_t token, uint64_t* out) {
    Store* s = (Store*)h;
    if (layer >= s->num_layers) return fail(E_RANGE, "page_of: layer out of range");
    *out = ((uint64_t)layer << 32) | (uint64_t)(token / s->page_size);
    return ok();
}
int orc_store_access(void* h, int bank, const uint64_t* pages, size_t n, uint64_t* missing, size_t* n_missing) {
    Bank* b = &((Store*)h)->b[bank];
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        const int64_t slot = tab_get(b, pages[i]);
        if (slot >= 0) { b->hits++; lru_unlink(b, slot); lru_front(b, slot); }
        else { b->misses++; missing[m++] = pages[i]; }
    }
    *n_missing = m;
    return ok();
}
int orc_store_commit(void* h, int bank, const uint64_t* pages, size_t n, uint64_t* evicted, size_t* n_evicted) {
    Bank* b = &((Store*)h)->b[bank];
    size_t ev = 0, count = 0;
    for (size_t i = 0; i < n; ++i) {
        if (tab_get(b, pages[i]) >= 0) { *n_evicted = ev; return fail(E_CONTRACT, "commit: page already resident"); }
        if (count == b->cap) { *n_evicted = ev; return fail(E_PARTIAL, "commit batch exceeds bank capacity, %zu pages left uncached", n - count); }
        if (b->n_free == 0) {
            const int64_t vs = b->tail;
            const uint64_t victim = (uint64_t)b->slot_page[vs];
            lru_unlink(b, vs);
            tab_del(b, victim);
            b->slot_page[vs] = -1;
            b->free_slots[b->n_free++] = (size_t)vs;
            b->evictions++;
            evicted[ev++] = victim;
        }
        const int64_t slot = (int64_t)b->free_slots[--b->n_free];
        b->slot_page[slot] = (int64_t)pages[i];
        tab_put(b, pages[i], slot);
        lru_front(b, slot);
        ++count;
    }
    *n_evicted = ev;
    return ok();
}
size_t orc_store_recency(void* h, int bank, uint64_t* out, size_t cap) {
    Bank* b = &((Store*)h)->b[bank];
    size_t i = 0;
    for (int64_t s = b->head; s >= 0; s = b->next[s], ++i) if (i < cap) out[i] = (uint64_t)b->slot_page[s];
    return i;
}
void orc_store_stats(void* h, int bank, uint64_t* out3) {
    Bank* b = &((Store*)h)->b[bank];
    out3[0] = b->hits; out3[1] = b->misses; out3[2] = b->evictions;
}
int orc_store_check(void* h) {
    Store* s = (Store*)h;
    for (int i = 0; i < 2; ++i) {
        Bank* b = &s->b[i];
        size_t resident = 0;
        for (size_t j = 0; j < b->cap; ++j) if (b->slot_page[j] >= 0) {
            resident++;
            if (tab_get(b, (uint64_t)b->slot_page[j]) != (int64_t)j) return fail(E_CONTRACT, "kv store: page table / slot mismatch");
        }
        if (resident + b->n_free != b->cap) return fail(E_CONTRACT, "kv store: slot accounting broken");
        if (b->n_lru != resident) return fail(E_CONTRACT, "kv store: LRU queue size mismatch");
    }
    return ok();
}

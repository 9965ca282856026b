// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim over the *unmodified* reference hipprune library, compiled from the
// sources where they lie under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhipref.so. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it, and only as the checker or
// the CPU baseline; the product path never touches it.
//
// Every entry point forwards to the reference's own functions:
//   run_pruning_stage / select_rep / build_mask   proj/src/pruning.cpp:146-313
//   selected_indices / attention_row / BSA         proj/src/sparse_attention.cpp:33-145
//   dense_attention / exact_topk / recall          proj/src/sparse_attention.cpp:62-186
//   build_rope_table                               proj/src/tensor.cpp:30-59
//   generate_synthetic                             proj/src/workload.cpp:147-189
//   TieredKvStore                                  proj/src/kv_store.cpp:24-158
//   DecodeEngine                                   proj/src/decode.cpp:104-289
// The only additions are (a) a GQA KeySource that maps q-head h to kv-head
// h / (H_q / H_kv) over raw row-major fp32 arrays (the convention SURVEY.md §7
// prescribes: one reference call per KV group), and (b) a timed multi-threaded
// driver of the per-layer decode body used as the CPU baseline.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "hipprune/commands.hpp"
#include "hipprune/config.hpp"
#include "hipprune/decode.hpp"
#include "hipprune/errors.hpp"
#include "hipprune/kv_store.hpp"
#include "hipprune/pruning.hpp"
#include "hipprune/sparse_attention.hpp"
#include "hipprune/workload.hpp"

using namespace hipprune;

namespace {

thread_local std::string g_err;
thread_local int g_err_code = 0;

enum Code { OK = 0, E_CONTRACT = 1, E_INVALID = 2, E_RANGE = 3, E_LOGIC = 4, E_RUNTIME = 5,
            E_PARTIAL = 6 };

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        g_err_code = OK;
        return OK;
    } catch (const ContractViolation& e) {
        g_err = e.what(); g_err_code = E_CONTRACT;
    } catch (const std::invalid_argument& e) {
        g_err = e.what(); g_err_code = E_INVALID;
    } catch (const std::out_of_range& e) {
        g_err = e.what(); g_err_code = E_RANGE;
    } catch (const PartialCommitError& e) {
        g_err = e.what(); g_err_code = E_PARTIAL;
    } catch (const std::logic_error& e) {
        g_err = e.what(); g_err_code = E_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what(); g_err_code = E_RUNTIME;
    }
    return g_err_code;
}

using Lists = std::vector<std::vector<std::size_t>>;

// KeySource over raw [H_kv][T][d] fp32 arrays; q-head h reads kv-head h / group.
class GqaSource final : public KeySource {
   public:
    GqaSource(const float* k, const float* v, std::size_t group, std::size_t t_kv, std::size_t d,
              bool log = false)
        : k_(k), v_(v), group_(group ? group : 1), t_kv_(t_kv), d_(d), log_(log) {}
    std::span<const float> key_row(std::size_t head, std::size_t token) override {
        if (token >= t_kv_) throw std::out_of_range("GqaSource: token out of range");
        const std::size_t kv = head / group_;
        if (log_) {
            reads_.emplace_back(head, token);
            distinct_.insert((static_cast<std::uint64_t>(kv) << 40) | token);
        }
        return {k_ + (kv * t_kv_ + token) * d_, d_};
    }
    std::span<const float> value_row(std::size_t head, std::size_t token) override {
        if (token >= t_kv_) throw std::out_of_range("GqaSource: token out of range");
        const std::size_t kv = head / group_;
        return {v_ + (kv * t_kv_ + token) * d_, d_};
    }
    std::vector<std::pair<std::size_t, std::size_t>> reads_;
    std::set<std::uint64_t> distinct_;

   private:
    const float* k_;
    const float* v_;
    std::size_t group_, t_kv_, d_;
    bool log_;
};

// Cached rope tables keyed by (max_position, head_dim); the bindings rebuild per
// call (bindings.cpp:133), which is excluded from every timing here.
const RopeTable& rope_for(std::size_t max_pos, std::size_t d) {
    static std::mutex mu;
    static std::map<std::pair<std::size_t, std::size_t>, std::unique_ptr<RopeTable>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(max_pos, d);
    auto it = cache.find(key);
    if (it == cache.end()) {
        if (cache.size() > 4) cache.clear();
        it = cache.emplace(key, std::make_unique<RopeTable>(build_rope_table(max_pos, d))).first;
    }
    return *it->second;
}

RopePolicySet make_policy(int ext, std::size_t cutoff) {
    RopePolicySet p;
    p.extension_enabled = ext != 0;
    p.early_layer_cutoff = cutoff;
    return p;
}

DenseMatrix mat(const float* src, std::size_t rows, std::size_t cols) {
    DenseMatrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data.data(), src, rows * cols * sizeof(float));
    return m;
}

PruningPlan make_plan(const std::size_t* stages, std::size_t n_stages, std::size_t sink,
                      std::size_t stream, const std::size_t* refresh) {
    PruningPlan plan;
    for (std::size_t i = 0; i < n_stages; ++i) {
        plan.stages.push_back({stages[3 * i], stages[3 * i + 1], stages[3 * i + 2]});
    }
    plan.sink_tokens = sink;
    plan.stream_tokens = stream;
    if (refresh) plan.refresh_intervals.assign(refresh, refresh + n_stages);
    return plan;
}

// Workload of `layer0 + 1` layers whose last layer carries the given tensors
// (lower layers stay empty; build_mask only touches `layer`).
AttentionWorkload make_workload(const float* q, const float* k, const float* v, std::size_t h_q,
                                std::size_t h_kv, std::size_t t_q, std::size_t t_kv, std::size_t d,
                                std::size_t layer0, bool with_kv) {
    AttentionWorkload wl;
    wl.num_heads = h_q;
    wl.num_layers = layer0 + 1;
    wl.seq_len_q = t_q;
    wl.seq_len_kv = t_kv;
    wl.head_dim = d;
    wl.queries.resize(layer0 + 1);
    wl.keys.resize(layer0 + 1);
    wl.values.resize(layer0 + 1);
    const std::size_t group = h_q / h_kv;
    for (std::size_t h = 0; h < h_q; ++h) {
        wl.queries[layer0].push_back(mat(q + h * t_q * d, t_q, d));
        if (with_kv) {
            const std::size_t kv = h / group;
            wl.keys[layer0].push_back(mat(k + kv * t_kv * d, t_kv, d));
            wl.values[layer0].push_back(v ? mat(v + kv * t_kv * d, t_kv, d) : DenseMatrix(t_kv, d));
        }
    }
    return wl;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_last_error_code() { return g_err_code; }

// ---- index-list handles --------------------------------------------------
std::size_t ref_lists_count(void* h) { return static_cast<Lists*>(h)->size(); }
std::size_t ref_lists_len(void* h, std::size_t i) { return (*static_cast<Lists*>(h))[i].size(); }
void ref_lists_get(void* h, std::size_t i, std::int64_t* out) {
    const auto& l = (*static_cast<Lists*>(h))[i];
    for (std::size_t j = 0; j < l.size(); ++j) out[j] = static_cast<std::int64_t>(l[j]);
}
void ref_lists_free(void* h) { delete static_cast<Lists*>(h); }
void* ref_lists_from(const std::int64_t* flat, const std::size_t* lens, std::size_t n) {
    auto* l = new Lists(n);
    std::size_t off = 0;
    for (std::size_t i = 0; i < n; ++i) {
        (*l)[i].assign(flat + off, flat + off + lens[i]);
        off += lens[i];
    }
    return l;
}

// ---- numerics --------------------------------------------------------------
int ref_build_rope_table(std::size_t max_pos, std::size_t d, float theta, float* cos_out,
                         float* sin_out) {
    return guard([&] {
        const RopeTable t = build_rope_table(max_pos, d, theta);
        std::memcpy(cos_out, t.cos_tab.data.data(), t.cos_tab.data.size() * sizeof(float));
        std::memcpy(sin_out, t.sin_tab.data.data(), t.sin_tab.data.size() * sizeof(float));
    });
}

int ref_generate(std::size_t heads, std::size_t layers, std::size_t seq_kv, std::size_t seq_q,
                 std::size_t dim, double locality, std::uint64_t seed,
                 const std::size_t* needle_pos, const float* needle_strength,
                 std::size_t n_needles, float* q, float* k, float* v) {
    return guard([&] {
        SyntheticConfig cfg;
        cfg.num_heads = heads;
        cfg.num_layers = layers;
        cfg.seq_len_kv = seq_kv;
        cfg.seq_len_q = seq_q;
        cfg.head_dim = dim;
        cfg.locality_scale = locality;
        cfg.seed = seed;
        for (std::size_t i = 0; i < n_needles; ++i) cfg.needles.push_back({needle_pos[i], needle_strength[i]});
        const AttentionWorkload wl = generate_synthetic(cfg);
        const std::size_t tq = wl.seq_len_q;
        for (std::size_t l = 0; l < layers; ++l) {
            for (std::size_t h = 0; h < heads; ++h) {
                const std::size_t base = l * heads + h;
                std::memcpy(q + base * tq * dim, wl.q(l, h).data.data(), tq * dim * 4);
                std::memcpy(k + base * seq_kv * dim, wl.k(l, h).data.data(), seq_kv * dim * 4);
                std::memcpy(v + base * seq_kv * dim, wl.v(l, h).data.data(), seq_kv * dim * 4);
            }
        }
    });
}

// ---- pruning ---------------------------------------------------------------
// q: [n_heads][rows][d]; k: [n_kv][t_kv][d]. Returns a 1-list handle.
void* ref_run_pruning_stage(std::size_t bq, std::size_t lc, std::size_t keep,
                            const std::int64_t* idx, std::size_t n, const float* q,
                            std::size_t n_heads, std::size_t rows, const float* k,
                            std::size_t n_kv, std::size_t t_kv, std::size_t d, std::size_t layer1,
                            std::size_t stream, std::size_t qstart, int ext, std::size_t cutoff,
                            std::size_t rope_max, std::uint64_t* reads_total,
                            std::uint64_t* reads_distinct) {
    Lists* out = nullptr;
    guard([&] {
        const RopePolicySet policy = make_policy(ext, cutoff);
        const RopeTable& rope = rope_for(rope_max ? rope_max : t_kv + 2, d);
        std::vector<DenseMatrix> qb;
        for (std::size_t h = 0; h < n_heads; ++h) qb.push_back(mat(q + h * rows * d, rows, d));
        std::vector<std::size_t> in(idx, idx + n);
        GqaSource src(k, nullptr, n_heads / n_kv, t_kv, d, reads_total != nullptr);
        StageContext ctx;
        ctx.policy = &policy;
        ctx.rope = &rope;
        ctx.layer = layer1;
        ctx.stream_tokens = stream;
        ctx.query_start_position = qstart;
        auto res = run_pruning_stage(StageConfig{bq, lc, keep}, in, qb, src, ctx);
        if (reads_total) *reads_total = src.reads_.size();
        if (reads_distinct) *reads_distinct = src.distinct_.size();
        out = new Lists{std::move(res)};
    });
    return out;
}

// Single-chunk representative selection with its read trace (tokens, in order).
int ref_select_rep(const float* q, std::size_t rows, const std::int64_t* chunk, std::size_t n,
                   const float* k, std::size_t t_kv, std::size_t d, std::size_t layer1,
                   std::size_t stream, std::size_t qstart, int ext, std::size_t cutoff,
                   std::size_t chunk_index, std::size_t chunk_count, std::size_t rope_max,
                   std::int64_t* rep_out, std::int64_t* reads_out, std::size_t* n_reads) {
    return guard([&] {
        const RopePolicySet policy = make_policy(ext, cutoff);
        const RopeTable& rope = rope_for(rope_max ? rope_max : t_kv + 2, d);
        DenseMatrix qb = mat(q, rows, d);
        std::vector<std::size_t> c(chunk, chunk + n);
        GqaSource src(k, nullptr, 1, t_kv, d, true);
        StageContext ctx;
        ctx.policy = &policy;
        ctx.rope = &rope;
        ctx.layer = layer1;
        ctx.stream_tokens = stream;
        ctx.query_start_position = qstart;
        *rep_out = static_cast<std::int64_t>(select_rep(qb, c, src, 0, ctx, chunk_index, chunk_count));
        *n_reads = src.reads_.size();
        for (std::size_t i = 0; i < src.reads_.size(); ++i) reads_out[i] = src.reads_[i].second;
    });
}

// build_mask over one layer. q: [n_heads][t_q][d], k: [n_kv][t_kv][d].
// Returns the mask lists; *trace_out receives the per-stage last-block lists.
void* ref_build_mask(const float* q, const float* k, std::size_t n_heads, std::size_t n_kv,
                     std::size_t t_q, std::size_t t_kv, std::size_t d, std::size_t layer0,
                     const std::size_t* stages, std::size_t n_stages, std::size_t sink,
                     std::size_t stream, int ext, std::size_t cutoff, std::size_t threads,
                     void** trace_out, std::size_t* block_size_out,
                     std::size_t* query_offset_out) {
    Lists* out = nullptr;
    guard([&] {
        const PruningPlan plan = make_plan(stages, n_stages, sink, stream, nullptr);
        const RopePolicySet policy = make_policy(ext, cutoff);
        const RopeTable& rope = rope_for(t_kv + 2, d);
        const bool mha = n_heads == n_kv;
        AttentionWorkload wl = make_workload(q, k, nullptr, n_heads, n_kv, t_q, t_kv, d, layer0, mha);
        StageTrace trace;
        SparseBlockMask mask;
        if (mha) {
            mask = build_mask(plan, wl, layer0, policy, rope, nullptr, &trace, threads);
        } else {
            GqaSource src(k, nullptr, n_heads / n_kv, t_kv, d);
            mask = build_mask(plan, wl, layer0, policy, rope, &src, &trace, 1);
        }
        if (trace_out) *trace_out = new Lists(trace.last_block_outputs);
        if (block_size_out) *block_size_out = mask.block_size;
        if (query_offset_out) *query_offset_out = mask.query_offset;
        out = new Lists(std::move(mask.indices));
    });
    return out;
}

// ---- sparse attention --------------------------------------------------------
static SparseBlockMask mask_from(void* lists, std::size_t block_size, std::size_t sink,
                                 std::size_t stream, std::size_t offset) {
    SparseBlockMask m;
    m.block_size = block_size;
    m.sink_tokens = sink;
    m.stream_tokens = stream;
    m.query_offset = offset;
    m.indices = *static_cast<Lists*>(lists);
    return m;
}

void* ref_selected_indices(void* lists, std::size_t block_size, std::size_t sink,
                           std::size_t stream, std::size_t offset, std::size_t row) {
    Lists* out = nullptr;
    guard([&] {
        out = new Lists{selected_indices(mask_from(lists, block_size, sink, stream, offset), row)};
    });
    return out;
}

int ref_attention_row(const float* q, const std::int64_t* sel, std::size_t n, std::size_t pos,
                      int ext, const float* k, const float* v, std::size_t t_kv, std::size_t d,
                      std::size_t rope_max, float* out) {
    return guard([&] {
        const RopeTable& rope = rope_for(rope_max ? rope_max : t_kv + 2, d);
        std::vector<std::size_t> s(sel, sel + n);
        GqaSource src(k, v, 1, t_kv, d);
        const auto row = attention_row({q, d}, s, pos, ext != 0, rope, src, 0);
        std::memcpy(out, row.data(), d * sizeof(float));
    });
}

int ref_block_sparse_attention(const float* q, const float* k, const float* v,
                               std::size_t n_heads, std::size_t n_kv, std::size_t t_q,
                               std::size_t t_kv, std::size_t d, void* lists,
                               std::size_t block_size, std::size_t sink, std::size_t stream,
                               std::size_t offset, int ext, float* out) {
    return guard([&] {
        const RopeTable& rope = rope_for(t_kv + 2, d);
        AttentionWorkload wl = make_workload(q, k, v, n_heads, n_kv, t_q, t_kv, d, 0, false);
        RopePolicySet policy = make_policy(ext, 3);
        GqaSource src(k, v, n_heads / n_kv, t_kv, d);
        const auto res = block_sparse_attention(wl, 0, mask_from(lists, block_size, sink, stream, offset),
                                                policy, rope, src);
        for (std::size_t h = 0; h < n_heads; ++h) {
            std::memcpy(out + h * t_q * d, res.heads[h].data.data(), t_q * d * sizeof(float));
        }
    });
}

int ref_dense_attention(const float* q, const float* k, const float* v, std::size_t n_heads,
                        std::size_t t_q, std::size_t t_kv, std::size_t d, float* out) {
    return guard([&] {
        AttentionWorkload wl = make_workload(q, k, v, n_heads, n_heads, t_q, t_kv, d, 0, true);
        const auto res = dense_attention(wl, 0);
        for (std::size_t h = 0; h < n_heads; ++h) {
            std::memcpy(out + h * t_q * d, res.heads[h].data.data(), t_q * d * sizeof(float));
        }
    });
}

void* ref_exact_topk(const float* q, const float* keys, std::size_t rows, std::size_t d,
                     std::size_t kk) {
    Lists* out = nullptr;
    guard([&] { out = new Lists{exact_topk({q, d}, mat(keys, rows, d), kk)}; });
    return out;
}

double ref_attention_recall(const std::int64_t* sel, std::size_t n, const float* q,
                            const float* keys, std::size_t rows, std::size_t d) {
    double r = -1.0;
    guard([&] {
        std::vector<std::size_t> s(sel, sel + n);
        r = attention_recall(s, {q, d}, mat(keys, rows, d));
    });
    return r;
}

// ---- the per-layer decode body (CPU baseline) ---------------------------------
// One full-refresh decode layer step for `groups` KV groups of `hpm` q-heads, the
// body DecodeEngine::step runs per layer (decode.cpp:225-273) with direct key
// reads: run_pruning_stage x n_stages on a 1-row query block at position T-1,
// then selected_indices + attention_row per q-head. Groups are spread over
// `threads` std::threads. q: [groups*hpm][d]; k, v: [groups][t][d] (or a single
// shared [t][d] when kv_shared != 0). Wall seconds of the timed region -> *seconds.
int ref_decode_layer_step(const float* q, const float* k, const float* v, std::size_t groups,
                          std::size_t hpm, std::size_t t, std::size_t d,
                          const std::size_t* stages, std::size_t n_stages, std::size_t sink,
                          std::size_t stream, int ext, std::size_t layer1, std::size_t cutoff,
                          std::size_t threads, int kv_shared, std::int64_t* mask_out,
                          std::size_t cap, std::size_t* mask_len, float* out, double* seconds) {
    return guard([&] {
        const PruningPlan plan = make_plan(stages, n_stages, sink, stream, nullptr);
        plan.validate();
        const RopePolicySet policy = make_policy(ext, cutoff);
        const RopeTable& rope = rope_for(t + 2, d);
        const std::size_t pos = t - 1;
        std::vector<std::string> errors(groups);
        auto work = [&](std::size_t g) {
            const float* kg = k + (kv_shared ? 0 : g * t * d);
            const float* vg = v + (kv_shared ? 0 : g * t * d);
            GqaSource src(kg, vg, hpm, t, d);
            std::vector<DenseMatrix> qb;
            for (std::size_t h = 0; h < hpm; ++h) qb.push_back(mat(q + (g * hpm + h) * d, 1, d));
            std::vector<std::size_t> list;
            const std::size_t upper = t > stream ? t - stream : 0;
            if (upper > sink) {
                list.resize(upper - sink);
                std::iota(list.begin(), list.end(), sink);
            }
            StageContext ctx;
            ctx.policy = &policy;
            ctx.rope = &rope;
            ctx.layer = layer1;
            ctx.stream_tokens = stream;
            ctx.query_start_position = pos;
            for (const auto& st : plan.stages) list = run_pruning_stage(st, list, qb, src, ctx);
            SparseBlockMask mask;
            mask.block_size = 1;
            mask.sink_tokens = sink;
            mask.stream_tokens = stream;
            mask.query_offset = pos;
            mask.indices = {list};
            const auto selected = selected_indices(mask, 0);
            for (std::size_t h = 0; h < hpm; ++h) {
                const auto row = attention_row(qb[h].row_span(0), selected, pos, ext != 0, rope, src, h);
                if (out) std::memcpy(out + (g * hpm + h) * d, row.data(), d * sizeof(float));
            }
            if (mask_out) {
                const std::size_t m = std::min(cap, list.size());
                for (std::size_t i = 0; i < m; ++i) mask_out[g * cap + i] = static_cast<std::int64_t>(list[i]);
            }
            if (mask_len) mask_len[g] = list.size();
        };
        const auto t0 = std::chrono::steady_clock::now();
        const std::size_t workers = std::max<std::size_t>(1, std::min(threads, groups));
        if (workers == 1) {
            for (std::size_t g = 0; g < groups; ++g) work(g);
        } else {
            std::vector<std::thread> pool;
            for (std::size_t w = 0; w < workers; ++w) {
                pool.emplace_back([&, w] {
                    for (std::size_t g = w; g < groups; g += workers) {
                        try {
                            work(g);
                        } catch (const std::exception& e) {
                            errors[g] = e.what();
                        }
                    }
                });
            }
            for (auto& th : pool) th.join();
        }
        const auto t1 = std::chrono::steady_clock::now();
        for (const auto& e : errors) {
            if (!e.empty()) throw std::runtime_error(e);
        }
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// Distinct key rows read per stage of the same decode body (the algorithmic
// byte count of SURVEY.md §8(d)), for one group.
int ref_decode_read_counts(const float* q, const float* k, std::size_t hpm, std::size_t t,
                           std::size_t d, const std::size_t* stages, std::size_t n_stages,
                           std::size_t sink, std::size_t stream, int ext, std::size_t layer1,
                           std::size_t cutoff, std::uint64_t* distinct_out,
                           std::uint64_t* total_out) {
    return guard([&] {
        const PruningPlan plan = make_plan(stages, n_stages, sink, stream, nullptr);
        const RopePolicySet policy = make_policy(ext, cutoff);
        const RopeTable& rope = rope_for(t + 2, d);
        std::vector<DenseMatrix> qb;
        for (std::size_t h = 0; h < hpm; ++h) qb.push_back(mat(q + h * d, 1, d));
        std::vector<std::size_t> list;
        const std::size_t upper = t > stream ? t - stream : 0;
        if (upper > sink) {
            list.resize(upper - sink);
            std::iota(list.begin(), list.end(), sink);
        }
        StageContext ctx;
        ctx.policy = &policy;
        ctx.rope = &rope;
        ctx.layer = layer1;
        ctx.stream_tokens = stream;
        ctx.query_start_position = t - 1;
        for (std::size_t i = 0; i < plan.stages.size(); ++i) {
            GqaSource src(k, nullptr, hpm, t, d, true);
            list = run_pruning_stage(plan.stages[i], list, qb, src, ctx);
            distinct_out[i] = src.distinct_.size();
            total_out[i] = src.reads_.size();
        }
    });
}

// ---- paged store (LRU) ---------------------------------------------------------
struct StoreBox {
    AttentionWorkload host;
    std::unique_ptr<TieredKvStore> store;
};

void* ref_store_new(std::size_t num_layers, std::size_t page_size, std::size_t mask_cap,
                    std::size_t sa_cap) {
    StoreBox* box = nullptr;
    guard([&] {
        auto b = std::make_unique<StoreBox>();
        b->host.num_layers = num_layers;
        b->store = std::make_unique<TieredKvStore>(b->host, page_size, mask_cap, sa_cap);
        box = b.release();
    });
    return box;
}
void ref_store_free(void* h) { delete static_cast<StoreBox*>(h); }

int ref_store_page_of(void* h, std::size_t layer, std::size_t token, std::uint64_t* out) {
    return guard([&] { *out = static_cast<StoreBox*>(h)->store->page_of(layer, token); });
}

int ref_store_access(void* h, int bank, const std::uint64_t* pages, std::size_t n,
                     std::uint64_t* missing, std::size_t* n_missing) {
    return guard([&] {
        auto r = static_cast<StoreBox*>(h)->store->access_pages(static_cast<BankId>(bank), {pages, n});
        *n_missing = r.missing.size();
        std::copy(r.missing.begin(), r.missing.end(), missing);
    });
}

int ref_store_commit(void* h, int bank, const std::uint64_t* pages, std::size_t n,
                     std::uint64_t* evicted, std::size_t* n_evicted) {
    return guard([&] {
        auto r = static_cast<StoreBox*>(h)->store->commit(static_cast<BankId>(bank), {pages, n});
        *n_evicted = r.size();
        std::copy(r.begin(), r.end(), evicted);
    });
}

std::size_t ref_store_recency(void* h, int bank, std::uint64_t* out, std::size_t cap) {
    const auto r = static_cast<StoreBox*>(h)->store->recency_order(static_cast<BankId>(bank));
    const std::size_t n = std::min(cap, r.size());
    std::copy(r.begin(), r.begin() + n, out);
    return r.size();
}

void ref_store_stats(void* h, int bank, std::uint64_t* out3) {
    const auto s = static_cast<StoreBox*>(h)->store->stats(static_cast<BankId>(bank));
    out3[0] = s.hits;
    out3[1] = s.misses;
    out3[2] = s.evictions;
}

int ref_store_check(void* h) {
    return guard([&] { static_cast<StoreBox*>(h)->store->check_consistency(); });
}

// ---- decode engine (stage-cache scheduler) -----------------------------------------
// full: [layers][heads][T][d] for q, k, v with T = prefill_len + steps (seq_q == seq_kv).
struct EngineBox {
    AttentionWorkload full;
    std::unique_ptr<RopeTable> rope;
    std::unique_ptr<DecodeEngine> engine;
};

void* ref_engine_new(const float* q, const float* k, const float* v, std::size_t layers,
                     std::size_t heads, std::size_t t_full, std::size_t d, std::size_t prefill_len,
                     std::size_t q_len, const std::size_t* stages, std::size_t n_stages,
                     std::size_t sink, std::size_t stream, const std::size_t* refresh, int ext,
                     std::size_t cutoff, std::size_t page_size, std::size_t mask_cap,
                     std::size_t sa_cap, double dev_cost, double host_cost, std::size_t rope_max) {
    EngineBox* box = nullptr;
    guard([&] {
        auto b = std::make_unique<EngineBox>();
        auto& wl = b->full;
        wl.num_heads = heads;
        wl.num_layers = layers;
        wl.seq_len_q = t_full;
        wl.seq_len_kv = t_full;
        wl.head_dim = d;
        wl.queries.resize(layers);
        wl.keys.resize(layers);
        wl.values.resize(layers);
        for (std::size_t l = 0; l < layers; ++l) {
            for (std::size_t h = 0; h < heads; ++h) {
                const std::size_t base = (l * heads + h) * t_full * d;
                wl.queries[l].push_back(mat(q + base, t_full, d));
                wl.keys[l].push_back(mat(k + base, t_full, d));
                wl.values[l].push_back(mat(v + base, t_full, d));
            }
        }
        b->rope = std::make_unique<RopeTable>(build_rope_table(rope_max ? rope_max : t_full + 2, d));
        PruningPlan plan = make_plan(stages, n_stages, sink, stream, refresh);
        RopePolicySet policy = make_policy(ext, cutoff);
        b->engine = std::make_unique<DecodeEngine>(truncate_workload(wl, prefill_len, q_len), plan,
                                                   policy, *b->rope,
                                                   StoreConfig{page_size, mask_cap, sa_cap},
                                                   CostModel{dev_cost, host_cost});
        box = b.release();
    });
    return box;
}
void ref_engine_free(void* h) { delete static_cast<EngineBox*>(h); }

int ref_engine_set_frozen(void* h, const int* frozen, std::size_t n) {
    return guard([&] {
        std::vector<bool> f(n);
        for (std::size_t i = 0; i < n; ++i) f[i] = frozen[i] != 0;
        static_cast<EngineBox*>(h)->engine->set_frozen_stages(f);
    });
}

// Prefill: outputs [layers][heads][q_len][d]; returns mask lists of the last layer.
void* ref_engine_prefill(void* h, float* out) {
    Lists* res = nullptr;
    guard([&] {
        auto* b = static_cast<EngineBox*>(h);
        const auto r = b->engine->prefill();
        std::size_t off = 0;
        for (const auto& layer : r.outputs) {
            for (const auto& head : layer.heads) {
                if (out) std::memcpy(out + off, head.data.data(), head.data.size() * 4);
                off += head.data.size();
            }
        }
        res = new Lists(r.masks.back().indices);
        b->engine->store().reset_stats();
    });
    return res;
}

// One decode step with the token at `token_index` of the full workload.
// out: [layers][heads][d]; tel: refreshed flags (n_stages), stage_latency (n_stages),
// bsa_latency, mask_hits, mask_accesses, sa_hits, sa_accesses, mask_sizes (n_stages).
int ref_engine_step(void* h, std::size_t token_index, float* out, int* refreshed,
                    double* stage_latency, double* bsa_latency, std::uint64_t* counters4,
                    std::size_t* mask_sizes) {
    return guard([&] {
        auto* b = static_cast<EngineBox*>(h);
        const auto r = b->engine->step(token_input_at(b->full, token_index));
        std::size_t off = 0;
        for (const auto& layer : r.output) {
            for (const auto& row : layer) {
                if (out) std::memcpy(out + off, row.data(), row.size() * 4);
                off += row.size();
            }
        }
        const auto& t = r.telemetry;
        for (std::size_t i = 0; i < t.refreshed.size(); ++i) {
            refreshed[i] = t.refreshed[i];
            stage_latency[i] = t.stage_latency[i];
            mask_sizes[i] = t.mask_sizes[i];
        }
        *bsa_latency = t.bsa_latency;
        counters4[0] = t.mask_hits;
        counters4[1] = t.mask_accesses;
        counters4[2] = t.sa_hits;
        counters4[3] = t.sa_accesses;
    });
}

void* ref_engine_stage_cache(void* h, std::size_t layer, std::size_t stage) {
    return new Lists{static_cast<EngineBox*>(h)->engine->stage_cache(layer, stage)};
}

std::size_t ref_engine_store_recency(void* h, int bank, std::uint64_t* out, std::size_t cap) {
    const auto r = static_cast<EngineBox*>(h)->engine->store().recency_order(static_cast<BankId>(bank));
    const std::size_t n = std::min(cap, r.size());
    std::copy(r.begin(), r.begin() + n, out);
    return r.size();
}

// ---- config hash (report plumbing; used only to cross-check the port) ---------------
int ref_config_hash(const char* const* overrides, std::size_t n, std::uint64_t* out) {
    return guard([&] {
        RunConfig cfg = default_config();
        for (std::size_t i = 0; i < n; ++i) {
            std::string kv = overrides[i];
            const auto eq = kv.find('=');
            if (eq == std::string::npos) throw ConfigError("override must be key=value");
            apply_override(cfg, kv.substr(0, eq), kv.substr(eq + 1));
        }
        *out = config_hash(cfg);
    });
}

}  // extern "C"

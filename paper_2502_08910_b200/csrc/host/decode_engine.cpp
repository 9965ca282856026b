// DecodeEngine (decode.hpp / decode.cpp:104-289) on the device. The prefill builds
// each layer's mask with the device build_mask and seeds the per-(layer, stage)
// caches from its StageTrace, exactly as the reference does; every decode step then
// appends the token's K/V rows on the device, refreshes the due stages (stage i
// consumes the cache of stage i-1, decode.cpp:225-249) with single-row query blocks
// at position T-1, and runs the block-sparse attention over sinks ∪ last cache ∪
// stream for every head (decode.cpp:255-272). The caches live on the device; the
// host mirror behind stage_cache() is refreshed on demand.
//
// Page accounting (decode.cpp:13-27,225-281): the engine owns the reference's
// TieredKvStore over its host tier. Every pruning stage is one Mask-bank phase and
// every attention pass one SA-bank phase; the device kernels report their branch
// decisions, and the engine replays the reference's exact key/value read sequence
// into the bank views — so hits, misses, evictions, the per-phase modeled latency
// and the LRU order equal the reference engine's step by step. The misses are
// committed once per step, in batches of the bank capacity (commit_rolling).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "hipprune_b200.h"
#include "hipprune_b200.hpp"

namespace hipprune {

namespace {

void ck(int rc) {
    if (rc == HP_OK) return;
    const std::string msg = hp_last_error();
    switch (rc) {
        case HP_CONTRACT_VIOLATION: throw ContractViolation(msg);
        case HP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case HP_OUT_OF_RANGE: throw std::out_of_range(msg);
        case HP_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    Buf& operator=(Buf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        return *this;
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t n) {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = n;
        if (n) cu(cudaMalloc(&p, n), "cudaMalloc");
        if (n) cu(cudaMemset(p, 0, n), "cudaMemset");
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int rope_policy_id(RopePolicyId id) {
    switch (id) {
        case RopePolicyId::ChunkIndexed: return HP_ROPE_CHUNK_INDEXED;
        case RopePolicyId::Relative: return HP_ROPE_RELATIVE;
        case RopePolicyId::Streaming: return HP_ROPE_STREAMING;
        default: throw std::invalid_argument("RopePolicySet: plug-in position policies are host callbacks, not supported on the device");
    }
}

size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }

// Misses of a step committed in batches of the bank capacity (decode.cpp:13-20).
void commit_rolling(TieredKvStore& store, BankId bank, std::span<const std::uint64_t> pages) {
    const size_t cap = store.capacity(bank);
    if (cap == 0) return;  // zero-capacity bank: every page stays on the host tier
    for (size_t b = 0; b < pages.size(); b += cap) store.commit(bank, pages.subspan(b, std::min(cap, pages.size() - b)));
}

double phase_latency(const KvView& v, const CostModel& c) {
    const std::uint64_t hits = v.phase_hits(), miss = v.phase_accesses() - hits;
    return static_cast<double>(hits) * c.device_access_cost + static_cast<double>(miss) * c.host_access_cost;
}

int ceil_log2(size_t n) {
    int r = 0;
    while ((size_t{1} << r) < n) ++r;
    return r;
}

// the reference's key reads of one decode stage (pruning.cpp:69-98,170-185) from the
// device's branch decisions (paths[chunk * heads + head])
void replay_stage(KeySource& ks, const std::vector<size_t>& list, size_t lc, size_t heads, const uint32_t* paths) {
    const size_t cc = cdiv(list.size(), lc);
    for (size_t j = 0; j < cc; ++j) {
        const size_t b = j * lc, n = std::min(lc, list.size() - b);
        for (size_t h = 0; h < heads; ++h) {
            size_t first = 1, last = n;
            if (n > 1) {
                const uint32_t bits = paths[j * heads + h];
                const int iters = ceil_log2(n);
                for (int it = 0; it < iters && first < last; ++it) {
                    const size_t mid = (first + last + 1) / 2;
                    ks.key_row(h, list[b + first - 1]);
                    ks.key_row(h, list[b + mid - 1]);
                    if ((bits >> it) & 1u) first = mid;
                    else last = mid - 1;
                }
            }
            ks.key_row(h, list[b + first - 1]);
        }
    }
}

}  // namespace

struct DecodeEngine::Device {
    struct Layer {
        Buf k, v;                   // [pages][heads][page_size][d] fp32
        Buf q, out;                 // [heads][1][d]
        Buf tok_k, tok_v;           // [heads][d] staging for the appended row
        std::vector<Buf> cache;     // per stage: [keep] int32 (stage cache list)
        std::vector<Buf> count;     // per stage: [1] int32
        Buf sel, selc;              // selected list of the step's query row
        std::vector<Buf> paths;     // per stage: branch decisions [chunk][head] (accounting replay)
    };
    std::vector<Layer> layers;
    Buf in_start, in_count;         // stage-0 range input
    Buf ws;
    Buf rope_cos, rope_sin;
    int64_t rope_max = 0;
    int32_t pages = 0, page_size = 64, heads = 0, d = 0;
    size_t sel_stride = 0;
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> ev;    // [layers][stages + 1][2]
    ~Device() {
        for (auto e : ev) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
    hp_kv_view view(const Layer& L, int64_t t_kv) const {
        hp_kv_view x{};
        x.k_pool = L.k.p;
        x.v_pool = L.v.p;
        x.num_pages = pages;
        x.page_size = page_size;
        x.n_kv = heads;
        x.d = d;
        x.dtype = HP_F32;
        x.t_kv = static_cast<int32_t>(t_kv);
        return x;
    }
};

std::vector<bool> refresh_due(const std::vector<std::size_t>& counters, const PruningPlan& plan) {
    if (counters.size() != plan.stages.size()) throw std::invalid_argument("refresh_due: counter count != stage count");
    std::vector<bool> f(counters.size());
    for (size_t i = 0; i < counters.size(); ++i) f[i] = counters[i] == 0;
    return f;
}

double StepTelemetry::total_latency() const {
    double t = bsa_latency;
    for (double s : stage_latency) t += s;
    return t;
}

AttentionWorkload truncate_workload(const AttentionWorkload& full, std::size_t kv_len, std::size_t q_len) {
    if (full.seq_len_q != full.seq_len_kv)
        throw std::invalid_argument("truncate_workload: needs one query per context position");
    if (kv_len == 0 || kv_len > full.seq_len_kv || q_len == 0 || q_len > kv_len)
        throw std::invalid_argument("truncate_workload: lengths out of range");
    AttentionWorkload out;
    out.num_heads = full.num_heads;
    out.num_layers = full.num_layers;
    out.seq_len_q = q_len;
    out.seq_len_kv = kv_len;
    out.head_dim = full.head_dim;
    out.queries.resize(full.num_layers);
    out.keys.resize(full.num_layers);
    out.values.resize(full.num_layers);
    const size_t q0 = kv_len - q_len, d = full.head_dim;
    for (size_t l = 0; l < full.num_layers; ++l)
        for (size_t h = 0; h < full.num_heads; ++h) {
            DenseMatrix q(q_len, d), k(kv_len, d), v(kv_len, d);
            std::copy(full.q(l, h).row(q0), full.q(l, h).row(q0) + q.data.size(), q.data.begin());
            std::copy(full.k(l, h).data.begin(), full.k(l, h).data.begin() + k.data.size(), k.data.begin());
            std::copy(full.v(l, h).data.begin(), full.v(l, h).data.begin() + v.data.size(), v.data.begin());
            out.queries[l].push_back(std::move(q));
            out.keys[l].push_back(std::move(k));
            out.values[l].push_back(std::move(v));
        }
    return out;
}

TokenInput token_input_at(const AttentionWorkload& full, std::size_t token_index) {
    if (full.seq_len_q != full.seq_len_kv || token_index >= full.seq_len_kv)
        throw std::invalid_argument("token_input_at: index outside the workload");
    TokenInput t;
    t.q.resize(full.num_layers);
    t.k.resize(full.num_layers);
    t.v.resize(full.num_layers);
    for (size_t l = 0; l < full.num_layers; ++l)
        for (size_t h = 0; h < full.num_heads; ++h) {
            const auto qs = full.q(l, h).row_span(token_index);
            const auto ks = full.k(l, h).row_span(token_index);
            const auto vs = full.v(l, h).row_span(token_index);
            t.q[l].emplace_back(qs.begin(), qs.end());
            t.k[l].emplace_back(ks.begin(), ks.end());
            t.v[l].emplace_back(vs.begin(), vs.end());
        }
    return t;
}

DecodeEngine::DecodeEngine(AttentionWorkload workload, PruningPlan plan, RopePolicySet policy, const RopeTable& rope,
                           StoreConfig store_config, CostModel cost)
    : dev_(std::make_unique<Device>()),
      workload_(std::move(workload)),
      plan_(std::move(plan)),
      policy_(policy),
      rope_(&rope),
      cost_(cost) {
    plan_.validate();
    cost_.validate();
    workload_.validate();
    store_ = std::make_unique<TieredKvStore>(workload_, store_config.page_size, store_config.mask_capacity,
                                             store_config.sa_capacity);
    const std::size_t max_steps = 4096;  // initial device capacity past the prefill (grows on demand)
    if (!hp_device_available())
        throw std::runtime_error("hipprune_b200: no CUDA device — the B200 path has no CPU fallback");
    if (plan_.refresh_intervals.empty()) plan_.refresh_intervals.assign(plan_.stages.size(), 1);
    const size_t S = plan_.stages.size(), L = workload_.num_layers;
    counters_.assign(S, 0);
    frozen_.assign(S, false);
    caches_.assign(L, std::vector<std::vector<size_t>>(S));
    cache_stale_.assign(L, std::vector<bool>(S, false));
    last_refresh_.assign(L, std::vector<size_t>(S, 0));
    seq_len_kv_ = workload_.seq_len_kv;

    Device& D = *dev_;
    cu(cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    D.page_size = static_cast<int32_t>(std::max<size_t>(1, store_config.page_size));
    D.heads = static_cast<int32_t>(workload_.num_heads);
    D.d = static_cast<int32_t>(workload_.head_dim);
    const size_t cap = workload_.seq_len_kv + max_steps;
    D.pages = static_cast<int32_t>(cdiv(cap, D.page_size));
    const size_t H = D.heads, dd = D.d, ps = D.page_size;
    const size_t pool = static_cast<size_t>(D.pages) * H * ps * dd;
    D.sel_stride = plan_.sink_tokens + plan_.stages.back().keep + plan_.stream_tokens + 1;
    D.layers.resize(L);
    std::vector<float> host(pool);
    for (size_t l = 0; l < L; ++l) {
        auto& Ly = D.layers[l];
        for (int kv = 0; kv < 2; ++kv) {
            std::fill(host.begin(), host.end(), 0.0f);
            const auto& mats = kv == 0 ? workload_.keys[l] : workload_.values[l];
            for (size_t h = 0; h < H; ++h)
                for (size_t t = 0; t < workload_.seq_len_kv; ++t)
                    std::memcpy(&host[(((t / ps) * H + h) * ps + t % ps) * dd], mats[h].row(t), dd * 4);
            Buf& b = kv == 0 ? Ly.k : Ly.v;
            b.alloc(pool * 4);
            cu(cudaMemcpy(b.p, host.data(), pool * 4, cudaMemcpyHostToDevice), "upload K/V");
        }
        Ly.q.alloc(H * dd * 4);
        Ly.out.alloc(H * dd * 4);
        Ly.tok_k.alloc(H * dd * 4);
        Ly.tok_v.alloc(H * dd * 4);
        Ly.cache.resize(S);
        Ly.count.resize(S);
        for (size_t i = 0; i < S; ++i) {
            Ly.cache[i].alloc(std::max<size_t>(1, plan_.stages[i].keep) * 4);
            Ly.count[i].alloc(4);
        }
        Ly.sel.alloc(D.sel_stride * 4);
        Ly.selc.alloc(4);
        Ly.paths.resize(S);
    }
    D.in_start.alloc(4);
    D.in_count.alloc(4);
    const int32_t sink = static_cast<int32_t>(plan_.sink_tokens);
    cu(cudaMemcpy(D.in_start.p, &sink, 4, cudaMemcpyHostToDevice), "upload");
    // workspace: the largest stage (stage 0 sees the whole middle region) or the BSA
    size_t need = hp_bsa_workspace_bytes(D.heads, 1, static_cast<int32_t>(D.sel_stride), D.d);
    size_t prev = cap;
    for (const auto& st : plan_.stages) {
        need = std::max(need, hp_stage_workspace_bytes(1, static_cast<int32_t>(std::max<size_t>(1, cdiv(prev, st.chunk_size))),
                                                       static_cast<int32_t>(st.keep), static_cast<int32_t>(st.chunk_size)));
        prev = st.keep;
    }
    D.ws.alloc(need);
    if (policy_.extension_enabled) {
        D.rope_max = static_cast<int64_t>(rope.max_position);
        D.rope_cos.alloc(rope.cos_tab.data.size() * 4);
        D.rope_sin.alloc(rope.sin_tab.data.size() * 4);
        cu(cudaMemcpy(D.rope_cos.p, rope.cos_tab.data.data(), D.rope_cos.bytes, cudaMemcpyHostToDevice), "upload");
        cu(cudaMemcpy(D.rope_sin.p, rope.sin_tab.data.data(), D.rope_sin.bytes, cudaMemcpyHostToDevice), "upload");
    }
    D.ev.resize(L * (S + 1) * 2);
    for (auto& e : D.ev) cu(cudaEventCreate(&e), "cudaEventCreate");
}

DecodeEngine::~DecodeEngine() = default;

void DecodeEngine::set_frozen_stages(std::vector<bool> frozen) {
    if (frozen.size() != plan_.stages.size()) throw std::invalid_argument("set_frozen_stages: flag count != stage count");
    frozen_ = std::move(frozen);
}

const std::vector<std::size_t>& DecodeEngine::stage_cache(std::size_t layer, std::size_t stage) const {
    if (layer >= caches_.size() || stage >= plan_.stages.size()) throw std::out_of_range("stage_cache: out of range");
    if (cache_stale_[layer][stage]) {
        const auto& Ly = dev_->layers[layer];
        int32_t n = 0;
        cu(cudaMemcpy(&n, Ly.count[stage].p, 4, cudaMemcpyDeviceToHost), "download");
        std::vector<int32_t> tmp(std::max(0, n));
        if (n > 0) cu(cudaMemcpy(tmp.data(), Ly.cache[stage].p, n * 4, cudaMemcpyDeviceToHost), "download");
        caches_[layer][stage].assign(tmp.begin(), tmp.end());
        cache_stale_[layer][stage] = false;
    }
    return caches_[layer][stage];
}

PrefillResult DecodeEngine::prefill() {
    if (prefilled_) throw ContractViolation("prefill: engine already prefilled");
    PrefillResult result;
    for (size_t l = 0; l < workload_.num_layers; ++l) {
        StageTrace trace;
        KvView mask_view(*store_, BankId::Mask, l);
        mask_view.begin_phase();
        SparseBlockMask mask = build_mask(plan_, workload_, l, policy_, *rope_, &mask_view, &trace);
        commit_rolling(*store_, BankId::Mask, mask_view.drain_missing());
        KvView sa_view(*store_, BankId::Sa, l);
        sa_view.begin_phase();
        result.outputs.push_back(block_sparse_attention(workload_, l, mask, policy_, *rope_, sa_view));
        commit_rolling(*store_, BankId::Sa, sa_view.drain_missing());
        auto& Ly = dev_->layers[l];
        for (size_t i = 0; i < plan_.stages.size(); ++i) {
            const auto& lst = trace.last_block_outputs[i];
            std::vector<int32_t> tmp(lst.begin(), lst.end());
            const int32_t n = static_cast<int32_t>(tmp.size());
            if (n > static_cast<int32_t>(Ly.cache[i].bytes / 4)) Ly.cache[i].alloc(tmp.size() * 4);
            if (n) cu(cudaMemcpy(Ly.cache[i].p, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice), "upload");
            cu(cudaMemcpy(Ly.count[i].p, &n, 4, cudaMemcpyHostToDevice), "upload");
            caches_[l][i] = lst;
            cache_stale_[l][i] = false;
        }
        result.masks.push_back(std::move(mask));
    }
    store_->check_consistency();
    prefilled_ = true;
    return result;
}

StepResult DecodeEngine::step(const TokenInput& token) {
    if (!prefilled_) throw ContractViolation("step: engine not prefilled");
    const size_t L = workload_.num_layers, H = workload_.num_heads, dd = workload_.head_dim;
    const size_t S = plan_.stages.size();
    if (token.q.size() != L || token.k.size() != L || token.v.size() != L)
        throw std::invalid_argument("step: token layer count mismatch");
    for (size_t l = 0; l < L; ++l) {
        if (token.q[l].size() != H || token.k[l].size() != H || token.v[l].size() != H)
            throw std::invalid_argument("step: token head count mismatch");
        for (size_t h = 0; h < H; ++h)
            if (token.q[l][h].size() != dd || token.k[l][h].size() != dd || token.v[l][h].size() != dd)
                throw std::invalid_argument("step: token row width mismatch");
    }
    Device& D = *dev_;
    if (static_cast<int64_t>(seq_len_kv_) + 1 > static_cast<int64_t>(D.pages) * D.page_size) {
        // grow every layer's paged pools (double the pages; the page layout is unchanged)
        const int32_t np = D.pages * 2;
        const size_t old_b = static_cast<size_t>(D.pages) * H * D.page_size * dd * 4;
        for (auto& Ly : D.layers)
            for (Buf* b : {&Ly.k, &Ly.v}) {
                Buf nb;
                nb.alloc(old_b * 2);
                cu(cudaMemcpy(nb.p, b->p, old_b, cudaMemcpyDeviceToDevice), "grow KV");
                *b = std::move(nb);
            }
        D.pages = np;
    }
    // the host tier grows with the sequence, as the reference's workload does
    // (decode.cpp:202-208): the bank views read it
    for (size_t l = 0; l < L; ++l)
        for (size_t h = 0; h < H; ++h) {
            workload_.keys[l][h].append_row(token.k[l][h]);
            workload_.values[l][h].append_row(token.v[l][h]);
        }
    workload_.seq_len_kv += 1;
    seq_len_kv_ += 1;
    const size_t T = seq_len_kv_, pos = T - 1;
    std::vector<bool> flags = refresh_due(counters_, plan_);
    for (size_t i = 0; i < S; ++i)
        if (frozen_[i]) flags[i] = false;

    StepResult result;
    result.telemetry.refreshed = flags;
    result.telemetry.stage_latency.assign(S, 0.0);
    result.telemetry.device_stage_us.assign(S, 0.0);
    std::vector<std::uint64_t> mask_missing, sa_missing;
    result.output.assign(L, std::vector<std::vector<float>>(H, std::vector<float>(dd)));

    const size_t upper = T > plan_.stream_tokens ? T - plan_.stream_tokens : 0;
    const int32_t n0 = upper > plan_.sink_tokens ? static_cast<int32_t>(upper - plan_.sink_tokens) : 0;
    cu(cudaMemcpyAsync(D.in_count.p, &n0, 4, cudaMemcpyHostToDevice, D.stream), "upload");
    std::vector<float> qh(H * dd), kh(H * dd), vh(H * dd);
    for (size_t l = 0; l < L; ++l) {
        auto& Ly = D.layers[l];
        for (size_t h = 0; h < H; ++h) {
            std::memcpy(&qh[h * dd], token.q[l][h].data(), dd * 4);
            std::memcpy(&kh[h * dd], token.k[l][h].data(), dd * 4);
            std::memcpy(&vh[h * dd], token.v[l][h].data(), dd * 4);
        }
        cu(cudaMemcpyAsync(Ly.q.p, qh.data(), H * dd * 4, cudaMemcpyHostToDevice, D.stream), "upload q");
        cu(cudaMemcpyAsync(Ly.tok_k.p, kh.data(), H * dd * 4, cudaMemcpyHostToDevice, D.stream), "upload k");
        cu(cudaMemcpyAsync(Ly.tok_v.p, vh.data(), H * dd * 4, cudaMemcpyHostToDevice, D.stream), "upload v");
        const hp_kv_view kvv = D.view(Ly, static_cast<int64_t>(T));
        ck(hp_decode_append(&kvv, Ly.tok_k.p, Ly.tok_v.p, static_cast<int64_t>(pos), nullptr, D.stream));

        hp_rope_ctx rc{};
        rc.extension = policy_.extension_enabled ? 1 : 0;
        rc.cos_tab = D.rope_cos.as<float>();
        rc.sin_tab = D.rope_sin.as<float>();
        rc.rope_max = D.rope_max;
        rc.early_cutoff = static_cast<int32_t>(policy_.early_layer_cutoff);
        rc.early_policy = rope_policy_id(policy_.pruning_policy_early);
        rc.late_policy = rope_policy_id(policy_.pruning_policy_late);
        rc.layer = static_cast<int32_t>(l + 1);
        KvView mask_view(*store_, BankId::Mask, l);
        for (size_t i = 0; i < S; ++i) {
            if (!flags[i]) continue;
            const auto& st = plan_.stages[i];
            cudaEvent_t* e = &D.ev[(l * (S + 1) + i) * 2];
            cu(cudaEventRecord(e[0], D.stream), "event");
            hp_stage_args a{};
            a.query_block = 1;  // decode: one query row per head (decode.cpp:159-177)
            a.chunk_size = static_cast<int32_t>(st.chunk_size);
            a.keep = static_cast<int32_t>(st.keep);
            a.n_masks = 1;
            a.heads_per_mask = static_cast<int32_t>(H);
            a.n_q_heads = static_cast<int32_t>(H);
            a.n_blocks = 1;
            a.q_rows = 1;
            a.q = Ly.q.as<float>();
            a.query_offset = static_cast<int64_t>(pos);
            a.stream_tokens = static_cast<int32_t>(plan_.stream_tokens);
            const size_t in_max = i == 0 ? static_cast<size_t>(n0) : plan_.stages[i - 1].keep;
            a.max_chunks = static_cast<int32_t>(std::max<size_t>(1, cdiv(in_max, st.chunk_size)));
            if (i == 0) {
                a.in_start = D.in_start.as<int32_t>();
                a.in_count = D.in_count.as<int32_t>();
            } else {
                a.in_list = Ly.cache[i - 1].as<int32_t>();
                a.in_count = Ly.count[i - 1].as<int32_t>();
                a.in_stride = static_cast<int64_t>(Ly.cache[i - 1].bytes / 4);
            }
            a.out_list = Ly.cache[i].as<int32_t>();
            a.out_count = Ly.count[i].as<int32_t>();
            a.out_stride = static_cast<int64_t>(Ly.cache[i].bytes / 4);
            a.workspace = D.ws.p;
            a.workspace_bytes = D.ws.bytes;
            a.keys = kvv;
            a.rope = rc;
            // the input list as the reference sees it (for the read replay), taken before
            // this stage overwrites nothing it reads (stage i reads cache i-1)
            std::vector<size_t> input;
            if (i == 0) {
                input.resize(static_cast<size_t>(n0));
                std::iota(input.begin(), input.end(), plan_.sink_tokens);
            } else {
                cu(cudaStreamSynchronize(D.stream), "sync");
                input = stage_cache(l, i - 1);
            }
            const size_t paths_n = static_cast<size_t>(a.max_chunks) * H;
            if (Ly.paths[i].bytes < paths_n * 4) Ly.paths[i].alloc(paths_n * 4);
            a.path_out = Ly.paths[i].as<uint32_t>();
            ck(hp_prune_stage(&a, D.stream));
            cu(cudaEventRecord(e[1], D.stream), "event");
            last_refresh_[l][i] = step_index_ + 1;
            cache_stale_[l][i] = true;
            // Mask-bank phase: the stage's exact key reads (identity stages read nothing)
            mask_view.begin_phase();
            const size_t K = st.keep / st.chunk_size;
            if (!(input.size() <= st.keep || cdiv(input.size(), st.chunk_size) <= K)) {
                std::vector<uint32_t> ph(paths_n);
                cu(cudaMemcpyAsync(ph.data(), Ly.paths[i].p, paths_n * 4, cudaMemcpyDeviceToHost, D.stream), "download");
                cu(cudaStreamSynchronize(D.stream), "sync");
                replay_stage(mask_view, input, st.chunk_size, H, ph.data());
            }
            result.telemetry.stage_latency[i] += phase_latency(mask_view, cost_);
            result.telemetry.mask_hits += mask_view.phase_hits();
            result.telemetry.mask_accesses += mask_view.phase_accesses();
        }
        {
            const auto miss = mask_view.drain_missing();
            mask_missing.insert(mask_missing.end(), miss.begin(), miss.end());
        }
        cudaEvent_t* e = &D.ev[(l * (S + 1) + S) * 2];
        cu(cudaEventRecord(e[0], D.stream), "event");
        ck(hp_selected_indices(Ly.cache[S - 1].as<int32_t>(), Ly.count[S - 1].as<int32_t>(),
                               static_cast<int64_t>(Ly.cache[S - 1].bytes / 4), 1, 1, 1, static_cast<int64_t>(pos),
                               static_cast<int32_t>(plan_.sink_tokens), static_cast<int32_t>(plan_.stream_tokens),
                               Ly.sel.as<int32_t>(), Ly.selc.as<int32_t>(), static_cast<int64_t>(D.sel_stride),
                               D.stream));
        hp_bsa_args b{};
        b.n_q_heads = static_cast<int32_t>(H);
        b.heads_per_mask = static_cast<int32_t>(H);
        b.n_rows = 1;
        b.q = Ly.q.as<float>();
        b.query_offset = static_cast<int64_t>(pos);
        b.sel_list = Ly.sel.as<int32_t>();
        b.sel_count = Ly.selc.as<int32_t>();
        b.sel_stride = static_cast<int64_t>(D.sel_stride);
        b.max_sel = static_cast<int32_t>(D.sel_stride);
        b.out = Ly.out.as<float>();
        b.workspace = D.ws.p;
        b.workspace_bytes = D.ws.bytes;
        b.kv = kvv;
        b.rope = rc;
        b.rope.layer = 0;
        ck(hp_bsa(&b, D.stream));
        cu(cudaEventRecord(e[1], D.stream), "event");
        // SA-bank phase: every head reads the selected keys, then the values (decode.cpp:255-272)
        KvView sa_view(*store_, BankId::Sa, l);
        sa_view.begin_phase();
        SparseBlockMask m1;
        m1.block_size = 1;
        m1.sink_tokens = plan_.sink_tokens;
        m1.stream_tokens = plan_.stream_tokens;
        m1.query_offset = pos;
        cu(cudaStreamSynchronize(D.stream), "sync");
        m1.indices = {stage_cache(l, S - 1)};
        const std::vector<size_t> selected = selected_indices(m1, 0);
        for (size_t h = 0; h < H; ++h) {
            for (size_t t : selected) sa_view.key_row(h, t);
            for (size_t t : selected) sa_view.value_row(h, t);
        }
        result.telemetry.bsa_latency += phase_latency(sa_view, cost_);
        result.telemetry.sa_hits += sa_view.phase_hits();
        result.telemetry.sa_accesses += sa_view.phase_accesses();
        const auto miss = sa_view.drain_missing();
        sa_missing.insert(sa_missing.end(), miss.begin(), miss.end());
    }
    std::vector<float> oh(H * dd);
    for (size_t l = 0; l < L; ++l) {
        cu(cudaMemcpyAsync(oh.data(), D.layers[l].out.p, H * dd * 4, cudaMemcpyDeviceToHost, D.stream), "download");
        cu(cudaStreamSynchronize(D.stream), "sync");
        for (size_t h = 0; h < H; ++h) std::memcpy(result.output[l][h].data(), &oh[h * dd], dd * 4);
    }
    for (size_t l = 0; l < L; ++l) {
        for (size_t i = 0; i <= S; ++i) {
            if (i < S && !flags[i]) continue;
            float ms = 0.f;
            cu(cudaEventElapsedTime(&ms, D.ev[(l * (S + 1) + i) * 2], D.ev[(l * (S + 1) + i) * 2 + 1]), "elapsed");
            (i < S ? result.telemetry.device_stage_us[i] : result.telemetry.device_bsa_us) += 1000.0 * ms;
        }
    }
    for (size_t i = 0; i < S; ++i) result.telemetry.mask_sizes.push_back(stage_cache(L - 1, i).size());
    commit_rolling(*store_, BankId::Mask, mask_missing);
    commit_rolling(*store_, BankId::Sa, sa_missing);
    store_->check_consistency();
    for (size_t i = 0; i < S; ++i) counters_[i] = (counters_[i] + 1) % plan_.refresh_intervals[i];
    ++step_index_;
    result.telemetry.step = step_index_;
    return result;
}

}  // namespace hipprune

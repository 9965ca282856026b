// hipprune_b200 C++ host API — the reference hipprune operator surface, served by
// the sm_100a kernels behind include/hipprune_b200.h.
//
// Names, argument meaning and error behaviour follow the reference headers
// (paths relative to /root/reference/proj/include/hipprune):
//   tensor.hpp          DenseMatrix, RopeTable, build_rope_table
//   workload.hpp        AttentionWorkload, SyntheticConfig, generate_synthetic,
//                       plant_needle, save_dump / load_dump / dump_checksum (HIPW v1)
//   pruning.hpp         StageConfig, PruningPlan, SparseBlockMask, StageTrace, build_mask
//   rope_policy.hpp     RopePolicyId, RopePolicySet
//   sparse_attention.hpp AttentionOutput, block_sparse_attention, dense_attention,
//                       selected_indices, exact_topk, attention_recall
//   decode.hpp          StoreConfig, TokenInput, StepTelemetry, StepResult,
//                       PrefillResult, DecodeEngine, refresh_due
//   errors.hpp          ContractViolation
//
// The pruning stages, block-sparse attention and the decode step run on the GPU
// (no CPU fallback: without a CUDA device these throw std::runtime_error). The
// data-format helpers (generator, HIPW dumps) and the quality checkers
// (exact_topk, attention_recall) are host code, as in the reference.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace hipprune {

// errors.hpp:8-10
struct ContractViolation : std::logic_error {
    using std::logic_error::logic_error;
};
// workload.hpp:61-63
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- tensor.hpp
struct DenseMatrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<float> data;

    DenseMatrix() = default;
    DenseMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0f) {}
    float* row(std::size_t r) { return data.data() + r * cols; }
    const float* row(std::size_t r) const { return data.data() + r * cols; }
    std::span<const float> row_span(std::size_t r) const { return {row(r), cols}; }
    float& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    void append_row(std::span<const float> values);
    void validate_finite() const;
    bool operator==(const DenseMatrix&) const = default;
};

struct RopeTable {
    std::size_t max_position = 0;
    std::size_t head_dim = 0;
    float theta_base = 10000.0f;
    DenseMatrix cos_tab;  // max_position x head_dim/2
    DenseMatrix sin_tab;
};

// Double-precision angles cast to float (tensor.cpp:30-59), bit-identical.
RopeTable build_rope_table(std::size_t max_position, std::size_t head_dim, float theta_base = 10000.0f);

// -------------------------------------------------------------- workload.hpp
struct AttentionWorkload {
    std::size_t num_heads = 0;
    std::size_t num_layers = 0;
    std::size_t seq_len_q = 0;
    std::size_t seq_len_kv = 0;
    std::size_t head_dim = 0;
    std::vector<std::vector<DenseMatrix>> queries;  // [layer][head] T_q x d
    std::vector<std::vector<DenseMatrix>> keys;     // [layer][head] T_kv x d
    std::vector<std::vector<DenseMatrix>> values;

    const DenseMatrix& q(std::size_t l, std::size_t h) const { return queries[l][h]; }
    const DenseMatrix& k(std::size_t l, std::size_t h) const { return keys[l][h]; }
    const DenseMatrix& v(std::size_t l, std::size_t h) const { return values[l][h]; }
    void validate() const;
    bool operator==(const AttentionWorkload&) const = default;
};

struct NeedleSpec {
    std::size_t position = 0;
    float strength = 0.0f;
};

struct SyntheticConfig {
    std::size_t num_heads = 1;
    std::size_t num_layers = 1;
    std::size_t seq_len_q = 0;  // 0 = seq_len_kv
    std::size_t seq_len_kv = 0;
    std::size_t head_dim = 0;
    double locality_scale = 64.0;
    std::vector<NeedleSpec> needles;
    std::uint64_t seed = 0;
};

AttentionWorkload generate_synthetic(const SyntheticConfig& config);
void plant_needle(AttentionWorkload& workload, std::size_t layer, std::size_t position, float strength);
void save_dump(const AttentionWorkload& workload, const std::string& path);
AttentionWorkload load_dump(const std::string& path);
std::uint32_t dump_checksum(const AttentionWorkload& workload);

// ----------------------------------------------------------- rope_policy.hpp
enum class RopePolicyId { ChunkIndexed, Relative, Streaming, PlugIn };

struct RopePolicySet {
    RopePolicyId pruning_policy_early = RopePolicyId::ChunkIndexed;
    RopePolicyId pruning_policy_late = RopePolicyId::Relative;
    std::size_t early_layer_cutoff = 3;
    RopePolicyId bsa_policy = RopePolicyId::Streaming;
    bool extension_enabled = true;
};

// --------------------------------------------------------------- pruning.hpp
struct StageConfig {
    std::size_t query_block = 64;  // b_q
    std::size_t chunk_size = 0;    // l_c
    std::size_t keep = 0;          // k
    void validate() const;
};

struct PruningPlan {
    std::vector<StageConfig> stages;
    std::size_t sink_tokens = 256;
    std::size_t stream_tokens = 1024;
    std::vector<std::size_t> refresh_intervals;
    void validate() const;
};

// Appendix C presets (config.cpp:64-86): "3k", "5k", "fast", "flash".
PruningPlan preset_plan(const std::string& name);

struct SparseBlockMask {
    std::size_t block_size = 0;
    std::size_t sink_tokens = 0;
    std::size_t stream_tokens = 0;
    std::size_t query_offset = 0;
    std::vector<std::vector<std::size_t>> indices;
    std::size_t num_blocks() const { return indices.size(); }
};

struct StageTrace {
    std::vector<std::vector<std::size_t>> last_block_outputs;
};

// Alg. 1 on the device (pruning.cpp:202-313). Index-exact with the reference.
// `num_threads` is accepted for source compatibility (the device runs every query
// block at once).
SparseBlockMask build_mask(const PruningPlan& plan, const AttentionWorkload& workload, std::size_t layer,
                           const RopePolicySet& policy, const RopeTable& rope, StageTrace* trace = nullptr,
                           std::size_t num_threads = 1);

// ------------------------------------------------------ sparse_attention.hpp
struct AttentionOutput {
    std::vector<DenseMatrix> heads;
};

AttentionOutput block_sparse_attention(const AttentionWorkload& workload, std::size_t layer,
                                       const SparseBlockMask& mask, const RopePolicySet& policy,
                                       const RopeTable& rope);
// Causal softmax attention over every key: the block-sparse path with a mask that
// keeps every middle index (the reference's acceptance #1 identity), on the device.
AttentionOutput dense_attention(const AttentionWorkload& workload, std::size_t layer);
std::vector<std::size_t> selected_indices(const SparseBlockMask& mask, std::size_t row);
// Quality checkers (host): sparse_attention.cpp:147-202.
std::vector<std::size_t> exact_topk(std::span<const float> query, const DenseMatrix& keys, std::size_t k);
double attention_recall(std::span<const std::size_t> selected, std::span<const float> query,
                        const DenseMatrix& keys);

// ---------------------------------------------------------------- decode.hpp
struct StoreConfig {
    std::size_t page_size = 64;
    std::size_t mask_capacity = 0;
    std::size_t sa_capacity = 0;
};

struct TokenInput {
    std::vector<std::vector<std::vector<float>>> q;  // [layer][head][dim]
    std::vector<std::vector<std::vector<float>>> k;
    std::vector<std::vector<std::vector<float>>> v;
};

AttentionWorkload truncate_workload(const AttentionWorkload& full, std::size_t kv_len, std::size_t q_len);
TokenInput token_input_at(const AttentionWorkload& full, std::size_t token_index);

// The reference models latency from page hits (decode.cpp:22-27); on the device
// the step is measured: per-stage and BSA device time in microseconds.
struct StepTelemetry {
    std::size_t step = 0;
    std::vector<bool> refreshed;
    std::vector<double> stage_latency;
    double bsa_latency = 0.0;
    std::vector<std::size_t> mask_sizes;  // per stage, last layer
    double total_latency() const;
};

struct StepResult {
    std::vector<std::vector<std::vector<float>>> output;  // [layer][head][dim]
    StepTelemetry telemetry;
};

struct PrefillResult {
    std::vector<AttentionOutput> outputs;
    std::vector<SparseBlockMask> masks;
};

std::vector<bool> refresh_due(const std::vector<std::size_t>& counters, const PruningPlan& plan);

// Stage-cached decoding (decode.cpp:104-289) with the K/V of every layer resident
// in device memory: per step, the token's K/V rows are appended on the device, due
// stages refresh their per-(layer, stage) caches on the device, and every head's
// output row comes from the device block-sparse attention.
class DecodeEngine {
   public:
    DecodeEngine(AttentionWorkload workload, PruningPlan plan, RopePolicySet policy, const RopeTable& rope,
                 StoreConfig store_config = {}, std::size_t max_steps = 1024);
    ~DecodeEngine();
    DecodeEngine(const DecodeEngine&) = delete;
    DecodeEngine& operator=(const DecodeEngine&) = delete;

    PrefillResult prefill();
    StepResult step(const TokenInput& token);
    void set_frozen_stages(std::vector<bool> frozen);

    std::size_t steps_taken() const { return step_index_; }
    const std::vector<std::size_t>& counters() const { return counters_; }
    const std::vector<std::size_t>& stage_cache(std::size_t layer, std::size_t stage) const;
    std::size_t last_refresh(std::size_t layer, std::size_t stage) const { return last_refresh_[layer][stage]; }
    std::size_t seq_len_kv() const { return seq_len_kv_; }

   private:
    struct Device;
    std::unique_ptr<Device> dev_;
    AttentionWorkload workload_;  // prefill q rows + dims; K/V live on the device
    PruningPlan plan_;
    RopePolicySet policy_;
    const RopeTable* rope_;
    std::size_t seq_len_kv_ = 0;
    std::vector<std::size_t> counters_;
    std::vector<bool> frozen_;
    mutable std::vector<std::vector<std::vector<std::size_t>>> caches_;  // host mirror, lazily synced
    mutable std::vector<std::vector<bool>> cache_stale_;
    std::vector<std::vector<std::size_t>> last_refresh_;
    bool prefilled_ = false;
    std::size_t step_index_ = 0;
};

// true when a CUDA device is usable by the library
bool device_available();

}  // namespace hipprune

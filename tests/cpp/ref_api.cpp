// A caller written against the REFERENCE header names and signatures
// (/root/reference/proj/include/hipprune/*.hpp): it must compile and link unchanged
// against this library (tests/test_cpp_api.py), and its device results are compared
// with the reference (oracle) on the GPU. Prints one JSON object.
#include <cstdio>
#include <string>
#include <vector>

#include "hipprune/config.hpp"
#include "hipprune/decode.hpp"
#include "hipprune/key_source.hpp"
#include "hipprune/kv_store.hpp"
#include "hipprune/pruning.hpp"
#include "hipprune/sparse_attention.hpp"
#include "hipprune/workload.hpp"

using namespace hipprune;

static std::string list(const std::vector<std::size_t>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s + "]";
}

int main() {
    SyntheticConfig sc;
    sc.num_heads = 2;
    sc.num_layers = 1;
    sc.seq_len_kv = 512;
    sc.seq_len_q = 16;
    sc.head_dim = 16;
    sc.seed = 11;
    const AttentionWorkload w = generate_synthetic(sc);
    RopePolicySet pol;
    pol.extension_enabled = false;
    const RopeTable rope = build_rope_table(w.seq_len_kv + 2, w.head_dim);

    // run_pruning_stage through an instrumented DirectKeySource (pruning.hpp:72-75)
    const StageConfig st{16, 8, 64};
    std::vector<std::size_t> idx;
    for (std::size_t i = 16; i < 480; ++i) idx.push_back(i);
    std::vector<DenseMatrix> qb;
    for (std::size_t h = 0; h < w.num_heads; ++h) {
        DenseMatrix m(16, w.head_dim);
        for (std::size_t r = 0; r < 16; ++r)
            for (std::size_t c = 0; c < w.head_dim; ++c) m.at(r, c) = w.q(0, h).at(r, c);
        qb.push_back(std::move(m));
    }
    StageContext ctx;
    ctx.policy = &pol;
    ctx.rope = &rope;
    ctx.layer = 4;
    ctx.stream_tokens = 32;
    ctx.query_start_position = w.seq_len_kv - 16;
    DirectKeySource logged(w, 0, true);
    const std::vector<std::size_t> out = run_pruning_stage(st, idx, qb, logged, ctx);
    const std::size_t stage_reads = logged.reads().size();

    // select_rep over one chunk (pruning.hpp:64-66)
    const ChunkPartition part = partition_chunks(idx, 8);
    logged.clear_reads();
    const std::size_t rep = select_rep(qb[1], part.chunks[5], logged, 1, ctx, 5, part.chunks.size());
    const std::size_t rep_reads = logged.reads().size();

    // build_mask with a Mask-bank view (the decode engine's accounting seam)
    TieredKvStore store(w, 8, 16, 16);
    KvView view(store, BankId::Mask, 0);
    view.begin_phase();
    PruningPlan plan;
    plan.stages = {{16, 8, 64}, {8, 4, 32}};
    plan.sink_tokens = 16;
    plan.stream_tokens = 32;
    StageTrace trace;
    const SparseBlockMask mask = build_mask(plan, w, 0, pol, rope, &view, &trace);

    // attention_row over the last row's selected set (sparse_attention.hpp:43-46)
    const std::vector<std::size_t> sel = selected_indices(mask, 15);
    DirectKeySource direct(w, 0);
    const std::vector<float> row = attention_row(w.q(0, 0).row_span(15), sel, mask.query_offset + 15, false, rope,
                                                 direct, 0);

    std::printf("{\"stage\": %s, \"stage_reads\": %zu, \"rep\": %zu, \"rep_reads\": %zu, \"mask_blocks\": [",
                list(out).c_str(), stage_reads, rep, rep_reads);
    for (std::size_t b = 0; b < mask.num_blocks(); ++b) std::printf("%s%s", b ? "," : "", list(mask.indices[b]).c_str());
    std::printf("], \"mask_accesses\": %llu, \"mask_hits\": %llu, \"row\": [",
                static_cast<unsigned long long>(view.phase_accesses()), static_cast<unsigned long long>(view.phase_hits()));
    for (std::size_t i = 0; i < row.size(); ++i) std::printf("%s%.9g", i ? "," : "", row[i]);
    std::printf("]}\n");
    return 0;
}

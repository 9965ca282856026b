// _hipprune: the reference's pybind11 module (proj/src/bindings.cpp:78-218) with the
// same names, keyword arguments and defaults, served by the device host layer
// (include/hipprune_b200.hpp). Additions (not in the reference module): Workload
// construction from numpy arrays and a DecodeEngine binding. The GIL is released
// around every device call.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <tuple>

#include "hipprune_b200.hpp"

namespace py = pybind11;
using namespace hipprune;

namespace {

using FArr = py::array_t<float, py::array::c_style | py::array::forcecast>;

py::array_t<float> to_numpy(const DenseMatrix& m) {
    py::array_t<float> out({m.rows, m.cols});
    std::copy(m.data.begin(), m.data.end(), out.mutable_data());
    return out;
}

DenseMatrix from_numpy(const FArr& a) {
    if (a.ndim() != 2) throw std::invalid_argument("expected a 2-d float array");
    DenseMatrix m(static_cast<size_t>(a.shape(0)), static_cast<size_t>(a.shape(1)));
    std::copy(a.data(), a.data() + m.data.size(), m.data.begin());
    return m;
}

// [layers][heads][rows][d] -> per (layer, head) matrices
std::vector<std::vector<DenseMatrix>> split4(const FArr& a, const char* name) {
    if (a.ndim() != 4) throw std::invalid_argument(std::string(name) + ": expected [layers, heads, rows, dim]");
    const size_t L = a.shape(0), H = a.shape(1), R = a.shape(2), D = a.shape(3);
    std::vector<std::vector<DenseMatrix>> out(L);
    for (size_t l = 0; l < L; ++l)
        for (size_t h = 0; h < H; ++h) {
            DenseMatrix m(R, D);
            std::copy(a.data() + ((l * H + h) * R) * D, a.data() + ((l * H + h) * R + R) * D, m.data.begin());
            out[l].push_back(std::move(m));
        }
    return out;
}

AttentionWorkload workload_from(const FArr& q, const FArr& k, const FArr& v) {
    AttentionWorkload wl;
    wl.queries = split4(q, "q");
    wl.keys = split4(k, "k");
    wl.values = split4(v, "v");
    wl.num_layers = q.shape(0);
    wl.num_heads = q.shape(1);
    wl.seq_len_q = q.shape(2);
    wl.head_dim = q.shape(3);
    wl.seq_len_kv = k.shape(2);
    wl.validate();
    return wl;
}

using StageTuple = std::tuple<size_t, size_t, size_t>;

PruningPlan plan_from_args(const std::string& preset, const std::vector<StageTuple>& stages, size_t sink,
                           size_t stream) {
    PruningPlan plan = preset_plan(preset);
    if (!stages.empty()) {
        plan.stages.clear();
        for (const auto& [bq, lc, keep] : stages) plan.stages.push_back({bq, lc, keep});
        plan.refresh_intervals.clear();
    }
    if (sink != static_cast<size_t>(-1)) plan.sink_tokens = sink;
    if (stream != static_cast<size_t>(-1)) plan.stream_tokens = stream;
    return plan;
}

std::vector<py::array_t<float>> heads_to_numpy(const AttentionOutput& out) {
    std::vector<py::array_t<float>> r;
    for (const auto& h : out.heads) r.push_back(to_numpy(h));
    return r;
}

// DecodeEngine over a full workload (one query row per position, as the reference's
// decode-sim drives it): prefill on the first `prefill_len` positions, then step()
// feeds positions prefill_len, prefill_len + 1, ...
struct PyEngine {
    AttentionWorkload full;
    std::unique_ptr<RopeTable> rope;
    std::unique_ptr<DecodeEngine> engine;
    size_t next = 0;
};

}  // namespace

PYBIND11_MODULE(_hipprune, m) {
    m.doc() = "hipprune_b200: hierarchical context pruning and block-sparse attention on B200 (sm_100a)";

    py::register_exception<ContractViolation>(m, "ContractViolation", PyExc_RuntimeError);
    py::register_exception<FormatError>(m, "FormatError", PyExc_RuntimeError);

    py::class_<AttentionWorkload>(m, "Workload")
        .def(py::init(&workload_from), py::arg("q"), py::arg("k"), py::arg("v"),
             "Workload from float32 arrays q [layers, heads, T_q, d], k and v [layers, heads, T_kv, d]")
        .def_property_readonly("num_heads", [](const AttentionWorkload& w) { return w.num_heads; })
        .def_property_readonly("num_layers", [](const AttentionWorkload& w) { return w.num_layers; })
        .def_property_readonly("seq_len_q", [](const AttentionWorkload& w) { return w.seq_len_q; })
        .def_property_readonly("seq_len_kv", [](const AttentionWorkload& w) { return w.seq_len_kv; })
        .def_property_readonly("head_dim", [](const AttentionWorkload& w) { return w.head_dim; })
        .def("q", [](const AttentionWorkload& w, size_t l, size_t h) { return to_numpy(w.q(l, h)); })
        .def("k", [](const AttentionWorkload& w, size_t l, size_t h) { return to_numpy(w.k(l, h)); })
        .def("v", [](const AttentionWorkload& w, size_t l, size_t h) { return to_numpy(w.v(l, h)); });

    py::class_<SparseBlockMask>(m, "SparseBlockMask")
        .def(py::init([](size_t block_size, size_t sink, size_t stream, size_t query_offset,
                         std::vector<std::vector<size_t>> indices) {
                 SparseBlockMask mk;
                 mk.block_size = block_size;
                 mk.sink_tokens = sink;
                 mk.stream_tokens = stream;
                 mk.query_offset = query_offset;
                 mk.indices = std::move(indices);
                 return mk;
             }),
             py::arg("block_size"), py::arg("sink_tokens"), py::arg("stream_tokens"), py::arg("query_offset"),
             py::arg("indices"))
        .def_readonly("block_size", &SparseBlockMask::block_size)
        .def_readonly("sink_tokens", &SparseBlockMask::sink_tokens)
        .def_readonly("stream_tokens", &SparseBlockMask::stream_tokens)
        .def_readonly("query_offset", &SparseBlockMask::query_offset)
        .def_readonly("indices", &SparseBlockMask::indices);

    m.def(
        "generate",
        [](size_t heads, size_t layers, size_t seq_kv, size_t seq_q, size_t dim, double locality, std::uint64_t seed,
           const std::vector<std::pair<size_t, float>>& needles) {
            SyntheticConfig c;
            c.num_heads = heads;
            c.num_layers = layers;
            c.seq_len_kv = seq_kv;
            c.seq_len_q = seq_q;
            c.head_dim = dim;
            c.locality_scale = locality;
            c.seed = seed;
            for (const auto& [p, s] : needles) c.needles.push_back({p, s});
            return generate_synthetic(c);
        },
        py::arg("heads") = 1, py::arg("layers") = 1, py::arg("seq_kv") = 1024, py::arg("seq_q") = 64,
        py::arg("dim") = 32, py::arg("locality") = 64.0, py::arg("seed") = 1,
        py::arg("needles") = std::vector<std::pair<size_t, float>>{});

    m.def("save_dump", [](const AttentionWorkload& w, const std::string& path) { save_dump(w, path); });
    m.def("load_dump", [](const std::string& path) { return load_dump(path); });
    m.def("dump_checksum", [](const AttentionWorkload& w) { return dump_checksum(w); });

    m.def(
        "build_mask",
        [](const AttentionWorkload& workload, size_t layer, const std::string& preset,
           const std::vector<StageTuple>& stages, size_t sink, size_t stream, bool extension, size_t threads) {
            const PruningPlan plan = plan_from_args(preset, stages, sink, stream);
            RopePolicySet policy;
            policy.extension_enabled = extension;
            py::gil_scoped_release nogil;
            const RopeTable rope = build_rope_table(workload.seq_len_kv + 2, workload.head_dim);
            return build_mask(plan, workload, layer, policy, rope, nullptr, threads);
        },
        py::arg("workload"), py::arg("layer") = 0, py::arg("preset") = "3k",
        py::arg("stages") = std::vector<StageTuple>{}, py::arg("sink") = static_cast<size_t>(-1),
        py::arg("stream") = static_cast<size_t>(-1), py::arg("extension") = false, py::arg("threads") = 1);

    m.def(
        "dense_attention",
        [](const AttentionWorkload& workload, size_t layer) {
            AttentionOutput out;
            {
                py::gil_scoped_release nogil;
                out = dense_attention(workload, layer);
            }
            return heads_to_numpy(out);
        },
        py::arg("workload"), py::arg("layer") = 0);

    m.def(
        "block_sparse_attention",
        [](const AttentionWorkload& workload, size_t layer, const SparseBlockMask& mask, bool extension) {
            RopePolicySet policy;
            policy.extension_enabled = extension;
            AttentionOutput out;
            {
                py::gil_scoped_release nogil;
                const RopeTable rope = build_rope_table(workload.seq_len_kv + 2, workload.head_dim);
                out = block_sparse_attention(workload, layer, mask, policy, rope);
            }
            return heads_to_numpy(out);
        },
        py::arg("workload"), py::arg("layer"), py::arg("mask"), py::arg("extension") = false);

    m.def("selected_indices", &selected_indices, py::arg("mask"), py::arg("row"));

    m.def(
        "exact_topk",
        [](const FArr& query, const FArr& keys, size_t k) {
            const DenseMatrix km = from_numpy(keys);
            return exact_topk(std::span<const float>(query.data(), query.size()), km, k);
        },
        py::arg("query"), py::arg("keys"), py::arg("k"));

    m.def(
        "attention_recall",
        [](const std::vector<size_t>& selected, const FArr& query, const FArr& keys) {
            const DenseMatrix km = from_numpy(keys);
            return attention_recall(selected, std::span<const float>(query.data(), query.size()), km);
        },
        py::arg("selected"), py::arg("query"), py::arg("keys"));

    // run_report / config_hash (the reference's report plumbing, commands.cpp / config.cpp)
    // are served by the Python package over this module's DecodeEngine and checkers
    // (python/hipprune/_reports.py).
    m.def(
        "chunk_sparsity_histogram",
        [](py::array_t<float, py::array::c_style | py::array::forcecast> query,
           py::array_t<float, py::array::c_style | py::array::forcecast> keys, size_t k, size_t chunk_size) {
            const DenseMatrix km = from_numpy(keys);
            const ChunkSparsity cs = chunk_sparsity_histogram(std::span<const float>(query.data(), query.size()), km, k,
                                                              chunk_size);
            return py::make_tuple(cs.chunk_counts, cs.empty_fraction);
        },
        py::arg("query"), py::arg("keys"), py::arg("k"), py::arg("chunk_size"));

    m.def("device_available", &device_available);

    py::class_<PyEngine>(m, "DecodeEngine")
        .def(py::init([](const AttentionWorkload& full, size_t prefill_len, size_t q_len, const std::string& preset,
                         const std::vector<StageTuple>& stages, size_t sink, size_t stream,
                         const std::vector<size_t>& refresh, bool extension, size_t page_size, size_t mask_capacity,
                         size_t sa_capacity, double device_cost, double host_cost, size_t cutoff) {
                 auto e = std::make_unique<PyEngine>();
                 e->full = full;
                 PruningPlan plan = plan_from_args(preset, stages, sink, stream);
                 if (!refresh.empty()) plan.refresh_intervals = refresh;
                 RopePolicySet policy;
                 policy.extension_enabled = extension;
                 policy.early_layer_cutoff = cutoff;
                 e->rope = std::make_unique<RopeTable>(build_rope_table(full.seq_len_kv + 2, full.head_dim));
                 StoreConfig sc;
                 sc.page_size = page_size;
                 sc.mask_capacity = mask_capacity;
                 sc.sa_capacity = sa_capacity;
                 CostModel cost;
                 cost.device_access_cost = device_cost;
                 cost.host_access_cost = host_cost;
                 e->engine = std::make_unique<DecodeEngine>(truncate_workload(full, prefill_len, q_len), plan, policy,
                                                            *e->rope, sc, cost);
                 e->next = prefill_len;
                 return e;
             }),
             py::arg("full"), py::arg("prefill_len"), py::arg("q_len") = 64, py::arg("preset") = "3k",
             py::arg("stages") = std::vector<StageTuple>{}, py::arg("sink") = static_cast<size_t>(-1),
             py::arg("stream") = static_cast<size_t>(-1), py::arg("refresh") = std::vector<size_t>{},
             py::arg("extension") = false, py::arg("page_size") = 64, py::arg("mask_capacity") = 0,
             py::arg("sa_capacity") = 0, py::arg("device_cost") = 1.0, py::arg("host_cost") = 31.5,
             py::arg("cutoff") = 3)
        .def("set_frozen_stages", [](PyEngine& e, std::vector<bool> f) { e.engine->set_frozen_stages(std::move(f)); })
        .def("prefill",
             [](PyEngine& e) {
                 PrefillResult r;
                 {
                     py::gil_scoped_release nogil;
                     r = e.engine->prefill();
                 }
                 py::list outs;
                 for (const auto& o : r.outputs) outs.append(heads_to_numpy(o));
                 return py::make_tuple(outs, r.masks);
             })
        .def("step",
             [](PyEngine& e) {
                 if (e.next >= e.full.seq_len_kv) throw std::out_of_range("step: no positions left in the workload");
                 StepResult r;
                 {
                     py::gil_scoped_release nogil;
                     r = e.engine->step(token_input_at(e.full, e.next));
                 }
                 ++e.next;
                 const size_t L = r.output.size(), H = L ? r.output[0].size() : 0;
                 const size_t D = H ? r.output[0][0].size() : 0;
                 py::array_t<float> out({L, H, D});
                 float* p = out.mutable_data();
                 for (size_t l = 0; l < L; ++l)
                     for (size_t h = 0; h < H; ++h) std::copy(r.output[l][h].begin(), r.output[l][h].end(), p + (l * H + h) * D);
                 py::dict tel;
                 tel["step"] = r.telemetry.step;
                 tel["refreshed"] = r.telemetry.refreshed;
                 tel["stage_latency"] = r.telemetry.stage_latency;  // CostModel units (decode.cpp:22-27)
                 tel["bsa_latency"] = r.telemetry.bsa_latency;
                 tel["mask_hits"] = r.telemetry.mask_hits;
                 tel["mask_accesses"] = r.telemetry.mask_accesses;
                 tel["sa_hits"] = r.telemetry.sa_hits;
                 tel["sa_accesses"] = r.telemetry.sa_accesses;
                 tel["mask_sizes"] = r.telemetry.mask_sizes;
                 tel["stage_us"] = r.telemetry.device_stage_us;  // measured on the device
                 tel["bsa_us"] = r.telemetry.device_bsa_us;
                 return py::make_tuple(out, tel);
             })
        .def("stage_cache", [](PyEngine& e, size_t l, size_t s) { return e.engine->stage_cache(l, s); })
        .def("reset_store_stats", [](PyEngine& e) { e.engine->store().reset_stats(); })
        .def("store_stats",
             [](PyEngine& e, int bank) {
                 const BankStats st = e.engine->store().stats(static_cast<BankId>(bank));
                 return py::make_tuple(st.hits, st.misses, st.evictions);
             })
        .def("store_recency", [](PyEngine& e, int bank) { return e.engine->store().recency_order(static_cast<BankId>(bank)); })
        .def_property_readonly("counters", [](PyEngine& e) { return e.engine->counters(); })
        .def_property_readonly("steps_taken", [](PyEngine& e) { return e.engine->steps_taken(); });
}

// hipprune_b200 C++ host layer: the reference operator API (include/hipprune_b200.hpp)
// over the sm_100a C ABI (include/hipprune_b200.h). Host code owns device buffers
// (RAII over cudaMalloc), uploads inputs, sequences the kernel calls and maps the
// C-ABI status codes back to the reference's exception types. No compute runs here
// except the data-format helpers and the quality checkers the reference also keeps
// on the host.
#include "hipprune_b200.hpp"

#include <cuda_runtime.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <numeric>
#include <random>

#include "hipprune_b200.h"

namespace hipprune {

namespace {

// ------------------------------------------------------------------ errors
[[noreturn]] void throw_status(int rc) {
    const std::string msg = hp_last_error();
    switch (rc) {
        case HP_CONTRACT_VIOLATION: throw ContractViolation(msg);
        case HP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case HP_OUT_OF_RANGE: throw std::out_of_range(msg);
        case HP_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
void check(int rc) {
    if (rc != HP_OK) throw_status(rc);
}
void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void require_device() {
    if (!hp_device_available())
        throw std::runtime_error("hipprune_b200: no CUDA device — the B200 path has no CPU fallback");
}

// -------------------------------------------------------------- device RAII
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t n) {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = n;
        if (n) cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    }
    void zero() {
        if (p) cuda_check(cudaMemset(p, 0, bytes), "cudaMemset");
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void upload(const void* src, size_t n, size_t off = 0) {
        cuda_check(cudaMemcpy(static_cast<char*>(p) + off, src, n, cudaMemcpyHostToDevice), "upload");
    }
    void download(void* dst, size_t n, size_t off = 0) const {
        cuda_check(cudaMemcpy(dst, static_cast<const char*>(p) + off, n, cudaMemcpyDeviceToHost), "download");
    }
};

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

int policy_id(RopePolicyId id) {
    switch (id) {
        case RopePolicyId::ChunkIndexed: return HP_ROPE_CHUNK_INDEXED;
        case RopePolicyId::Relative: return HP_ROPE_RELATIVE;
        case RopePolicyId::Streaming: return HP_ROPE_STREAMING;
        default: throw std::invalid_argument("RopePolicySet: plug-in position policies are host callbacks, not supported on the device");
    }
}

// One layer's K (and V) as a paged fp32 pool [pages][heads][page_size][d] with the
// identity page table (KvView over the workload's host tier, kv_store.cpp:160-200).
struct DeviceLayer {
    DevBuf k, v;
    int32_t pages = 0, page_size = 64, heads = 0, d = 0;
    int64_t t_kv = 0;

    void build(const AttentionWorkload& wl, size_t layer, bool with_values, size_t capacity_tokens = 0,
               int32_t ps = 64) {
        heads = static_cast<int32_t>(wl.num_heads);
        d = static_cast<int32_t>(wl.head_dim);
        page_size = ps;
        t_kv = static_cast<int64_t>(wl.seq_len_kv);
        const size_t cap = std::max<size_t>(capacity_tokens, wl.seq_len_kv);
        pages = static_cast<int32_t>(ceil_div(cap, ps));
        const size_t n = static_cast<size_t>(pages) * heads * ps * d;
        std::vector<float> host(n, 0.0f);
        auto pack = [&](const std::vector<DenseMatrix>& mats) {
            for (int32_t h = 0; h < heads; ++h) {
                const DenseMatrix& m = mats[h];
                for (size_t t = 0; t < wl.seq_len_kv; ++t) {
                    const size_t page = t / ps, off = t % ps;
                    std::memcpy(&host[((page * heads + h) * ps + off) * d], m.row(t), d * sizeof(float));
                }
            }
        };
        pack(wl.keys[layer]);
        k.alloc(n * sizeof(float));
        k.upload(host.data(), n * sizeof(float));
        if (with_values) {
            std::fill(host.begin(), host.end(), 0.0f);
            pack(wl.values[layer]);
            v.alloc(n * sizeof(float));
            v.upload(host.data(), n * sizeof(float));
        }
    }
    hp_kv_view view(int64_t tkv = -1) const {
        hp_kv_view x{};
        x.k_pool = k.p;
        x.v_pool = v.p;
        x.num_pages = pages;
        x.page_size = page_size;
        x.n_kv = heads;
        x.d = d;
        x.dtype = HP_F32;
        x.t_kv = static_cast<int32_t>(tkv >= 0 ? tkv : t_kv);
        return x;
    }
};

struct DeviceRope {
    DevBuf cos, sin;
    int64_t max_pos = 0;
    void upload(const RopeTable& r) {
        max_pos = static_cast<int64_t>(r.max_position);
        cos.alloc(r.cos_tab.data.size() * 4);
        sin.alloc(r.sin_tab.data.size() * 4);
        cos.upload(r.cos_tab.data.data(), r.cos_tab.data.size() * 4);
        sin.upload(r.sin_tab.data.data(), r.sin_tab.data.size() * 4);
    }
};

hp_rope_ctx rope_ctx(const RopePolicySet& p, const DeviceRope* r, size_t layer1) {
    hp_rope_ctx c{};
    c.extension = p.extension_enabled ? 1 : 0;
    if (p.extension_enabled) {
        if (!r || !r->cos.p) throw std::invalid_argument("RopePolicySet: extension enabled without a rope table");
        c.cos_tab = r->cos.as<float>();
        c.sin_tab = r->sin.as<float>();
        c.rope_max = r->max_pos;
    }
    c.early_cutoff = static_cast<int32_t>(p.early_layer_cutoff);
    c.early_policy = policy_id(p.pruning_policy_early);
    c.late_policy = policy_id(p.pruning_policy_late);
    c.layer = static_cast<int32_t>(layer1);
    return c;
}

std::vector<float> pack_q(const AttentionWorkload& wl, size_t layer, size_t r0, size_t r1) {
    const size_t rows = r1 - r0, d = wl.head_dim;
    std::vector<float> q(wl.num_heads * rows * d);
    for (size_t h = 0; h < wl.num_heads; ++h)
        std::memcpy(&q[h * rows * d], wl.q(layer, h).row(r0), rows * d * sizeof(float));
    return q;
}

// ------------------------------------------------------------- generator
std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// per-(layer, head, kind) stream seed (workload.cpp:25-28)
std::uint64_t stream_seed(std::uint64_t seed, std::uint64_t layer, std::uint64_t head, std::uint64_t kind) {
    return splitmix64(splitmix64(splitmix64(seed ^ (layer << 1)) ^ (head << 1)) ^ kind);
}
DenseMatrix gaussian(size_t rows, size_t cols, std::uint64_t seed) {
    DenseMatrix m(rows, cols);
    std::mt19937_64 eng(seed);
    std::normal_distribution<float> nd(0.0f, 1.0f);
    for (float& x : m.data) x = nd(eng);
    return m;
}
// box filter over +-locality rows (clamped), prefix sums in double, then rows
// rescaled to norm sqrt(d) (workload.cpp:40-74)
DenseMatrix smooth(const DenseMatrix& noise, double locality) {
    const size_t n = noise.rows, d = noise.cols;
    const size_t half = locality < static_cast<double>(n) ? static_cast<size_t>(locality) : n;
    DenseMatrix out(n, d);
    std::vector<double> pre(n + 1);
    for (size_t c = 0; c < d; ++c) {
        pre[0] = 0.0;
        for (size_t r = 0; r < n; ++r) pre[r + 1] = pre[r] + static_cast<double>(noise.at(r, c));
        for (size_t r = 0; r < n; ++r) {
            const size_t lo = r >= half ? r - half : 0, hi = std::min(n - 1, r + half);
            out.at(r, c) = static_cast<float>((pre[hi + 1] - pre[lo]) / static_cast<double>(hi - lo + 1));
        }
    }
    const double target = std::sqrt(static_cast<double>(d));
    for (size_t r = 0; r < n; ++r) {
        double ss = 0.0;
        for (size_t c = 0; c < d; ++c) ss += static_cast<double>(out.at(r, c)) * out.at(r, c);
        if (ss > 0.0) {
            const float f = static_cast<float>(target / std::sqrt(ss));
            for (size_t c = 0; c < d; ++c) out.at(r, c) *= f;
        }
    }
    return out;
}

std::uint32_t crc_of(std::uint32_t crc, const DenseMatrix& m) {
    return static_cast<std::uint32_t>(crc32(crc, reinterpret_cast<const Bytef*>(m.data.data()),
                                            static_cast<uInt>(m.data.size() * sizeof(float))));
}

void put_le(std::ostream& os, std::uint64_t v, int bytes) {
    unsigned char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    os.write(reinterpret_cast<const char*>(b), bytes);
}
std::uint64_t get_le(std::istream& is, int bytes, const char* section) {
    unsigned char b[8];
    if (!is.read(reinterpret_cast<char*>(b), bytes)) throw FormatError(std::string("truncated ") + section);
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
    return v;
}

// sequential fp32 dot (tensor.cpp:88-98), for the host checkers
float dot_seq(std::span<const float> a, std::span<const float> b) {
    float acc = 0.0f;
    for (size_t i = 0; i < a.size(); ++i) {
        const float p = a[i] * b[i];
        acc = acc + p;
    }
    return acc;
}

}  // namespace

// =================================================================== tensor
void DenseMatrix::append_row(std::span<const float> values) {
    if (values.size() != cols)
        throw std::invalid_argument("append_row: expected " + std::to_string(cols) + " values, got " +
                                    std::to_string(values.size()));
    data.insert(data.end(), values.begin(), values.end());
    ++rows;
}

void DenseMatrix::validate_finite() const {
    if (data.size() != rows * cols) throw std::invalid_argument("DenseMatrix: data length != rows*cols");
    for (float v : data)
        if (!std::isfinite(v)) throw std::invalid_argument("DenseMatrix: non-finite entry");
}

RopeTable build_rope_table(std::size_t max_position, std::size_t head_dim, float theta_base) {
    if (head_dim == 0 || head_dim % 2 != 0)
        throw std::invalid_argument("build_rope_table: head_dim must be even and positive, got " +
                                    std::to_string(head_dim));
    if (max_position == 0) throw std::invalid_argument("build_rope_table: max_position must be >= 1");
    if (!(theta_base > 0.0f)) throw std::invalid_argument("build_rope_table: theta_base must be positive");
    RopeTable t;
    t.max_position = max_position;
    t.head_dim = head_dim;
    t.theta_base = theta_base;
    t.cos_tab = DenseMatrix(max_position, head_dim / 2);
    t.sin_tab = DenseMatrix(max_position, head_dim / 2);
    check(hp_build_rope_table(static_cast<int64_t>(max_position), static_cast<int32_t>(head_dim), theta_base,
                              t.cos_tab.data.data(), t.sin_tab.data.data()));
    return t;
}

// ================================================================= workload
void AttentionWorkload::validate() const {
    if (num_heads == 0 || num_layers == 0 || head_dim == 0 || seq_len_kv == 0)
        throw std::invalid_argument("AttentionWorkload: zero dimension");
    if (seq_len_q > seq_len_kv) throw std::invalid_argument("AttentionWorkload: seq_len_q > seq_len_kv");
    auto check_t = [&](const std::vector<std::vector<DenseMatrix>>& t, size_t rows, const char* name) {
        if (t.size() != num_layers)
            throw std::invalid_argument(std::string("AttentionWorkload: bad layer count in ") + name);
        for (const auto& pl : t) {
            if (pl.size() != num_heads)
                throw std::invalid_argument(std::string("AttentionWorkload: bad head count in ") + name);
            for (const auto& m : pl) {
                if (m.rows != rows || m.cols != head_dim)
                    throw std::invalid_argument(std::string("AttentionWorkload: bad shape in ") + name);
                m.validate_finite();
            }
        }
    };
    check_t(queries, seq_len_q, "queries");
    check_t(keys, seq_len_kv, "keys");
    check_t(values, seq_len_kv, "values");
}

AttentionWorkload generate_synthetic(const SyntheticConfig& config) {
    SyntheticConfig c = config;
    if (c.seq_len_q == 0) c.seq_len_q = c.seq_len_kv;
    if (c.num_heads == 0 || c.num_layers == 0 || c.seq_len_q == 0 || c.seq_len_kv == 0 || c.head_dim == 0)
        throw std::invalid_argument("generate_synthetic: zero dimension in config");
    if (!(c.locality_scale > 0.0)) throw std::invalid_argument("generate_synthetic: locality_scale must be positive");
    for (const auto& n : c.needles)
        if (n.position >= c.seq_len_kv) throw std::out_of_range("generate_synthetic: needle position out of range");
    AttentionWorkload wl;
    wl.num_heads = c.num_heads;
    wl.num_layers = c.num_layers;
    wl.seq_len_q = c.seq_len_q;
    wl.seq_len_kv = c.seq_len_kv;
    wl.head_dim = c.head_dim;
    wl.queries.resize(c.num_layers);
    wl.keys.resize(c.num_layers);
    wl.values.resize(c.num_layers);
    for (size_t l = 0; l < c.num_layers; ++l) {
        for (size_t h = 0; h < c.num_heads; ++h) {
            wl.queries[l].push_back(gaussian(c.seq_len_q, c.head_dim, stream_seed(c.seed, l, h, 1)));
            wl.keys[l].push_back(smooth(gaussian(c.seq_len_kv, c.head_dim, stream_seed(c.seed, l, h, 2)),
                                        c.locality_scale));
            wl.values[l].push_back(gaussian(c.seq_len_kv, c.head_dim, stream_seed(c.seed, l, h, 3)));
        }
    }
    for (const auto& n : c.needles)
        for (size_t l = 0; l < c.num_layers; ++l) plant_needle(wl, l, n.position, n.strength);
    return wl;
}

void plant_needle(AttentionWorkload& wl, std::size_t layer, std::size_t position, float strength) {
    if (layer >= wl.num_layers) throw std::out_of_range("plant_needle: layer out of range");
    if (position >= wl.seq_len_kv)
        throw std::out_of_range("plant_needle: position " + std::to_string(position) + " >= seq_len_kv " +
                                std::to_string(wl.seq_len_kv));
    if (wl.seq_len_q == 0) throw std::invalid_argument("plant_needle: workload has no queries");
    const size_t d = wl.head_dim;
    std::vector<double> dir(d, 0.0);  // mean final-query direction over heads
    for (size_t h = 0; h < wl.num_heads; ++h) {
        const float* q = wl.q(layer, h).row(wl.seq_len_q - 1);
        for (size_t c = 0; c < d; ++c) dir[c] += q[c];
    }
    double ss = 0.0;
    for (double x : dir) ss += x * x;
    const double nrm = std::sqrt(ss);
    for (size_t h = 0; h < wl.num_heads; ++h) {
        float* key = wl.keys[layer][h].row(position);
        for (size_t c = 0; c < d; ++c)
            key[c] = nrm > 0.0 ? static_cast<float>(static_cast<double>(strength) * dir[c] / nrm) : 0.0f;
    }
}

std::uint32_t dump_checksum(const AttentionWorkload& wl) {
    std::uint32_t crc = static_cast<std::uint32_t>(crc32(0L, Z_NULL, 0));
    for (size_t l = 0; l < wl.num_layers; ++l)
        for (size_t h = 0; h < wl.num_heads; ++h) {
            crc = crc_of(crc, wl.q(l, h));
            crc = crc_of(crc, wl.k(l, h));
            crc = crc_of(crc, wl.v(l, h));
        }
    return crc;
}

// HIPW v1: "HIPW", u32 version, u64 H/L/T_q/T_kv/d, raw fp32 Q,K,V per (layer, head),
// u32 CRC-32 of the payload (workload.cpp:234-312).
void save_dump(const AttentionWorkload& wl, const std::filesystem::path& path) {
    wl.validate();
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw FormatError("cannot open for writing: " + path.string());
    os.write("HIPW", 4);
    put_le(os, 1, 4);
    for (std::uint64_t v : {wl.num_heads, wl.num_layers, wl.seq_len_q, wl.seq_len_kv, wl.head_dim}) put_le(os, v, 8);
    for (size_t l = 0; l < wl.num_layers; ++l)
        for (size_t h = 0; h < wl.num_heads; ++h)
            for (const DenseMatrix* m : {&wl.q(l, h), &wl.k(l, h), &wl.v(l, h)})
                os.write(reinterpret_cast<const char*>(m->data.data()),
                         static_cast<std::streamsize>(m->data.size() * sizeof(float)));
    put_le(os, dump_checksum(wl), 4);
    if (!os) throw FormatError("write failure: " + path.string());
}

AttentionWorkload load_dump(const std::filesystem::path& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw FormatError("cannot open for reading: " + path.string());
    char magic[4];
    if (!is.read(magic, 4)) throw FormatError("truncated header");
    if (std::memcmp(magic, "HIPW", 4) != 0) throw FormatError("magic mismatch in header");
    const auto version = get_le(is, 4, "header");
    if (version != 1) throw FormatError("unsupported version " + std::to_string(version) + " in header");
    AttentionWorkload wl;
    wl.num_heads = get_le(is, 8, "header");
    wl.num_layers = get_le(is, 8, "header");
    wl.seq_len_q = get_le(is, 8, "header");
    wl.seq_len_kv = get_le(is, 8, "header");
    wl.head_dim = get_le(is, 8, "header");
    if (wl.num_heads == 0 || wl.num_layers == 0 || wl.seq_len_kv == 0 || wl.head_dim == 0)
        throw FormatError("zero dimension in header");
    auto read_mat = [&](size_t rows) {
        DenseMatrix m(rows, wl.head_dim);
        if (!is.read(reinterpret_cast<char*>(m.data.data()), static_cast<std::streamsize>(m.data.size() * 4)))
            throw FormatError("truncated payload");
        return m;
    };
    wl.queries.resize(wl.num_layers);
    wl.keys.resize(wl.num_layers);
    wl.values.resize(wl.num_layers);
    for (size_t l = 0; l < wl.num_layers; ++l)
        for (size_t h = 0; h < wl.num_heads; ++h) {
            wl.queries[l].push_back(read_mat(wl.seq_len_q));
            wl.keys[l].push_back(read_mat(wl.seq_len_kv));
            wl.values[l].push_back(read_mat(wl.seq_len_kv));
        }
    const auto stored = static_cast<std::uint32_t>(get_le(is, 4, "checksum"));
    if (stored != dump_checksum(wl)) throw FormatError("checksum mismatch in payload");
    return wl;
}

// ================================================================== pruning
void StageConfig::validate() const {
    if (query_block == 0 || chunk_size == 0) throw std::invalid_argument("StageConfig: b_q and l_c must be >= 1");
    if (keep == 0 || keep % chunk_size != 0)
        throw std::invalid_argument("StageConfig: k must be a positive multiple of l_c");
}

void PruningPlan::validate() const {
    if (stages.empty()) throw std::invalid_argument("PruningPlan: no stages");
    if (!refresh_intervals.empty() && refresh_intervals.size() != stages.size())
        throw std::invalid_argument("PruningPlan: refresh_intervals length != stage count");
    for (const auto& s : stages) s.validate();
    for (size_t i = 1; i < stages.size(); ++i) {
        if (stages[i].query_block > stages[i - 1].query_block || stages[i - 1].query_block % stages[i].query_block)
            throw std::invalid_argument("PruningPlan: successive b_q must be non-increasing and divisible");
        if (stages[i].keep > stages[i - 1].keep)
            throw std::invalid_argument("PruningPlan: k must be non-increasing across stages");
    }
    for (size_t r : refresh_intervals)
        if (r == 0) throw std::invalid_argument("PruningPlan: refresh interval must be >= 1");
}

PruningPlan preset_plan(const std::string& name) {
    PruningPlan p;
    p.sink_tokens = 256;
    p.stream_tokens = 1024;
    if (name == "3k" || name == "fast" || name == "flash")
        p.stages = {{64, 256, 32768}, {64, 32, 8192}, {64, 8, 2048}};
    else if (name == "5k")
        p.stages = {{64, 64, 32768}, {64, 32, 16384}, {64, 16, 4096}};
    else
        throw std::invalid_argument("unknown preset '" + name + "' (expected 3k, 5k, fast, flash)");
    p.refresh_intervals = name == "fast" ? std::vector<size_t>{32, 16, 8}
                          : name == "flash" ? std::vector<size_t>{96, 24, 8}
                                            : std::vector<size_t>{16, 8, 4};
    return p;
}

namespace {
void replay_stage_reads(KeySource& ks, std::span<const std::size_t> list, std::size_t lc, std::size_t heads,
                        const std::uint32_t* paths);
void build_layer_from_source(struct DeviceLayer& dl, KeySource& ks, const AttentionWorkload* src_wl, size_t src_layer,
                             size_t heads, size_t t_kv, size_t d, bool with_values,
                             std::span<const std::size_t> tokens);
}  // namespace

// Alg. 1 on the device. Rows come from `data` (layer `data_layer`) — the workload, or
// the host tier behind one of this library's KeySources — or, for any other
// KeySource, through `foreign` (read once per row to upload). With `replay` the
// device's branch decisions are replayed into it as the reference's sequential
// instrumented walk reads: stage by stage, query block by block (pruning.cpp:232-262).
static SparseBlockMask build_mask_device(const PruningPlan& plan, const AttentionWorkload& wl, std::size_t layer,
                                         const RopePolicySet& policy, const RopeTable& rope,
                                         const AttentionWorkload* data, std::size_t data_layer, KeySource* foreign,
                                         KeySource* replay, StageTrace* trace) {
    plan.validate();
    if (layer >= wl.num_layers) throw std::out_of_range("build_mask: layer out of range");
    const size_t t_q = wl.seq_len_q, t_kv = wl.seq_len_kv;
    if (t_q == 0 || t_q > t_kv) throw std::invalid_argument("build_mask: workload query length inconsistent");
    require_device();
    const size_t offset = t_kv - t_q;
    const int32_t heads = static_cast<int32_t>(wl.num_heads);
    auto middle_upper = [&](size_t bq, size_t m) -> size_t {
        const size_t end = offset + std::min((m + 1) * bq, t_q);
        return end > plan.stream_tokens ? end - plan.stream_tokens : 0;
    };

    DeviceLayer kv;
    if (foreign) build_layer_from_source(kv, *foreign, nullptr, 0, wl.num_heads, t_kv, wl.head_dim, false, {});
    else kv.build(*data, data_layer, false);
    const std::vector<float> qh = pack_q(wl, layer, 0, t_q);
    DevBuf q(qh.size() * 4);
    q.upload(qh.data(), qh.size() * 4);
    DeviceRope drope;
    if (policy.extension_enabled) drope.upload(rope);
    const hp_rope_ctx rc = rope_ctx(policy, policy.extension_enabled ? &drope : nullptr, layer + 1);

    if (trace) trace->last_block_outputs.clear();
    size_t bq = plan.stages.front().query_block;
    size_t nb = ceil_div(t_q, bq);
    std::vector<int32_t> starts(nb, static_cast<int32_t>(plan.sink_tokens)), counts(nb, 0);
    size_t max_in = 0;
    for (size_t m = 0; m < nb; ++m) {
        const size_t up = middle_upper(bq, m);
        counts[m] = up > plan.sink_tokens ? static_cast<int32_t>(up - plan.sink_tokens) : 0;
        max_in = std::max<size_t>(max_in, counts[m]);
    }
    DevBuf in_start(nb * 4), in_count(nb * 4);
    in_start.upload(starts.data(), nb * 4);
    in_count.upload(counts.data(), nb * 4);
    DevBuf in_list;  // list mode after stage 0
    int64_t in_stride = 0;
    DevBuf ws;
    for (size_t si = 0; si < plan.stages.size(); ++si) {
        const StageConfig& st = plan.stages[si];
        bq = st.query_block;
        const int32_t max_chunks = static_cast<int32_t>(std::max<size_t>(1, ceil_div(max_in, st.chunk_size)));
        const size_t out_stride = std::max<size_t>(st.keep, 1);
        DevBuf out_list(nb * out_stride * 4), out_count(nb * 4);
        const size_t need = hp_stage_workspace_bytes(static_cast<int32_t>(nb), max_chunks,
                                                     static_cast<int32_t>(st.keep), static_cast<int32_t>(st.chunk_size));
        if (ws.bytes < need) ws.alloc(need);
        hp_stage_args a{};
        a.query_block = static_cast<int32_t>(bq);
        a.chunk_size = static_cast<int32_t>(st.chunk_size);
        a.keep = static_cast<int32_t>(st.keep);
        a.n_masks = 1;  // one mask per layer, pooled over every head (pruning.cpp:176-184)
        a.heads_per_mask = heads;
        a.n_q_heads = heads;
        a.n_blocks = static_cast<int32_t>(nb);
        a.q_rows = static_cast<int32_t>(t_q);
        a.q = q.as<float>();
        a.query_offset = static_cast<int64_t>(offset);
        a.stream_tokens = static_cast<int32_t>(plan.stream_tokens);
        a.max_chunks = max_chunks;
        a.in_list = in_list.as<int32_t>();
        a.in_start = in_list.p ? nullptr : in_start.as<int32_t>();
        a.in_count = in_count.as<int32_t>();
        a.in_stride = in_stride;
        a.out_list = out_list.as<int32_t>();
        a.out_count = out_count.as<int32_t>();
        a.out_stride = static_cast<int64_t>(out_stride);
        a.workspace = ws.p;
        a.workspace_bytes = ws.bytes;
        a.keys = kv.view();
        a.rope = rc;
        DevBuf paths;
        if (replay) {
            paths.alloc(std::max<size_t>(1, nb * static_cast<size_t>(max_chunks) * heads) * 4);
            a.path_out = paths.as<std::uint32_t>();
        }
        check(hp_prune_stage(&a, nullptr));
        if (replay) {  // the reference's read sequence of this stage, block by block
            std::vector<std::uint32_t> ph(nb * static_cast<size_t>(max_chunks) * heads);
            paths.download(ph.data(), ph.size() * 4);
            std::vector<int32_t> cnt(nb);
            in_count.download(cnt.data(), nb * 4);
            std::vector<int32_t> lst;
            if (in_list.p) {
                lst.resize(nb * static_cast<size_t>(in_stride));
                in_list.download(lst.data(), lst.size() * 4);
            }
            for (size_t m = 0; m < nb; ++m) {
                const size_t n = static_cast<size_t>(cnt[m]);
                if (n <= st.keep || ceil_div(n, st.chunk_size) <= st.keep / st.chunk_size) continue;  // identity
                std::vector<std::size_t> list(n);
                for (size_t i = 0; i < n; ++i)
                    list[i] = in_list.p ? static_cast<size_t>(lst[m * in_stride + i]) : plan.sink_tokens + i;
                replay_stage_reads(*replay, list, st.chunk_size, static_cast<size_t>(heads),
                                   ph.data() + m * static_cast<size_t>(max_chunks) * heads);
            }
        }
        if (trace) {
            int32_t c = 0;
            out_count.download(&c, 4, (nb - 1) * 4);
            std::vector<int32_t> tmp(c);
            if (c) out_list.download(tmp.data(), c * 4, (nb - 1) * out_stride * 4);
            trace->last_block_outputs.emplace_back(tmp.begin(), tmp.end());
        }
        in_list = std::move(out_list);
        in_count = std::move(out_count);
        in_stride = static_cast<int64_t>(out_stride);
        max_in = st.keep;
        if (si + 1 < plan.stages.size() && plan.stages[si + 1].query_block != bq) {
            const size_t bq_next = plan.stages[si + 1].query_block;
            const size_t nb2 = ceil_div(t_q, bq_next);
            DevBuf nl(nb2 * out_stride * 4), nc(nb2 * 4);
            check(hp_remap_blocks(in_list.as<int32_t>(), in_count.as<int32_t>(), in_stride, 1,
                                  static_cast<int32_t>(nb), static_cast<int32_t>(bq), static_cast<int32_t>(bq_next),
                                  static_cast<int32_t>(t_q), static_cast<int64_t>(offset),
                                  static_cast<int32_t>(plan.stream_tokens), nl.as<int32_t>(), nc.as<int32_t>(),
                                  static_cast<int64_t>(out_stride), nullptr));
            in_list = std::move(nl);
            in_count = std::move(nc);
            nb = nb2;
        }
    }
    std::vector<int32_t> cnt(nb), lists(nb * in_stride);
    in_count.download(cnt.data(), nb * 4);
    in_list.download(lists.data(), lists.size() * 4);
    SparseBlockMask mask;
    mask.block_size = plan.stages.back().query_block;
    mask.sink_tokens = plan.sink_tokens;
    mask.stream_tokens = plan.stream_tokens;
    mask.query_offset = offset;
    mask.indices.resize(nb);
    for (size_t m = 0; m < nb; ++m)
        mask.indices[m].assign(lists.begin() + m * in_stride, lists.begin() + m * in_stride + cnt[m]);
    return mask;
}

SparseBlockMask build_mask(const PruningPlan& plan, const AttentionWorkload& wl, std::size_t layer,
                           const RopePolicySet& policy, const RopeTable& rope, KeySource* keys, StageTrace* trace,
                           std::size_t) {
    if (keys == nullptr) return build_mask_device(plan, wl, layer, policy, rope, &wl, layer, nullptr, nullptr, trace);
    if (auto* d = dynamic_cast<DirectKeySource*>(keys))
        return build_mask_device(plan, wl, layer, policy, rope, &d->workload(), d->layer(), nullptr, keys, trace);
    if (auto* v = dynamic_cast<KvView*>(keys))
        return build_mask_device(plan, wl, layer, policy, rope, &v->host(), v->layer(), nullptr, keys, trace);
    return build_mask_device(plan, wl, layer, policy, rope, nullptr, 0, keys, nullptr, trace);
}

SparseBlockMask build_mask(const PruningPlan& plan, const AttentionWorkload& wl, std::size_t layer,
                           const RopePolicySet& policy, const RopeTable& rope, StageTrace* trace,
                           std::size_t num_threads) {
    return build_mask(plan, wl, layer, policy, rope, static_cast<KeySource*>(nullptr), trace, num_threads);
}

// ========================================================= sparse attention
namespace {

// Row slices of the block-sparse attention on the device (selected lists per row,
// then split-K attention). mask_lists: [n_blocks][stride] int32 on the device.
void bsa_rows(const AttentionWorkload& wl, size_t layer, const DeviceLayer& kv, const int32_t* d_mask_lists,
              const int32_t* d_mask_counts, size_t mask_stride, size_t max_mask, size_t block_size,
              size_t query_offset, size_t sink, size_t stream, const RopePolicySet& policy, const DeviceRope* rope,
              AttentionOutput& out) {
    const size_t t_q = wl.seq_len_q, d = wl.head_dim, H = wl.num_heads;
    const size_t sel_stride = std::min<size_t>(sink + max_mask + stream + 1, wl.seq_len_kv + 1);
    // rows per slice: keep the selected lists under ~256 MB
    const size_t slice = std::max<size_t>(
        block_size, std::min<size_t>(t_q, (256u << 20) / (sel_stride * 4) / block_size * block_size));
    out.heads.assign(H, DenseMatrix(t_q, d));
    const hp_rope_ctx rc = rope_ctx(policy, policy.extension_enabled ? rope : nullptr, 0);
    DevBuf sel, selc, q, o, ws;
    for (size_t r0 = 0; r0 < t_q; r0 += slice) {
        const size_t r1 = std::min(t_q, r0 + slice), rows = r1 - r0;
        const size_t b0 = r0 / block_size;
        if (sel.bytes < rows * sel_stride * 4) sel.alloc(rows * sel_stride * 4);
        if (selc.bytes < rows * 4) selc.alloc(rows * 4);
        check(hp_selected_indices(d_mask_lists + b0 * mask_stride, d_mask_counts + b0,
                                  static_cast<int64_t>(mask_stride), 1, static_cast<int32_t>(rows),
                                  static_cast<int32_t>(block_size), static_cast<int64_t>(query_offset + r0),
                                  static_cast<int32_t>(sink), static_cast<int32_t>(stream), sel.as<int32_t>(),
                                  selc.as<int32_t>(), static_cast<int64_t>(sel_stride), nullptr));
        const std::vector<float> qh = pack_q(wl, layer, r0, r1);
        if (q.bytes < qh.size() * 4) q.alloc(qh.size() * 4);
        q.upload(qh.data(), qh.size() * 4);
        if (o.bytes < qh.size() * 4) o.alloc(qh.size() * 4);
        const size_t need = hp_bsa_workspace_bytes(static_cast<int32_t>(H), static_cast<int32_t>(rows),
                                                   static_cast<int32_t>(sel_stride), static_cast<int32_t>(d));
        if (ws.bytes < need) ws.alloc(need);
        hp_bsa_args a{};
        a.n_q_heads = static_cast<int32_t>(H);
        a.heads_per_mask = static_cast<int32_t>(H);
        a.n_rows = static_cast<int32_t>(rows);
        a.q = q.as<float>();
        a.query_offset = static_cast<int64_t>(query_offset + r0);
        a.sel_list = sel.as<int32_t>();
        a.sel_count = selc.as<int32_t>();
        a.sel_stride = static_cast<int64_t>(sel_stride);
        a.max_sel = static_cast<int32_t>(sel_stride);
        a.out = o.as<float>();
        a.workspace = ws.p;
        a.workspace_bytes = ws.bytes;
        a.kv = kv.view();
        a.rope = rc;
        check(hp_bsa(&a, nullptr));
        std::vector<float> oh(qh.size());
        o.download(oh.data(), oh.size() * 4);
        for (size_t h = 0; h < H; ++h)
            std::memcpy(out.heads[h].row(r0), &oh[h * rows * d], rows * d * 4);
    }
}

}  // namespace

AttentionOutput block_sparse_attention(const AttentionWorkload& wl, std::size_t layer, const SparseBlockMask& mask,
                                       const RopePolicySet& policy, const RopeTable& rope) {
    if (layer >= wl.num_layers) throw std::out_of_range("block_sparse_attention: layer out of range");
    if (mask.block_size == 0 || mask.num_blocks() != ceil_div(wl.seq_len_q, mask.block_size))
        throw std::invalid_argument("block_sparse_attention: mask does not cover the queries");
    if (policy.extension_enabled && policy.bsa_policy != RopePolicyId::Streaming)
        throw std::invalid_argument("block_sparse_attention: unsupported BSA position policy");
    require_device();
    DeviceLayer kv;
    kv.build(wl, layer, true);
    DeviceRope drope;
    if (policy.extension_enabled) drope.upload(rope);
    size_t stride = 1;
    for (const auto& l : mask.indices) stride = std::max(stride, l.size());
    std::vector<int32_t> lists(mask.num_blocks() * stride, 0), counts(mask.num_blocks());
    for (size_t b = 0; b < mask.num_blocks(); ++b) {
        counts[b] = static_cast<int32_t>(mask.indices[b].size());
        for (size_t i = 0; i < mask.indices[b].size(); ++i) {
            if (mask.indices[b][i] >= wl.seq_len_kv) throw std::out_of_range("block_sparse_attention: mask index out of range");
            lists[b * stride + i] = static_cast<int32_t>(mask.indices[b][i]);
        }
    }
    DevBuf dl(lists.size() * 4), dc(counts.size() * 4);
    dl.upload(lists.data(), lists.size() * 4);
    dc.upload(counts.data(), counts.size() * 4);
    AttentionOutput out;
    bsa_rows(wl, layer, kv, dl.as<int32_t>(), dc.as<int32_t>(), stride, stride, mask.block_size, mask.query_offset,
             mask.sink_tokens, mask.stream_tokens, policy, &drope, out);
    return out;
}

AttentionOutput dense_attention(const AttentionWorkload& wl, std::size_t layer) {
    if (layer >= wl.num_layers) throw std::out_of_range("dense_attention: layer out of range");
    require_device();
    DeviceLayer kv;
    kv.build(wl, layer, true);
    // every row shares one middle list holding every token (list stride 0, block size
    // 1); no sinks, no stream window: each row attends causally to [0, pos]
    // (sparse_attention.cpp:62-93)
    const size_t t_kv = wl.seq_len_kv;
    std::vector<int32_t> all(t_kv);
    std::iota(all.begin(), all.end(), 0);
    const std::vector<int32_t> cnt(wl.seq_len_q, static_cast<int32_t>(t_kv));
    DevBuf dl(t_kv * 4), dc(cnt.size() * 4);
    dl.upload(all.data(), t_kv * 4);
    dc.upload(cnt.data(), cnt.size() * 4);
    RopePolicySet raw;
    raw.extension_enabled = false;
    AttentionOutput out;
    bsa_rows(wl, layer, kv, dl.as<int32_t>(), dc.as<int32_t>(), 0, t_kv, 1, t_kv - wl.seq_len_q, 0, 0, raw,
             nullptr, out);
    return out;
}

std::vector<std::size_t> selected_indices(const SparseBlockMask& mask, std::size_t row) {
    if (mask.block_size == 0) throw std::out_of_range("selected_indices: row outside the mask");
    const size_t block = row / mask.block_size;
    if (block >= mask.num_blocks()) throw std::out_of_range("selected_indices: row outside the mask");
    const size_t pos = mask.query_offset + row;
    const size_t sink_end = std::min(mask.sink_tokens, pos + 1);
    const size_t stream_begin = std::max(pos + 1 > mask.stream_tokens ? pos + 1 - mask.stream_tokens : 0, sink_end);
    std::vector<size_t> sel;
    for (size_t j = 0; j < sink_end; ++j) sel.push_back(j);
    for (size_t idx : mask.indices[block])
        if (idx >= sink_end && idx < stream_begin) sel.push_back(idx);
    for (size_t j = stream_begin; j <= pos; ++j) sel.push_back(j);
    return sel;
}

std::vector<std::size_t> exact_topk(std::span<const float> query, const DenseMatrix& keys, std::size_t k) {
    if (k > keys.rows) throw std::invalid_argument("exact_topk: k exceeds the key count");
    std::vector<float> sc(keys.rows);
    for (size_t j = 0; j < keys.rows; ++j) sc[j] = dot_seq(query, keys.row_span(j));
    std::vector<size_t> order(keys.rows);
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return sc[a] > sc[b]; });
    order.resize(k);
    return order;
}

double attention_recall(std::span<const std::size_t> selected, std::span<const float> query, const DenseMatrix& keys) {
    std::vector<char> in(keys.rows, 0);
    for (size_t i : selected) {
        if (i >= keys.rows) throw std::out_of_range("attention_recall: selected index out of range");
        in[i] = 1;
    }
    const float scale = 1.0f / std::sqrt(static_cast<float>(keys.cols));
    std::vector<float> sc(keys.rows);
    float mx = -std::numeric_limits<float>::infinity();
    for (size_t j = 0; j < keys.rows; ++j) {
        sc[j] = dot_seq(query, keys.row_span(j)) * scale;
        mx = std::max(mx, sc[j]);
    }
    double tot = 0.0, cap = 0.0;
    for (size_t j = 0; j < keys.rows; ++j) {
        const double w = std::exp(static_cast<double>(sc[j]) - mx);
        tot += w;
        if (in[j]) cap += w;
    }
    return cap / tot;
}

bool device_available() { return hp_device_available() != 0; }

// ===================================================== reference host helpers
// tensor.cpp / rope_policy.cpp restated: the arithmetic contract the kernels reproduce.
void apply_rope_inplace(std::span<float> vec, std::size_t position, const RopeTable& table) {
    if (vec.size() != table.head_dim)
        throw std::invalid_argument("apply_rope: vector length " + std::to_string(vec.size()) + " != head_dim " +
                                    std::to_string(table.head_dim));
    if (position >= table.max_position)
        throw std::out_of_range("apply_rope: position " + std::to_string(position) + " >= max_position " +
                                std::to_string(table.max_position));
    const size_t half = table.head_dim / 2;
    const float* c = table.cos_tab.row(position);
    const float* sn = table.sin_tab.row(position);
    for (size_t i = 0; i < half; ++i) {
        const float x = vec[i], y = vec[i + half];
        const float xc = x * c[i], ys = y * sn[i], xs = x * sn[i], yc = y * c[i];
        vec[i] = xc - ys;
        vec[i + half] = xs + yc;
    }
}

std::vector<float> apply_rope(std::span<const float> vec, std::size_t position, const RopeTable& table) {
    std::vector<float> out(vec.begin(), vec.end());
    apply_rope_inplace(out, position, table);
    return out;
}

float dot_f32(std::span<const float> a, std::span<const float> b) {
    if (a.size() != b.size())
        throw std::invalid_argument("dot_f32: length mismatch " + std::to_string(a.size()) + " vs " +
                                    std::to_string(b.size()));
    return dot_seq(a, b);
}

float block_scores(const DenseMatrix& qblock, std::span<const float> key) {
    if (qblock.cols != key.size())
        throw std::invalid_argument("block_scores: qblock cols " + std::to_string(qblock.cols) + " != key length " +
                                    std::to_string(key.size()));
    if (qblock.rows == 0) throw std::invalid_argument("block_scores: empty query block");
    float best = dot_seq(qblock.row_span(0), key);
    for (size_t t = 1; t < qblock.rows; ++t) best = std::max(best, dot_seq(qblock.row_span(t), key));
    return best;
}

namespace {
RopePolicyId pruning_policy_of(const RopePolicySet& p, std::size_t layer) {
    return layer > p.early_layer_cutoff ? p.pruning_policy_late : p.pruning_policy_early;
}
}  // namespace

std::size_t query_position(const RopePolicySet& policy, std::size_t layer, const PositionContext& ctx) {
    switch (pruning_policy_of(policy, layer)) {
        case RopePolicyId::Relative: return ctx.stream_tokens + 1;
        case RopePolicyId::ChunkIndexed: return std::min(ctx.query_position, ctx.chunk_count + ctx.stream_tokens);
        case RopePolicyId::PlugIn:
            if (!policy.plugin) throw std::logic_error("query_position: PlugIn policy without a registered hook");
            return policy.plugin(true, layer, ctx);
        default: break;
    }
    throw std::logic_error("query_position: policy not applicable to pruning");
}

std::size_t key_position(const RopePolicySet& policy, std::size_t layer, const PositionContext& ctx) {
    if (ctx.branch != 1 && ctx.branch != 2) throw std::logic_error("key_position: branch must be 1 or 2");
    switch (pruning_policy_of(policy, layer)) {
        case RopePolicyId::Relative: return static_cast<std::size_t>(ctx.branch - 1);
        case RopePolicyId::ChunkIndexed: return ctx.chunk_index;
        case RopePolicyId::PlugIn:
            if (!policy.plugin) throw std::logic_error("key_position: PlugIn policy without a registered hook");
            return policy.plugin(false, layer, ctx);
        default: break;
    }
    throw std::logic_error("key_position: policy not applicable to pruning");
}

std::vector<std::size_t> streaming_positions(std::span<const std::size_t> selected, std::size_t query_pos,
                                             std::size_t) {
    const size_t n = selected.size();
    if (n > query_pos + 1)
        throw std::logic_error("streaming_positions: " + std::to_string(n) + " selected tokens cannot fit below position " +
                               std::to_string(query_pos));
    std::vector<std::size_t> pos(n);
    for (size_t i = 0; i < n; ++i) pos[i] = query_pos + 1 - n + i;
    return pos;
}

ChunkPartition partition_chunks(std::span<const std::size_t> indices, std::size_t chunk_size) {
    if (chunk_size == 0) throw std::invalid_argument("partition_chunks: chunk_size must be >= 1");
    ChunkPartition out;
    for (size_t b = 0; b < indices.size(); b += chunk_size)
        out.chunks.emplace_back(indices.begin() + b, indices.begin() + std::min(indices.size(), b + chunk_size));
    return out;
}

ChunkSparsity chunk_sparsity_histogram(std::span<const float> query, const DenseMatrix& keys, std::size_t k,
                                       std::size_t chunk_size) {
    if (chunk_size == 0 || chunk_size > keys.rows)
        throw std::invalid_argument("chunk_sparsity_histogram: chunk size out of range");
    const std::vector<std::size_t> top = exact_topk(query, keys, k);
    ChunkSparsity out;
    out.chunk_counts.assign(ceil_div(keys.rows, chunk_size), 0);
    for (size_t i : top) ++out.chunk_counts[i / chunk_size];
    const size_t empty = static_cast<size_t>(std::count(out.chunk_counts.begin(), out.chunk_counts.end(), size_t{0}));
    out.empty_fraction = static_cast<double>(empty) / static_cast<double>(out.chunk_counts.size());
    return out;
}

// ========================================================= KeySource operators
namespace {

int ceil_log2(size_t n) {
    int r = 0;
    while ((size_t{1} << r) < n) ++r;
    return r;
}

// The reference's key reads of one stage (run_pruning_stage + select_rep_rotated,
// pruning.cpp:69-98,170-185), replayed from the device's branch decisions:
// chunk by chunk, head by head, per iteration chunk[first-1] then chunk[mid-1],
// then the representative once more for its branch-2 score.
void replay_stage_reads(KeySource& ks, std::span<const std::size_t> list, std::size_t lc, std::size_t heads,
                        const std::uint32_t* paths) {
    const size_t cc = ceil_div(list.size(), lc);
    for (size_t j = 0; j < cc; ++j) {
        const size_t b = j * lc, n = std::min(lc, list.size() - b);
        for (size_t h = 0; h < heads; ++h) {
            size_t first = 1, last = n;
            if (n > 1) {
                const std::uint32_t bits = paths[j * heads + h];
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

// select_rep's own reads (no trailing representative read) for one chunk
size_t replay_select_rep(KeySource& ks, std::span<const std::size_t> chunk, std::size_t head, std::uint32_t bits) {
    size_t first = 1, last = chunk.size();
    const int iters = ceil_log2(chunk.size());
    for (int it = 0; it < iters && first < last; ++it) {
        const size_t mid = (first + last + 1) / 2;
        ks.key_row(head, chunk[first - 1]);
        ks.key_row(head, chunk[mid - 1]);
        if ((bits >> it) & 1u) first = mid;
        else last = mid - 1;
    }
    return chunk[first - 1];
}

// K (and V) rows of a device layer [pages][heads][64][d] fp32: the workload layer when
// known, else through the source (`tokens` — or every token below t_kv — read once)
void build_layer_from_source(DeviceLayer& dl, KeySource& ks, const AttentionWorkload* src_wl, size_t src_layer,
                             size_t heads, size_t t_kv, size_t d, bool with_values,
                             std::span<const std::size_t> tokens) {
    if (src_wl) {
        dl.build(*src_wl, src_layer, with_values);
        return;
    }
    const int32_t ps = 64;
    dl.heads = static_cast<int32_t>(heads);
    dl.d = static_cast<int32_t>(d);
    dl.page_size = ps;
    dl.t_kv = static_cast<int64_t>(t_kv);
    dl.pages = static_cast<int32_t>(std::max<size_t>(1, ceil_div(t_kv, ps)));
    const size_t n = static_cast<size_t>(dl.pages) * heads * ps * d;
    std::vector<float> hk(n, 0.0f), hv(with_values ? n : 0, 0.0f);
    auto put = [&](size_t h, size_t t) {
        const size_t o = (((t / ps) * heads + h) * ps + t % ps) * d;
        const auto kr = ks.key_row(h, t);
        if (kr.size() != d) throw std::invalid_argument("KeySource: key row width != head_dim");
        std::memcpy(&hk[o], kr.data(), d * 4);
        if (with_values) {
            const auto vr = ks.value_row(h, t);
            if (vr.size() != d) throw std::invalid_argument("KeySource: value row width != head_dim");
            std::memcpy(&hv[o], vr.data(), d * 4);
        }
    };
    for (size_t h = 0; h < heads; ++h) {
        if (tokens.empty())
            for (size_t t = 0; t < t_kv; ++t) put(h, t);
        else
            for (size_t t : tokens) put(h, t);
    }
    dl.k.alloc(n * 4);
    dl.k.upload(hk.data(), n * 4);
    if (with_values) {
        dl.v.alloc(n * 4);
        dl.v.upload(hv.data(), n * 4);
    }
}

struct SourceInfo {
    const AttentionWorkload* wl = nullptr;
    size_t layer = 0;
    bool ours = false;  // a DirectKeySource / KvView: read its host tier, replay the reads
};
SourceInfo source_info(KeySource& ks) {
    if (auto* d = dynamic_cast<DirectKeySource*>(&ks)) return {&d->workload(), d->layer(), true};
    if (auto* v = dynamic_cast<KvView*>(&ks)) return {&v->host(), v->layer(), true};
    return {};
}

void check_sorted_unique(std::span<const std::size_t> idx, const char* where) {
    for (size_t i = 1; i < idx.size(); ++i)
        if (idx[i] <= idx[i - 1]) throw ContractViolation(std::string(where) + ": indices must be sorted and duplicate-free");
}

// One stage on the device over one list (one mask pooling `qblocks.size()` heads).
// Returns the output list; `paths` (if given) receives the branch decisions [chunk][head].
std::vector<std::size_t> stage_on_device(const StageConfig& stage, std::span<const std::size_t> list,
                                         std::span<const DenseMatrix> qblocks, KeySource& keys, const StageContext& ctx,
                                         bool descend_always, std::vector<std::uint32_t>* paths) {
    if (!ctx.policy) throw std::invalid_argument("StageContext: policy is required");
    const size_t H = qblocks.size();
    if (H == 0) throw std::invalid_argument("run_pruning_stage: no query blocks");
    const size_t rows = qblocks[0].rows, d = qblocks[0].cols;
    for (const auto& q : qblocks)
        if (q.rows != rows || q.cols != d || rows == 0) throw std::invalid_argument("run_pruning_stage: query block shapes differ");
    if (list.empty()) return {};
    if (list.back() >= static_cast<size_t>(1u << 31)) throw std::out_of_range("run_pruning_stage: token index beyond 2^31");
    require_device();
    const SourceInfo si = source_info(keys);
    const size_t t_kv = list.back() + 1;
    DeviceLayer kv;
    build_layer_from_source(kv, keys, si.wl, si.layer, H, si.wl ? si.wl->seq_len_kv : t_kv, d, false, list);
    if (si.wl && (kv.heads != static_cast<int32_t>(H) || kv.d != static_cast<int32_t>(d)))
        throw std::invalid_argument("run_pruning_stage: query heads / dims do not match the key source");
    std::vector<float> qh(H * rows * d);
    for (size_t h = 0; h < H; ++h) std::memcpy(&qh[h * rows * d], qblocks[h].data.data(), rows * d * 4);
    DevBuf q(qh.size() * 4);
    q.upload(qh.data(), qh.size() * 4);
    std::vector<int32_t> li(list.begin(), list.end());
    const int32_t n = static_cast<int32_t>(li.size());
    DevBuf dl(li.size() * 4), dc(4), ol(std::max<size_t>(stage.keep, li.size()) * 4), oc(4);
    dl.upload(li.data(), li.size() * 4);
    dc.upload(&n, 4);
    const int32_t cc = static_cast<int32_t>(ceil_div(li.size(), stage.chunk_size));
    const size_t need = hp_stage_workspace_bytes(1, cc, static_cast<int32_t>(stage.keep), static_cast<int32_t>(stage.chunk_size));
    DevBuf ws(need);
    DeviceRope drope;
    if (ctx.policy->extension_enabled) {
        if (!ctx.rope) throw std::invalid_argument("StageContext: extension enabled without a rope table");
        drope.upload(*ctx.rope);
    }
    DevBuf dp;
    if (paths) dp.alloc(static_cast<size_t>(cc) * H * 4);
    hp_stage_args a{};
    a.query_block = static_cast<int32_t>(rows);
    a.chunk_size = static_cast<int32_t>(stage.chunk_size);
    a.keep = static_cast<int32_t>(stage.keep);
    a.n_masks = 1;
    a.heads_per_mask = static_cast<int32_t>(H);
    a.n_q_heads = static_cast<int32_t>(H);
    a.n_blocks = 1;
    a.q_rows = static_cast<int32_t>(rows);
    a.q = q.as<float>();
    a.query_offset = static_cast<int64_t>(ctx.query_start_position);
    a.stream_tokens = static_cast<int32_t>(ctx.stream_tokens);
    a.max_chunks = cc;
    a.in_list = dl.as<int32_t>();
    a.in_count = dc.as<int32_t>();
    a.in_stride = n;
    a.out_list = ol.as<int32_t>();
    a.out_count = oc.as<int32_t>();
    a.out_stride = static_cast<int64_t>(ol.bytes / 4);
    a.workspace = ws.p;
    a.workspace_bytes = ws.bytes;
    a.keys = kv.view();
    a.rope = rope_ctx(*ctx.policy, ctx.policy->extension_enabled ? &drope : nullptr, ctx.layer);
    a.path_out = paths ? dp.as<std::uint32_t>() : nullptr;
    a.descend_always = descend_always ? 1 : 0;
    check(hp_prune_stage(&a, nullptr));
    int32_t c = 0;
    oc.download(&c, 4);
    std::vector<int32_t> out(std::max(0, c));
    if (c > 0) ol.download(out.data(), static_cast<size_t>(c) * 4);
    if (paths) {
        paths->resize(static_cast<size_t>(cc) * H);
        dp.download(paths->data(), paths->size() * 4);
    }
    return std::vector<std::size_t>(out.begin(), out.end());
}

}  // namespace

std::vector<std::size_t> run_pruning_stage(const StageConfig& stage, std::span<const std::size_t> indices,
                                           std::span<const DenseMatrix> qblocks, KeySource& keys,
                                           const StageContext& ctx) {
    stage.validate();
    check_sorted_unique(indices, "run_pruning_stage");
    if (indices.size() <= stage.keep) return {indices.begin(), indices.end()};  // identity: no reads
    if (ceil_div(indices.size(), stage.chunk_size) <= stage.keep / stage.chunk_size)
        return {indices.begin(), indices.end()};
    const bool ours = source_info(keys).ours;
    std::vector<std::uint32_t> paths;
    std::vector<std::size_t> out = stage_on_device(stage, indices, qblocks, keys, ctx, false, ours ? &paths : nullptr);
    if (ours) replay_stage_reads(keys, indices, stage.chunk_size, qblocks.size(), paths.data());
    return out;
}

std::size_t select_rep(const DenseMatrix& qblock, std::span<const std::size_t> chunk, KeySource& keys,
                       std::size_t head, const StageContext& ctx, std::size_t chunk_index, std::size_t chunk_count) {
    if (chunk.empty()) throw ContractViolation("select_rep: empty chunk");
    if (chunk.size() == 1) return chunk[0];
    if (!ctx.policy) throw std::invalid_argument("StageContext: policy is required");
    // one device stage whose chunk `chunk_index` of `chunk_count` is this chunk (the
    // chunk position sets the RoPE positions; copies elsewhere only keep them aligned)
    const size_t n = chunk.size();
    const bool ext = ctx.policy->extension_enabled;
    const size_t copies = ext ? std::max<size_t>(chunk_count, chunk_index + 1) : 1;
    const size_t at = ext ? chunk_index : 0;
    std::vector<std::size_t> list;
    list.reserve(copies * n);
    for (size_t c = 0; c < copies; ++c) list.insert(list.end(), chunk.begin(), chunk.end());
    // a single-head key source view: rows of `head` as kv head 0
    struct HeadSource final : KeySource {
        KeySource* ks;
        size_t head;
        std::span<const float> key_row(std::size_t, std::size_t t) override { return ks->key_row(head, t); }
        std::span<const float> value_row(std::size_t, std::size_t t) override { return ks->value_row(head, t); }
    } one;
    one.ks = &keys;
    one.head = head;
    const SourceInfo si = source_info(keys);
    StageConfig st{qblock.rows, n, n};
    std::vector<std::uint32_t> paths;
    std::vector<DenseMatrix> qb{qblock};
    if (si.wl) {  // the source's host tier, one head
        AttentionWorkload w1;
        w1.num_heads = 1;
        w1.num_layers = 1;
        w1.seq_len_kv = si.wl->seq_len_kv;
        w1.head_dim = qblock.cols;
        w1.keys = {{si.wl->k(si.layer, head)}};
        w1.values = {{DenseMatrix()}};
        DirectKeySource direct(w1, 0);
        stage_on_device(st, list, qb, direct, ctx, true, &paths);
    } else {
        stage_on_device(st, list, qb, one, ctx, true, &paths);
    }
    const std::uint32_t bits = paths[at];
    if (si.ours) return replay_select_rep(keys, chunk, head, bits);
    size_t first = 1, last = n;
    const int iters = ceil_log2(n);
    for (int it = 0; it < iters && first < last; ++it) {
        const size_t mid = (first + last + 1) / 2;
        if ((bits >> it) & 1u) first = mid;
        else last = mid - 1;
    }
    return chunk[first - 1];
}

std::vector<float> attention_row(std::span<const float> q_row, std::span<const std::size_t> selected,
                                 std::size_t query_position, bool extension_enabled, const RopeTable& rope,
                                 KeySource& kv, std::size_t head) {
    if (selected.empty()) throw std::invalid_argument("attention_row: empty selected set");
    const size_t d = q_row.size();
    if (extension_enabled) {
        streaming_positions(selected, query_position, 0);  // throws as the reference does
        if (query_position >= rope.max_position)
            throw std::out_of_range("apply_rope: position " + std::to_string(query_position) + " >= max_position " +
                                    std::to_string(rope.max_position));
    }
    for (size_t i = 1; i < selected.size(); ++i)
        if (selected[i] <= selected[i - 1]) throw ContractViolation("attention_row: selected indices must be ascending");
    if (selected.back() >= static_cast<size_t>(1u << 31)) throw std::out_of_range("attention_row: token index beyond 2^31");
    require_device();
    const SourceInfo si = source_info(kv);
    // the head's K/V rows as a one-head device layer
    struct HeadSource final : KeySource {
        KeySource* ks;
        size_t head;
        std::span<const float> key_row(std::size_t, std::size_t t) override { return ks->key_row(head, t); }
        std::span<const float> value_row(std::size_t, std::size_t t) override { return ks->value_row(head, t); }
    } one;
    one.ks = &kv;
    one.head = head;
    DeviceLayer dl;
    if (si.wl) {
        AttentionWorkload w1;
        w1.num_heads = 1;
        w1.num_layers = 1;
        w1.seq_len_kv = si.wl->seq_len_kv;
        w1.head_dim = d;
        w1.keys = {{si.wl->k(si.layer, head)}};
        w1.values = {{si.wl->v(si.layer, head)}};
        dl.build(w1, 0, true);
    } else {
        build_layer_from_source(dl, one, nullptr, 0, 1, selected.back() + 1, d, true, selected);
    }
    std::vector<int32_t> sel(selected.begin(), selected.end());
    const int32_t n = static_cast<int32_t>(sel.size());
    DevBuf ds(sel.size() * 4), dc(4), q(d * 4), o(d * 4);
    ds.upload(sel.data(), sel.size() * 4);
    dc.upload(&n, 4);
    q.upload(q_row.data(), d * 4);
    DeviceRope drope;
    RopePolicySet pol;
    pol.extension_enabled = extension_enabled;
    if (extension_enabled) drope.upload(rope);
    const size_t need = hp_bsa_workspace_bytes(1, 1, n, static_cast<int32_t>(d));
    DevBuf ws(need);
    hp_bsa_args a{};
    a.n_q_heads = 1;
    a.heads_per_mask = 1;
    a.n_rows = 1;
    a.q = q.as<float>();
    a.query_offset = static_cast<int64_t>(query_position);
    a.sel_list = ds.as<int32_t>();
    a.sel_count = dc.as<int32_t>();
    a.sel_stride = n;
    a.max_sel = n;
    a.out = o.as<float>();
    a.workspace = ws.p;
    a.workspace_bytes = ws.bytes;
    a.kv = dl.view();
    a.rope = rope_ctx(pol, extension_enabled ? &drope : nullptr, 0);
    check(hp_bsa(&a, nullptr));
    std::vector<float> out(d);
    o.download(out.data(), d * 4);
    if (si.ours) {  // the reference's reads: every key row, then every value row
        for (size_t t : selected) kv.key_row(head, t);
        for (size_t t : selected) kv.value_row(head, t);
    }
    return out;
}

AttentionOutput block_sparse_attention(const AttentionWorkload& wl, std::size_t layer, const SparseBlockMask& mask,
                                       const RopePolicySet& policy, const RopeTable& rope, KeySource& kvs) {
    if (layer >= wl.num_layers) throw std::out_of_range("block_sparse_attention: layer out of range");
    if (mask.block_size == 0 || mask.num_blocks() != ceil_div(wl.seq_len_q, mask.block_size))
        throw std::invalid_argument("block_sparse_attention: mask does not cover the queries");
    if (policy.extension_enabled && policy.bsa_policy != RopePolicyId::Streaming)
        throw std::invalid_argument("block_sparse_attention: unsupported BSA position policy");
    const SourceInfo si = source_info(kvs);
    AttentionOutput out;
    if (si.wl && si.wl == &wl && si.layer == layer) {
        out = block_sparse_attention(wl, layer, mask, policy, rope);
    } else {
        // rows through the source: a workload copy whose layer holds them
        require_device();
        AttentionWorkload w = wl;
        for (size_t h = 0; h < wl.num_heads; ++h)
            for (size_t t = 0; t < wl.seq_len_kv; ++t) {
                const auto kr = si.wl ? si.wl->k(si.layer, h).row_span(t) : kvs.key_row(h, t);
                const auto vr = si.wl ? si.wl->v(si.layer, h).row_span(t) : kvs.value_row(h, t);
                std::memcpy(w.keys[layer][h].row(t), kr.data(), wl.head_dim * 4);
                std::memcpy(w.values[layer][h].row(t), vr.data(), wl.head_dim * 4);
            }
        out = block_sparse_attention(w, layer, mask, policy, rope);
    }
    if (si.ours) {  // head by head, row by row: keys then values (sparse_attention.cpp:128-140)
        for (size_t h = 0; h < wl.num_heads; ++h)
            for (size_t r = 0; r < wl.seq_len_q; ++r) {
                const std::vector<std::size_t> sel = selected_indices(mask, r);
                for (size_t t : sel) kvs.key_row(h, t);
                for (size_t t : sel) kvs.value_row(h, t);
            }
    }
    return out;
}

}  // namespace hipprune

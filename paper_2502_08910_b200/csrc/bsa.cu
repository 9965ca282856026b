// Block-sparse attention over selected index lists (decode + row-wise prefill).
//
// Replaces selected_indices / attention_row / softmax_weighted_sum /
// block_sparse_attention (reference proj/src/sparse_attention.cpp:15-60,95-145).
// Memory-bound split-K: each CTA owns a contiguous slice of one row's selected
// list for HC q-heads that share a kv head and a mask (GQA: the K/V row is
// gathered once and used by all HC heads). Scores s_j = (q·k_j)/sqrt(d) with the
// reference's scale; softmax by warp-shuffle online max/sum; partial (m, l, o)
// triples are merged by a log-sum-exp combine. With the extension on, keys sit
// at the reference's streaming positions pos+1-n+j and q at pos (RoPE fused into
// the gather). Results match the reference within 1e-3 relative (fp32 math from
// identical fp32 / bf16-rounded inputs; only the summation order differs).

#include <algorithm>
#include <cmath>

#include "common.cuh"

using namespace hpk;

namespace {

constexpr int kBsaThreads = 128;   // 4 warps
constexpr int kKeysPerWarp = 8;    // per tile
constexpr int kTile = kBsaThreads / 32 * kKeysPerWarp;  // 32 list positions per tile
constexpr int kMaxHC = 8;

// selected_indices (sparse_attention.cpp:95-112) for n_rows rows of every mask.
__global__ void selected_kernel(const int32_t* mask_list, const int32_t* mask_count,
                                int64_t mask_stride, int n_rows, int n_mask_blocks, int block_size,
                                int64_t offset, int sink, int stream, int32_t* sel, int32_t* cnt,
                                int64_t sel_stride) {
    __shared__ int scan_tmp[32];
    const int mr = blockIdx.x;
    const int m = mr / n_rows, r = mr % n_rows;
    const int blk = r / block_size;
    int32_t* out = sel + static_cast<int64_t>(mr) * sel_stride;
    if (blk >= n_mask_blocks) {
        if (threadIdx.x == 0) cnt[mr] = -1;
        return;
    }
    const int64_t pos = offset + r;
    const int64_t sink_end = min64(sink, pos + 1);
    int64_t stream_begin = pos + 1 > stream ? pos + 1 - stream : 0;
    stream_begin = max64(stream_begin, sink_end);
    const int32_t* src = mask_list + (static_cast<int64_t>(m) * n_mask_blocks + blk) * mask_stride;
    const int n = mask_count[m * n_mask_blocks + blk];
    // count first to check capacity
    int base = static_cast<int>(sink_end);
    const int64_t total_bound = sink_end + n + (pos + 1 - stream_begin);
    const bool fits = total_bound <= sel_stride;
    for (int64_t i = threadIdx.x; i < sink_end && fits; i += blockDim.x) out[i] = static_cast<int32_t>(i);
    for (int tile = 0; tile < n; tile += blockDim.x) {
        const int i = tile + threadIdx.x;
        const int32_t idx = i < n ? src[i] : 0;
        const int keep = i < n && idx >= sink_end && idx < stream_begin;
        int tot;
        const int rk = block_exclusive_scan<256>(keep, scan_tmp, &tot) + base;
        if (keep && fits) out[rk] = idx;
        base += tot;
    }
    const int64_t n_stream = pos + 1 - stream_begin;
    for (int64_t i = threadIdx.x; i < n_stream && fits; i += blockDim.x) out[base + i] = static_cast<int32_t>(stream_begin + i);
    if (threadIdx.x == 0) {
        if (!fits) cnt[mr] = -1;
        else cnt[mr] = static_cast<int32_t>(base + n_stream);
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Split-K attention. grid = (splits, n_rows, n_q_heads / HC). Lane L holds elements
// i = L + 32c (c < NC) of the first half and their RoPE partners i + d/2.
template <typename T, int NC, int HC, bool EXT>
__global__ void __launch_bounds__(kBsaThreads) bsa_kernel(const hp_bsa_args a, int splits,
                                                         int tiles_per_split, float* ws,
                                                         int* status) {
    constexpr int hc = HC;
    __shared__ float sm_m[4][HC], sm_l[4][HC];
    __shared__ float sm_o[4][HC][2 * NC * 32];
    const int d = a.kv.d, half = d >> 1;
    const int split = blockIdx.x, r = blockIdx.y, h0 = blockIdx.z * hc;
    const int lane = threadIdx.x & 31, w = warp_id();
    const int mask = h0 / a.heads_per_mask;
    const int kv = h0 / (a.n_q_heads / a.kv.n_kv);
    const int64_t mr = static_cast<int64_t>(mask) * a.n_rows + r;
    const int cnt = a.sel_count[mr];
    const int32_t* list = a.sel_list + mr * a.sel_stride;
    const int64_t pos = a.query_offset + r;
    const float scale = 1.0f / sqrtf(static_cast<float>(d));
    const int eb = sizeof(T);

    // q for hc heads (rotated at pos when the extension is on)
    float qx[HC][NC], qy[HC][NC];
    const float* cq = EXT ? a.rope.cos_tab + pos * half : nullptr;
    const float* sq = EXT ? a.rope.sin_tab + pos * half : nullptr;
#pragma unroll
    for (int hh = 0; hh < HC; ++hh) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int i = lane + 32 * c;
            float x = 0.f, y = 0.f;
            if (hh < hc && i < half) {
                const float* qrow = a.q + (static_cast<int64_t>(h0 + hh) * a.n_rows + r) * d;
                x = qrow[i]; y = qrow[i + half];
                if (EXT) {
                    const float cc = cq[i], ss = sq[i];
                    const float rx = x * cc - y * ss, ry = x * ss + y * cc;
                    x = rx; y = ry;
                }
            }
            qx[hh][c] = x; qy[hh][c] = y;
        }
    }

    float m_run[HC], l_run[HC], ox[HC][NC], oy[HC][NC];
#pragma unroll
    for (int hh = 0; hh < HC; ++hh) {
        m_run[hh] = -INFINITY; l_run[hh] = 0.f;
#pragma unroll
        for (int c = 0; c < NC; ++c) { ox[hh][c] = 0.f; oy[hh][c] = 0.f; }
    }

    const int p_begin = split * tiles_per_split * kTile;
    const int p_end = min(cnt, p_begin + tiles_per_split * kTile);
    for (int tb = p_begin; tb < p_end; tb += kTile) {
        // gather this warp's 16 K rows (all loads issued before use)
        float kx[kKeysPerWarp][NC], ky[kKeysPerWarp][NC];
        int toks[kKeysPerWarp];
#pragma unroll
        for (int k = 0; k < kKeysPerWarp; ++k) {
            const int p = tb + w * kKeysPerWarp + k;
            toks[k] = p < p_end ? list[p] : -1;
        }
#pragma unroll
        for (int k = 0; k < kKeysPerWarp; ++k) {
            const T* row = toks[k] >= 0 ? reinterpret_cast<const T*>(kv_row_ptr(a.kv, a.kv.k_pool, a.kv.k_host, kv, toks[k], eb)) : nullptr;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int i = lane + 32 * c;
                kx[k][c] = (row && i < half) ? load_elem(row, i) : 0.f;
                ky[k][c] = (row && i < half) ? load_elem(row, i + half) : 0.f;
            }
        }
        float s[HC][kKeysPerWarp];
#pragma unroll
        for (int k = 0; k < kKeysPerWarp; ++k) {
            const int p = tb + w * kKeysPerWarp + k;
            if (EXT && toks[k] >= 0) {
                const int64_t kp = pos + 1 - cnt + p;  // streaming_positions (rope_policy.cpp:59-72)
                const float* ck = a.rope.cos_tab + kp * half;
                const float* sk = a.rope.sin_tab + kp * half;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const int i = lane + 32 * c;
                    if (i < half) {
                        const float x = kx[k][c], y = ky[k][c], cc = ck[i], ss = sk[i];
                        kx[k][c] = x * cc - y * ss;
                        ky[k][c] = x * ss + y * cc;
                    }
                }
            }
#pragma unroll
            for (int hh = 0; hh < HC; ++hh) {
                float part = 0.f;
#pragma unroll
                for (int c = 0; c < NC; ++c) part += qx[hh][c] * kx[k][c] + qy[hh][c] * ky[k][c];
                part = warp_sum(part);
                s[hh][k] = toks[k] >= 0 ? part * scale : -INFINITY;
            }
        }
        // V rows
#pragma unroll
        for (int k = 0; k < kKeysPerWarp; ++k) {
            const T* row = toks[k] >= 0 ? reinterpret_cast<const T*>(kv_row_ptr(a.kv, a.kv.v_pool, a.kv.v_host, kv, toks[k], eb)) : nullptr;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int i = lane + 32 * c;
                kx[k][c] = (row && i < half) ? load_elem(row, i) : 0.f;
                ky[k][c] = (row && i < half) ? load_elem(row, i + half) : 0.f;
            }
        }
#pragma unroll
        for (int hh = 0; hh < HC; ++hh) {
            float mt = m_run[hh];
#pragma unroll
            for (int k = 0; k < kKeysPerWarp; ++k) mt = fmaxf(mt, s[hh][k]);
            if (mt == -INFINITY) continue;
            const float alpha = expf(m_run[hh] - mt);
            float l = l_run[hh] * alpha;
#pragma unroll
            for (int c = 0; c < NC; ++c) { ox[hh][c] *= alpha; oy[hh][c] *= alpha; }
#pragma unroll
            for (int k = 0; k < kKeysPerWarp; ++k) {
                const float pk = expf(s[hh][k] - mt);
                l += pk;
#pragma unroll
                for (int c = 0; c < NC; ++c) { ox[hh][c] += pk * kx[k][c]; oy[hh][c] += pk * ky[k][c]; }
            }
            m_run[hh] = mt; l_run[hh] = l;
        }
    }
    // merge the 4 warps
#pragma unroll
    for (int hh = 0; hh < HC; ++hh) {
        if (hh >= hc) break;
        if (lane == 0) { sm_m[w][hh] = m_run[hh]; sm_l[w][hh] = l_run[hh]; }
#pragma unroll
        for (int c = 0; c < NC; ++c) { sm_o[w][hh][lane + 32 * c] = ox[hh][c]; sm_o[w][hh][NC * 32 + lane + 32 * c] = oy[hh][c]; }
    }
    __syncthreads();
    for (int hh = 0; hh < hc; ++hh) {
        float M = -INFINITY;
        for (int ww = 0; ww < 4; ++ww) M = fmaxf(M, sm_m[ww][hh]);
        float L = 0.f, f[4];
        for (int ww = 0; ww < 4; ++ww) {
            f[ww] = sm_m[ww][hh] == -INFINITY ? 0.f : expf(sm_m[ww][hh] - M);
            L += sm_l[ww][hh] * f[ww];
        }
        const int64_t hr = static_cast<int64_t>(h0 + hh) * a.n_rows + r;
        for (int e = threadIdx.x; e < d; e += blockDim.x) {
            const int idx = e < half ? e : NC * 32 + (e - half);
            float o = 0.f;
            for (int ww = 0; ww < 4; ++ww) o += sm_o[ww][hh][idx] * f[ww];
            if (splits == 1) {
                a.out[hr * d + e] = L > 0.f ? o / L : NAN;
                if (a.part_o) a.part_o[hr * d + e] = L > 0.f ? o / L : 0.f;
            } else {
                ws[((static_cast<int64_t>(split) * a.n_q_heads * a.n_rows + hr) * (d + 2)) + 2 + e] = o;
            }
        }
        if (threadIdx.x == 0) {
            if (splits == 1) {
                if (a.part_m) { a.part_m[hr] = M; a.part_l[hr] = L; }
                if (!(L > 0.f)) atomicOr(status, 16);
            } else {
                float* wp = ws + (static_cast<int64_t>(split) * a.n_q_heads * a.n_rows + hr) * (d + 2);
                wp[0] = M; wp[1] = L;
            }
        }
    }
}

__global__ void bsa_combine_kernel(const hp_bsa_args a, int splits, const float* ws, int* status) {
    const int64_t hr = blockIdx.x;
    const int d = a.kv.d;
    const int64_t nhr = static_cast<int64_t>(a.n_q_heads) * a.n_rows;
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) {
        const float* wp = ws + (s * nhr + hr) * (d + 2);
        if (wp[1] > 0.f) M = fmaxf(M, wp[0]);
    }
    float L = 0.f;
    for (int s = 0; s < splits; ++s) {
        const float* wp = ws + (s * nhr + hr) * (d + 2);
        if (wp[1] > 0.f) L += wp[1] * expf(wp[0] - M);
    }
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < splits; ++s) {
            const float* wp = ws + (s * nhr + hr) * (d + 2);
            if (wp[1] > 0.f) o += wp[2 + e] * expf(wp[0] - M);
        }
        const float v = L > 0.f ? o / L : NAN;
        a.out[hr * d + e] = v;
        if (a.part_o) a.part_o[hr * d + e] = L > 0.f ? v : 0.f;
    }
    if (threadIdx.x == 0) {
        if (a.part_m) { a.part_m[hr] = M; a.part_l[hr] = L; }
        if (!(L > 0.f)) atomicOr(status, 16);
    }
}

__global__ void lse_merge_kernel(const float* m, const float* l, const float* o, int n_shards,
                                 int n, int d, float* out) {
    const int i = blockIdx.x;
    float M = -INFINITY;
    for (int s = 0; s < n_shards; ++s)
        if (l[s * n + i] > 0.f) M = fmaxf(M, m[s * n + i]);
    float L = 0.f;
    for (int s = 0; s < n_shards; ++s)
        if (l[s * n + i] > 0.f) L += l[s * n + i] * expf(m[s * n + i] - M);
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < n_shards; ++s)
            if (l[s * n + i] > 0.f) acc += o[(static_cast<int64_t>(s) * n + i) * d + e] * l[s * n + i] * expf(m[s * n + i] - M);
        out[static_cast<int64_t>(i) * d + e] = L > 0.f ? acc / L : NAN;
    }
}

struct BsaPlan {
    int hc, nc, splits, tiles_per_split;
};

BsaPlan plan_bsa(const hp_bsa_args& a) {
    BsaPlan p{};
    const int g = a.n_q_heads / a.kv.n_kv;  // q-heads per kv head
    int hc = std::__gcd(g, a.heads_per_mask);
    hc = std::__gcd(hc, kMaxHC);  // 1, 2, 4 or 8
    const int half = a.kv.d / 2;
    p.nc = half <= 32 ? 1 : half <= 64 ? 2 : half <= 128 ? 4 : 8;
    if (p.nc > 2 && hc > 4) hc = 4;  // bound registers / shared memory
    p.hc = std::max(1, hc);
    const int tiles = std::max(1, (a.max_sel + kTile - 1) / kTile);
    const int64_t ctas_per_split = static_cast<int64_t>(a.n_rows) * (a.n_q_heads / p.hc);
    // aim for >= 4 waves of 148 SMs, but never split when the row x head grid is large
    int splits = 1;
    if (ctas_per_split < 4 * 148) splits = static_cast<int>(min64(tiles, (4 * 148 + ctas_per_split - 1) / ctas_per_split));
    splits = std::max(1, splits);
    p.tiles_per_split = (tiles + splits - 1) / splits;
    p.splits = (tiles + p.tiles_per_split - 1) / p.tiles_per_split;
    return p;
}

template <typename T, int NC, int HC, bool EXT>
cudaError_t launch_bsa(const hp_bsa_args& a, const BsaPlan& p, float* ws, int* status, cudaStream_t s) {
    dim3 grid(p.splits, a.n_rows, a.n_q_heads / HC);
    bsa_kernel<T, NC, HC, EXT><<<grid, kBsaThreads, 0, s>>>(a, p.splits, p.tiles_per_split, ws, status);
    return cudaGetLastError();
}

template <typename T, int NC, bool EXT>
cudaError_t launch_bsa_hc(const hp_bsa_args& a, const BsaPlan& p, float* ws, int* status, cudaStream_t s) {
    switch (p.hc) {
        case 1: return launch_bsa<T, NC, 1, EXT>(a, p, ws, status, s);
        case 2: return launch_bsa<T, NC, 2, EXT>(a, p, ws, status, s);
        case 4: return launch_bsa<T, NC, 4, EXT>(a, p, ws, status, s);
        default: return launch_bsa<T, NC, (NC <= 2 ? 8 : 4), EXT>(a, p, ws, status, s);
    }
}

template <typename T>
cudaError_t dispatch_bsa(const hp_bsa_args& a, const BsaPlan& p, float* ws, int* status, cudaStream_t s) {
    const bool ext = a.rope.extension != 0;
#define HP_NC(N) case N: return ext ? launch_bsa_hc<T, N, true>(a, p, ws, status, s) : launch_bsa_hc<T, N, false>(a, p, ws, status, s);
    switch (p.nc) {
        HP_NC(1) HP_NC(2) HP_NC(4) HP_NC(8)
    }
#undef HP_NC
    return cudaErrorInvalidValue;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" int hp_selected_indices(const int32_t* mask_list, const int32_t* mask_count,
                                   int64_t mask_stride, int32_t n_masks, int32_t n_rows,
                                   int32_t block_size, int64_t query_offset, int32_t sink_tokens,
                                   int32_t stream_tokens, int32_t* sel_list, int32_t* sel_count,
                                   int64_t sel_stride, void* stream) {
    if (block_size <= 0 || n_rows <= 0 || n_masks <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_selected_indices: bad geometry");
    const int n_mask_blocks = (n_rows + block_size - 1) / block_size;
    selected_kernel<<<n_masks * n_rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        mask_list, mask_count, mask_stride, n_rows, n_mask_blocks, block_size, query_offset,
        sink_tokens, stream_tokens, sel_list, sel_count, sel_stride);
    return hph::check_cuda(cudaGetLastError(), "selected_kernel");
}

extern "C" size_t hp_bsa_workspace_bytes(int32_t n_q_heads, int32_t n_rows, int32_t max_sel, int32_t d) {
    const int tiles = std::max(1, (max_sel + kTile - 1) / kTile);
    return align_up(static_cast<size_t>(tiles) * n_q_heads * n_rows * (d + 2) * 4, 256) + 256;
}

extern "C" int hp_bsa(const hp_bsa_args* ap, void* stream) {
    if (!ap) return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: null args");
    const hp_bsa_args& a = *ap;
    if (a.n_q_heads <= 0 || a.n_rows <= 0 || a.heads_per_mask <= 0 || a.kv.n_kv <= 0 ||
        a.n_q_heads % a.kv.n_kv != 0 || a.n_q_heads % a.heads_per_mask != 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: bad head geometry");
    if (a.kv.d <= 0 || a.kv.d % 2 || a.kv.d > 512)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: head_dim must be even and <= 512");
    if (a.kv.dtype != HP_F32 && a.kv.dtype != HP_BF16) return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: dtype");
    if (!a.q || !a.sel_list || !a.sel_count || !a.out || !a.kv.k_pool || !a.kv.v_pool)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: null pointer");
    if (a.max_sel <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "attention_row: empty selected set");
    if (a.rope.extension) {
        if (!a.rope.cos_tab || !a.rope.sin_tab) return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: rope table missing");
        const int64_t pmax = a.query_offset + a.n_rows - 1;
        if (pmax >= a.rope.rope_max)
            return hph::set_error(HP_OUT_OF_RANGE, "apply_rope: position %lld >= max_position %lld",
                                  static_cast<long long>(pmax), static_cast<long long>(a.rope.rope_max));
    }
    const BsaPlan p = plan_bsa(a);
    const size_t need = hp_bsa_workspace_bytes(a.n_q_heads, a.n_rows, a.max_sel, a.kv.d);
    if (!a.workspace || a.workspace_bytes < need)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_bsa: workspace too small (%zu < %zu)", a.workspace_bytes, need);
    float* ws = static_cast<float*>(a.workspace);
    int* status = reinterpret_cast<int*>(static_cast<char*>(a.workspace) + need - 256);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaError_t e = a.kv.dtype == HP_BF16 ? dispatch_bsa<bf16_t>(a, p, ws, status, s)
                                                : dispatch_bsa<float>(a, p, ws, status, s);
    if (int rc = hph::check_cuda(e, "bsa_kernel")) return rc;
    if (p.splits > 1) {
        bsa_combine_kernel<<<a.n_q_heads * a.n_rows, 128, 0, s>>>(a, p.splits, ws, status);
        return hph::check_cuda(cudaGetLastError(), "bsa_combine_kernel");
    }
    return HP_OK;
}

extern "C" int hp_lse_merge(const float* m, const float* l, const float* o, int32_t n_shards,
                            int32_t n, int32_t d, float* out, void* stream) {
    if (n_shards <= 0 || n <= 0 || d <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "hp_lse_merge: bad shape");
    lse_merge_kernel<<<n, 128, 0, static_cast<cudaStream_t>(stream)>>>(m, l, o, n_shards, n, d, out);
    return hph::check_cuda(cudaGetLastError(), "lse_merge_kernel");
}

// Device helpers shared by the fused decode kernels (decode.cu, layer.cu):
// list-chain resolution, the exact sequential dots, row staging, cluster / DSMEM.
// Reference semantics as stated in decode.cu.
#pragma once

#include "common.cuh"

namespace hpk {
namespace dec {

constexpr int kD = 128;

__device__ __forceinline__ int64_t ref_token(const hp_list_ref& L, int mask, int64_t pos) {
#pragma unroll 1
    for (int i = L.depth - 1; i >= 0; --i) {
        const uint32_t lc = static_cast<uint32_t>(L.lc[i]);
        const uint32_t p32 = static_cast<uint32_t>(pos);  // list positions < 2^31
        const uint32_t r = p32 / lc;
        pos = static_cast<int64_t>(L.sel[i][static_cast<int64_t>(mask) * L.sel_stride[i] + r]) * lc + (p32 - r * lc);
    }
    return L.base_list ? static_cast<int64_t>(L.base_list[mask * L.base_stride + pos]) : L.range_start + pos;
}

// ----------------------------------------------------------------------------- dots
// Sequential fp32 dot of q (shared, broadcast) with the lane's staged row. A row's
// 16-byte chunk c sits at slot c ^ swz (swz = row & (chunks - 1)): the lanes of a
// quarter-warp LDS.128 phase then hit distinct bank groups with no padding.
template <typename T>
__device__ __forceinline__ float dot_row(const unsigned char* row, int swz, const float* q);

template <>
__device__ __forceinline__ float dot_row<bf16_t>(const unsigned char* row, int swz, const float* q) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
        const uint4 w = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
        const float4 qa = q4[2 * c], qb = q4[2 * c + 1];
        acc = __fadd_rn(acc, __fmul_rn(qa.x, bf16_lo(w.x)));
        acc = __fadd_rn(acc, __fmul_rn(qa.y, bf16_hi(w.x)));
        acc = __fadd_rn(acc, __fmul_rn(qa.z, bf16_lo(w.y)));
        acc = __fadd_rn(acc, __fmul_rn(qa.w, bf16_hi(w.y)));
        acc = __fadd_rn(acc, __fmul_rn(qb.x, bf16_lo(w.z)));
        acc = __fadd_rn(acc, __fmul_rn(qb.y, bf16_hi(w.z)));
        acc = __fadd_rn(acc, __fmul_rn(qb.z, bf16_lo(w.w)));
        acc = __fadd_rn(acc, __fmul_rn(qb.w, bf16_hi(w.w)));
    }
    return acc;
}

template <>
__device__ __forceinline__ float dot_row<float>(const unsigned char* row, int swz, const float* q) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
        const float4 w = *reinterpret_cast<const float4*>(row + ((c ^ swz) << 4));
        const float4 qa = q4[c];
        acc = __fadd_rn(acc, __fmul_rn(qa.x, w.x));
        acc = __fadd_rn(acc, __fmul_rn(qa.y, w.y));
        acc = __fadd_rn(acc, __fmul_rn(qa.z, w.z));
        acc = __fadd_rn(acc, __fmul_rn(qa.w, w.w));
    }
    return acc;
}

// Same dot when every product q[i]*k[i] is exact in fp32 (q and k bf16 with |x| in
// [2^-63, 2^63] or 0): fma(q, k, acc) then rounds once, exactly like the reference's
// acc + (q*k). fma.rn.f32.bf16 (SASS FHFMA.BF16) takes both operands as bf16 halves,
// so one instruction per element and no unpacking; qb holds q as packed bf16 pairs.
__device__ __forceinline__ float dot_row_bf16x(const unsigned char* row, int swz, const uint32_t* qb) {
    const uint4* q4 = reinterpret_cast<const uint4*>(qb);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
        const uint4 w = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
        const uint4 q = q4[c];
        acc = fma_bf16(q.x, w.x, acc, false);
        acc = fma_bf16(q.x, w.x, acc, true);
        acc = fma_bf16(q.y, w.y, acc, false);
        acc = fma_bf16(q.y, w.y, acc, true);
        acc = fma_bf16(q.z, w.z, acc, false);
        acc = fma_bf16(q.z, w.z, acc, true);
        acc = fma_bf16(q.w, w.w, acc, false);
        acc = fma_bf16(q.w, w.w, acc, true);
    }
    return acc;
}


template <typename T>
__device__ __forceinline__ float elem(const unsigned char* row, int swz, int i) {
    constexpr int per = 16 / sizeof(T);
    const int c = i / per, o = i - c * per;
    return load_elem(reinterpret_cast<const T*>(row + ((c ^ swz) << 4)), o);
}

// Rotated dot: apply_rope_inplace (tensor.cpp:61-79) then the sequential dot, with
// x*c - y*s / x*s + y*c separately rounded.
template <typename T>
__device__ __forceinline__ float dot_row_rot(const unsigned char* row, int swz, const float* q,
                                             const float* cs, const float* sn) {
    float acc = 0.0f;
    constexpr int half = kD / 2;
#pragma unroll 2
    for (int i = 0; i < half; ++i) {
        const float x = elem<T>(row, swz, i), y = elem<T>(row, swz, i + half);
        const float r = __fsub_rn(__fmul_rn(x, __ldg(cs + i)), __fmul_rn(y, __ldg(sn + i)));
        acc = __fadd_rn(acc, __fmul_rn(q[i], r));
    }
#pragma unroll 2
    for (int i = 0; i < half; ++i) {
        const float x = elem<T>(row, swz, i), y = elem<T>(row, swz, i + half);
        const float r = __fadd_rn(__fmul_rn(x, __ldg(sn + i)), __fmul_rn(y, __ldg(cs + i)));
        acc = __fadd_rn(acc, __fmul_rn(q[half + i], r));
    }
    return acc;
}

// Both branches' rotated dots of one staged bf16 row in one pass (the same operations
// as dot_row_rot, element for element): 16-byte chunks c (x = elements 8c..8c+7) and
// c + 8 (y = their rotation partners) are unpacked once, the cos/sin of the two key
// positions come as float4 pairs (L1 broadcast), and the two accumulators advance in
// the reference's element order — first half (x*c - y*s), then second half (x*s + y*c).
// plain1: branch 1's key position is 0 (the relative policy, rope_policy.cpp:37-57) —
// cos 1 and sin 0 exactly in the table, so x*1 - y*0 == x and x*0 + y*1 == y (up to the
// sign of a zero, which no comparison sees) and branch 1 is the unrotated dot.
__device__ __forceinline__ void dot_row_rot2_bf16(const unsigned char* row, int swz, const float* q,
                                                  const float* cs1, const float* sn1, const float* cs2,
                                                  const float* sn2, bool same, float& out1, float& out2,
                                                  bool plain1 = false) {
    float a1 = 0.0f, a2 = 0.0f;
#pragma unroll
    for (int part = 0; part < 2; ++part) {  // 0: r_i = x c - y s (i < 64); 1: r = x s + y c
#pragma unroll 2
        for (int c = 0; c < 8; ++c) {
            const uint4 xv = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
            const uint4 yv = *reinterpret_cast<const uint4*>(row + (((c + 8) ^ swz) << 4));
            const float x[8] = {bf16_lo(xv.x), bf16_hi(xv.x), bf16_lo(xv.y), bf16_hi(xv.y),
                                bf16_lo(xv.z), bf16_hi(xv.z), bf16_lo(xv.w), bf16_hi(xv.w)};
            const float y[8] = {bf16_lo(yv.x), bf16_hi(yv.x), bf16_lo(yv.y), bf16_hi(yv.y),
                                bf16_lo(yv.z), bf16_hi(yv.z), bf16_lo(yv.w), bf16_hi(yv.w)};
            const float4 qa = *reinterpret_cast<const float4*>(q + part * 64 + 8 * c);
            const float4 qb = *reinterpret_cast<const float4*>(q + part * 64 + 8 * c + 4);
            const float qq[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
            if (plain1) {
#pragma unroll
                for (int e = 0; e < 8; ++e) a1 = __fadd_rn(a1, __fmul_rn(qq[e], part == 0 ? x[e] : y[e]));
            } else {
                const float4 c1a = __ldg(reinterpret_cast<const float4*>(cs1 + 8 * c));
                const float4 c1b = __ldg(reinterpret_cast<const float4*>(cs1 + 8 * c + 4));
                const float4 s1a = __ldg(reinterpret_cast<const float4*>(sn1 + 8 * c));
                const float4 s1b = __ldg(reinterpret_cast<const float4*>(sn1 + 8 * c + 4));
                const float cc1[8] = {c1a.x, c1a.y, c1a.z, c1a.w, c1b.x, c1b.y, c1b.z, c1b.w};
                const float ss1[8] = {s1a.x, s1a.y, s1a.z, s1a.w, s1b.x, s1b.y, s1b.z, s1b.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float r = part == 0 ? __fsub_rn(__fmul_rn(x[e], cc1[e]), __fmul_rn(y[e], ss1[e]))
                                              : __fadd_rn(__fmul_rn(x[e], ss1[e]), __fmul_rn(y[e], cc1[e]));
                    a1 = __fadd_rn(a1, __fmul_rn(qq[e], r));
                }
            }
            if (!same) {
                const float4 c2a = __ldg(reinterpret_cast<const float4*>(cs2 + 8 * c));
                const float4 c2b = __ldg(reinterpret_cast<const float4*>(cs2 + 8 * c + 4));
                const float4 s2a = __ldg(reinterpret_cast<const float4*>(sn2 + 8 * c));
                const float4 s2b = __ldg(reinterpret_cast<const float4*>(sn2 + 8 * c + 4));
                const float cc2[8] = {c2a.x, c2a.y, c2a.z, c2a.w, c2b.x, c2b.y, c2b.z, c2b.w};
                const float ss2[8] = {s2a.x, s2a.y, s2a.z, s2a.w, s2b.x, s2b.y, s2b.z, s2b.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float r = part == 0 ? __fsub_rn(__fmul_rn(x[e], cc2[e]), __fmul_rn(y[e], ss2[e]))
                                              : __fadd_rn(__fmul_rn(x[e], ss2[e]), __fmul_rn(y[e], cc2[e]));
                    a2 = __fadd_rn(a2, __fmul_rn(qq[e], r));
                }
            }
        }
    }
    out1 = a1;
    out2 = same ? a1 : a2;
}

// ------------------------------------------------------------------------ staging
template <typename T>
struct RowGeom {
    static constexpr int bytes = kD * sizeof(T);  // 256 or 512
    static constexpr int stride = bytes;          // XOR-swizzled chunks, no padding
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Gather one key row per active lane (tok >= 0) into its staging slot with 16-byte
// cp.async (LDGSTS): the warp walks its 32 rows, a 256 B row per 16 lanes per
// instruction, so every instruction moves 512 contiguous-by-row bytes. (One
// cp.async.bulk per lane was measured at 2.3x the step latency of this on B200:
// 1.22 vs 0.52 us per 32-row gather.) Rows of the mapped host tier are read the
// same way. Optionally warms L2 with the lane's two possible next-step rows
// (pf0/pf1, -1 = none): the descent direction is unknown until the compare, but
// both candidates are (latency-bound stages only). Whole warp must call.
template <typename T, bool WAIT = true>
__device__ __forceinline__ void stage_rows(const hp_kv_view& kv, int kvh, int64_t tok,
                                           unsigned char* wstage, int lane, int64_t pf0 = -1,
                                           int64_t pf1 = -1) {
    using G = RowGeom<T>;
    constexpr int chunks = G::bytes / 16;          // 16 (bf16) or 32 (fp32)
    constexpr int rows_per_instr = 32 / chunks;    // 2 or 1
    const char* p = tok >= 0 ? kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, tok, sizeof(T)) : nullptr;
    const unsigned long long pu = reinterpret_cast<unsigned long long>(p);
    const int c = lane % chunks, sub = lane / chunks;
#pragma unroll
    for (int r = 0; r < 32; r += rows_per_instr) {
        const int row = r + sub;
        const unsigned long long pp = __shfl_sync(0xffffffffu, pu, row);
        if (pp) cp_async16(wstage + row * G::stride + ((c ^ (row & (chunks - 1))) << 4),
                           reinterpret_cast<const char*>(pp) + (c << 4));
    }
    if (pf0 >= 0) {
        const char* q0 = kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, pf0, sizeof(T));
#pragma unroll
        for (int o = 0; o < G::bytes; o += 128) prefetch_l2(q0 + o);
    }
    if (pf1 >= 0) {
        const char* q1 = kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, pf1, sizeof(T));
#pragma unroll
        for (int o = 0; o < G::bytes; o += 128) prefetch_l2(q1 + o);
    }
    if constexpr (WAIT) {
        cp_async_wait_all();
        __syncwarp();
    }
}


// ---- lookahead descent helpers (decode_stage_look_kernel, hp_decode_layer)
constexpr int kLookSlots = 3;

__device__ __forceinline__ void dot3_bf16x(const unsigned char* r0, const unsigned char* r1, const unsigned char* r2,
                                           int swz, const uint32_t* qb, float& d0, float& d1, float& d2) {
    const uint4* q4 = reinterpret_cast<const uint4*>(qb);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll 2
    for (int c = 0; c < 16; ++c) {
        const int o = (c ^ swz) << 4;
        const uint4 q = q4[c];
        const uint4 x = *reinterpret_cast<const uint4*>(r0 + o);
        const uint4 y = *reinterpret_cast<const uint4*>(r1 + o);
        const uint4 z = *reinterpret_cast<const uint4*>(r2 + o);
        a0 = fma_bf16(q.x, x.x, a0, false); a1 = fma_bf16(q.x, y.x, a1, false); a2 = fma_bf16(q.x, z.x, a2, false);
        a0 = fma_bf16(q.x, x.x, a0, true);  a1 = fma_bf16(q.x, y.x, a1, true);  a2 = fma_bf16(q.x, z.x, a2, true);
        a0 = fma_bf16(q.y, x.y, a0, false); a1 = fma_bf16(q.y, y.y, a1, false); a2 = fma_bf16(q.y, z.y, a2, false);
        a0 = fma_bf16(q.y, x.y, a0, true);  a1 = fma_bf16(q.y, y.y, a1, true);  a2 = fma_bf16(q.y, z.y, a2, true);
        a0 = fma_bf16(q.z, x.z, a0, false); a1 = fma_bf16(q.z, y.z, a1, false); a2 = fma_bf16(q.z, z.z, a2, false);
        a0 = fma_bf16(q.z, x.z, a0, true);  a1 = fma_bf16(q.z, y.z, a1, true);  a2 = fma_bf16(q.z, z.z, a2, true);
        a0 = fma_bf16(q.w, x.w, a0, false); a1 = fma_bf16(q.w, y.w, a1, false); a2 = fma_bf16(q.w, z.w, a2, false);
        a0 = fma_bf16(q.w, x.w, a0, true);  a1 = fma_bf16(q.w, y.w, a1, true);  a2 = fma_bf16(q.w, z.w, a2, true);
    }
    d0 = a0; d1 = a1; d2 = a2;
}

// up to three rows per lane (tok < 0 = none) into slots s * 32 + lane; whole warp calls
template <bool WAIT = true>
__device__ __forceinline__ void stage_rows3(const hp_kv_view& kv, int kvh, int64_t t0, int64_t t1, int64_t t2,
                                            unsigned char* wstage, int lane) {
    using G = RowGeom<bf16_t>;
    constexpr int chunks = G::bytes / 16;
    constexpr int rows_per_instr = 32 / chunks;
    const int c = lane % chunks, sub = lane / chunks;
    const int64_t tk[kLookSlots] = {t0, t1, t2};
#pragma unroll
    for (int sl = 0; sl < kLookSlots; ++sl) {
        const char* p = tk[sl] >= 0 ? kv_row_ptr(kv, kv.k_pool, kv.k_host, kvh, tk[sl], 2) : nullptr;
        const unsigned long long pu = reinterpret_cast<unsigned long long>(p);
        unsigned char* base = wstage + static_cast<size_t>(sl) * 32 * G::stride;
#pragma unroll
        for (int r = 0; r < 32; r += rows_per_instr) {
            const int row = r + sub;
            const unsigned long long pp = __shfl_sync(0xffffffffu, pu, row);
            if (pp) cp_async16(base + row * G::stride + ((c ^ (row & (chunks - 1))) << 4),
                               reinterpret_cast<const char*>(pp) + (c << 4));
        }
    }
    if constexpr (WAIT) {
        cp_async_wait_all();
        __syncwarp();
    }
}


// thread-block cluster / distributed shared memory (sm_90+)
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, unsigned rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_dsmem_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}


}  // namespace dec
}  // namespace hpk

// Shared device helpers for the hipprune_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hipprune_b200.h"

namespace hpk {

constexpr int kWarp = 32;

// The warp index as a value the compiler can see is warp-uniform (a shuffle from lane
// 0). Branching on threadIdx.x >> 5 directly makes the compiler treat the branch as
// possibly divergent inside a warp and turn every shuffle after it into a
// WARPSYNC.COLLECTIVE emulation loop.
__device__ __forceinline__ int warp_id() { return __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0); }

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// ---- element access ---------------------------------------------------------
// bf16 -> fp32 is exact (bit shift); every K/V element enters the fp32 arithmetic
// with the value the reference sees after the same bf16 rounding of its inputs.
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T> struct Elem;
template <> struct Elem<float> { static constexpr int bytes = 4; static constexpr int id = HP_F32; };
struct bf16_t { uint16_t bits; };
template <> struct Elem<bf16_t> { static constexpr int bytes = 2; static constexpr int id = HP_BF16; };

__device__ __forceinline__ float load_elem(const float* p, int i) { return p[i]; }
__device__ __forceinline__ float load_elem(const bf16_t* p, int i) {
    return __uint_as_float(static_cast<uint32_t>(p[i].bits) << 16);
}

// ---- paged KV resolution (KvView::key_row, kv_store.cpp:160-163) ------------------
// page = token / page_size covers all kv heads of the layer (kv_store.cpp:50-56).
// Non-resident pages (slot < 0) resolve to the device-mapped host tier: the read is
// served over the host link and recorded as a miss for the step-end commit.
__device__ __forceinline__ const char* kv_row_ptr(const hp_kv_view& v, const void* pool,
                                                  const void* host, int kv, int64_t tok,
                                                  int elem_bytes) {
    // tokens < 2^31: 32-bit page split (a shift when page_size is a power of two)
    const uint32_t t32 = static_cast<uint32_t>(tok);
    const uint32_t ps = static_cast<uint32_t>(v.page_size);
    const int64_t page = (ps & (ps - 1)) == 0 ? (t32 >> (__ffs(ps) - 1)) : t32 / ps;
    const int64_t off = t32 - static_cast<uint32_t>(page) * ps;
    int64_t slot = v.page_table ? static_cast<int64_t>(v.page_table[page]) : page;
    const bool hit = slot >= 0;
    if (v.row_bits != nullptr && pool == v.k_pool) {
        const int64_t bit = kv * v.row_bits_stride + tok;
        atomicOr(v.row_bits + (bit >> 5), 1u << (bit & 31));
    }
    if (v.touched) {
        const uint8_t flag = hit ? 1 : 2;
        if (v.touched[page] != flag) v.touched[page] = flag;
    }
    if (hit) {
        return static_cast<const char*>(pool) +
               (((slot * v.n_kv + kv) * v.page_size + off) * v.d) * elem_bytes;
    }
    return static_cast<const char*>(host) +
           (((page * v.n_kv + kv) * v.page_size + off) * v.d) * elem_bytes;
}

// ---- RoPE policy (rope_policy.cpp:18-57) -----------------------------------------
__device__ __forceinline__ int pruning_policy(const hp_rope_ctx& r) {
    return r.layer > r.early_cutoff ? r.late_policy : r.early_policy;
}
__device__ __forceinline__ int64_t rope_q_position(const hp_rope_ctx& r, int64_t qpos,
                                                   int64_t stream, int64_t chunk_count) {
    if (pruning_policy(r) == HP_ROPE_RELATIVE) return stream + 1;
    const int64_t cap = chunk_count + stream;  // ChunkIndexed
    return qpos < cap ? qpos : cap;
}
__device__ __forceinline__ int64_t rope_k_position(const hp_rope_ctx& r, int branch,
                                                   int64_t chunk_index) {
    if (pruning_policy(r) == HP_ROPE_RELATIVE) return branch - 1;
    return chunk_index;
}

// ---- ordered keys for top-k --------------------------------------------------------
// Monotone map float -> uint32 (ascending). -0.0 is folded onto +0.0 so that equal
// scores compare equal exactly as the reference's operator> does (pruning.cpp:189-190).
__device__ __forceinline__ uint32_t order_key(float s) {
    if (s == 0.0f) s = 0.0f;
    const uint32_t u = __float_as_uint(s);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ---- block scans ---------------------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ int block_exclusive_scan(int v, int* smem_warp, int* total) {
    static_assert(kThreads % kWarp == 0 && kThreads <= 1024, "block size");
    constexpr int kWarps = kThreads / kWarp;
    const int lane = threadIdx.x & 31, w = warp_id();
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = lane < kWarps ? smem_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kWarps) smem_warp[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const int base = w ? smem_warp[w - 1] : 0;
    *total = smem_warp[kWarps - 1];
    __syncthreads();
    return base + x - v;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---- mbarrier + 1-D bulk copies (the TMA engine's non-tensor path) -------------------
// A row gather is one cp.async.bulk per row (256 B bf16 / 512 B fp32): the copy engine
// moves it global -> shared and signals completion as transaction bytes on an mbarrier,
// so a CTA can put all of its rows in flight with one instruction each and a single wait.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Row pointer plus residency (true = device slot; false = the mapped host tier, which
// the bulk copy engine does not read: such rows are copied with plain loads).
__device__ __forceinline__ bool kv_row_resident(const hp_kv_view& v, int64_t tok) {
    if (!v.page_table) return true;
    const uint32_t ps = static_cast<uint32_t>(v.page_size);
    const uint32_t page = static_cast<uint32_t>(tok) / ps;
    return v.page_table[page] >= 0;
}

// ---- programmatic dependent launch --------------------------------------------------
// Every decode kernel is launched with programmatic stream serialization: it lets its
// dependent grid launch as soon as all of its CTAs are running (launch_dependents at
// the top), and waits for its own predecessor's completion and memory (wait) before
// touching anything that predecessor wrote. The next kernel's launch and CTA
// rasterisation then overlap this kernel's tail instead of following it.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- exact-product dot helpers ---------------------------------------------------
// fma(q, k, acc) rounds once, exactly like the reference's acc + (q*k) when the product
// q*k is exact in fp32 (q and k bf16 with |x| in [2^-63, 2^63] or 0). fma.rn.f32.bf16
// (SASS FHFMA.BF16) takes both operands as bf16 halves of packed pairs.
__device__ __forceinline__ float fma_bf16(uint32_t a, uint32_t b, float c, bool hi) {
    float d;
    const uint16_t ah = static_cast<uint16_t>(hi ? a >> 16 : a & 0xffffu);
    const uint16_t bh = static_cast<uint16_t>(hi ? b >> 16 : b & 0xffffu);
    asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(ah), "h"(bh), "f"(c));
    return d;
}

// q is bf16-exact with |q| in [2^-63, 2^63] or 0 (so bf16 products stay exact).
__device__ __forceinline__ bool q_product_safe(float x) {
    const uint32_t u = __float_as_uint(x);
    if ((u & 0xffffu) != 0u) return false;
    const float ax = fabsf(x);
    return ax == 0.0f || (ax >= 1.0842022e-19f && ax <= 9.2233720e18f);
}

// ---- last-CTA ticket ---------------------------------------------------------------
// Called by all threads after the CTA's global writes. One thread takes the ticket
// with a gpu-scope acq_rel atomic: release publishes every write the CTA made
// before the barrier (PTX memory-model cumulativity through bar.sync), acquire
// orders the last CTA's later reads after all other CTAs' writes. One fence per
// CTA instead of a MEMBAR.GPU (+ L1 invalidate) in every thread. The last CTA
// resets the counter for the next launch / graph replay.
__device__ __forceinline__ bool cta_ticket_last(int* counter, int total, int* sh_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
        const bool last = prev == total - 1;
        if (last) *counter = 0;
        *sh_flag = last;
    }
    __syncthreads();
    return *sh_flag != 0;
}

// ---- phase tracer (off unless hp_trace_enable set a buffer) ------------------------
// Per-CTA %globaltimer stamps at named checkpoints of one kernel id, 8 slots per CTA.
// internal linkage: each translation unit that traces exports its own enable call
static __device__ unsigned long long* g_trace_buf = nullptr;
static __device__ int g_trace_kernel = -1;
static __device__ int g_cut_kernel = -1;  // dev build: early exit of kernel id at cut point
static __device__ int g_cut_at = -1;
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Phase-cut experiments (dev build only): returns true when kernel `kernel_id` should
// stop at cut point `at`, to time a kernel's prefix in isolation.
// Load once per kernel (dev_cut_point) and compare in registers: a global load per
// check would itself add a memory round trip at every cut point.
__device__ __forceinline__ int dev_cut_point(int kernel_id) {
#ifdef HP_TRACE
    return g_cut_kernel == kernel_id ? g_cut_at : -1;
#else
    (void)kernel_id;
    return -1;
#endif
}

// Compiled in only with -DHP_TRACE (the dev build `HP_TRACE=1 python -m
// paper_2502_08910_b200.build`): the enable check is a global load per call site.
__device__ __forceinline__ void trace(int kernel_id, int slot) {
#if !defined(HP_TRACE) || defined(HP_CUTS_ONLY)
    (void)kernel_id;
    (void)slot;
    return;
#endif
    unsigned long long* b = g_trace_buf;
    if (b != nullptr && g_trace_kernel == kernel_id && threadIdx.x == 0) {
        const unsigned cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        b[cta * 8 + slot] = globaltimer();
        b[(8192 + cta) * 8 + slot] = clock64();  // SM cycles at the same point
    }
}

}  // namespace hpk

// host-side error plumbing shared by the C-ABI translation units
namespace hph {
int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
}  // namespace hph

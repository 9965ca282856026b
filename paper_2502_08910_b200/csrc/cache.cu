// On-GPU LRU page cache over a pinned host tier (north-star item 3; replaces
// TieredKvStore::access_pages / commit + KvView::account, reference
// proj/src/kv_store.cpp:58-120,188-200).
//
// Residency is a page table (page -> slot, -1 = host only). The gathers of the
// pruning stages and the BSA resolve every row through it (common.cuh kv_row_ptr):
// a resident page is read from its device slot, a missing one straight from the
// device-mapped pinned host tier inside the same kernel (the miss is served in the
// pass that needs it, no fault/refetch round trip), and each page is flagged in
// `touched` (1 hit, 2 miss) — the KvView page accounting. hp_cache_commit is the
// step-end commit (decode.cpp:279-280): hit pages take the step's logical stamp;
// missing pages are installed into the least-recently-used slots (oldest stamp,
// lower slot first; free slots have stamp 0), each page copied host -> slot with
// 16-byte loads over the host link by a grid-wide copy kernel. Like the reference's
// commit_rolling (decode.cpp:13-20), a miss list longer than the cache leaves its
// last `num_slots` pages resident.
#include <algorithm>

#include "common.cuh"
#include "topk.cuh"

using namespace hpk;

namespace {

constexpr int kCommitThreads = 1024;
constexpr int kMaxCacheSlots = 16384;  // victim selection runs in one CTA's shared memory

struct CommitWs {
    uint32_t* clock;     // [1] device step clock (stamp 0 = auto: advance and use it)
    int32_t* miss;       // [num_pages] missing pages, ascending
    int32_t* copy_page;  // [num_slots] (page, slot) pairs to fill
    int32_t* copy_slot;
    int32_t* n_copy;     // [1]
};

__global__ void __launch_bounds__(kCommitThreads) commit_select_kernel(const hp_page_cache c, uint32_t stamp,
                                                                          CommitWs w, int32_t* stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TopkShared sh;
    __shared__ int sh_hits, sh_miss;
    const int t = threadIdx.x, nt = blockDim.x;
    if (stamp == 0) {  // graph-replayable: the step clock lives on the device
        __shared__ uint32_t sh_stamp;
        __syncthreads();
        if (t == 0) sh_stamp = ++(*w.clock) + 1;  // 1 is the warm-start stamp
        __syncthreads();
        stamp = sh_stamp;
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);             // [num_slots]
    int32_t* vict = reinterpret_cast<int32_t*>(keys + kMaxCacheSlots);  // [num_slots]
    if (t == 0) { sh_hits = 0; sh_miss = 0; }
    __syncthreads();
    // 1. hits take the step stamp; misses are compacted in page order
    const int per = (c.num_pages + nt - 1) / nt;
    const int p0 = min(c.num_pages, t * per), p1 = min(c.num_pages, p0 + per);
    int nmiss = 0, nhit = 0;
    for (int p = p0; p < p1; ++p) {
        const uint8_t f = c.touched[p];
        if (f == 1) {
            const int32_t s = c.page_table[p];
            if (s >= 0) c.slot_stamp[s] = stamp;
            ++nhit;
        } else if (f == 2) {
            ++nmiss;
        }
    }
    int r = block_scan_rt(nmiss, sh.scan);
    for (int p = p0; p < p1; ++p)
        if (c.touched[p] == 2) w.miss[r++] = p;
    atomicAdd(&sh_hits, nhit);
    atomicAdd(&sh_miss, nmiss);
    __syncthreads();
    const int M = sh_miss;
    const int V = min(M, c.num_slots);
    // 2. the V least-recently-used slots: largest ~stamp, ties to the lower slot
    for (int s = t; s < c.num_slots; s += nt) keys[s] = ~c.slot_stamp[s];
    __syncthreads();
    if (V > 0) cta_topk_smem(keys, c.num_slots, V, vict, sh);
    // 3. pair the last V misses with the victims; update the tables
    int evict = 0;
    for (int i = t; i < V; i += nt) {
        const int32_t page = w.miss[M - V + i];
        const int32_t slot = vict[i];
        const int32_t old = c.slot_page[slot];
        if (old >= 0) {
            c.page_table[old] = -1;
            ++evict;
        }
        c.page_table[page] = slot;
        c.slot_page[slot] = page;
        c.slot_stamp[slot] = stamp;
        w.copy_page[i] = page;
        w.copy_slot[i] = slot;
    }
    __syncthreads();
    for (int p = t; p < c.num_pages; p += nt) c.touched[p] = 0;
    evict = __reduce_add_sync(0xffffffffu, evict);
    if ((t & 31) == 0 && evict) atomicAdd(&stats[2], evict);
    if (t == 0) {
        *w.n_copy = V;
        atomicAdd(&stats[0], sh_hits);
        atomicAdd(&stats[1], M);
    }
}

// host tier -> slot for every (page, slot) pair: a page is n_kv * page_size rows of K
// (and V), contiguous in both layouts, moved as 16-byte words
__global__ void commit_copy_kernel(const hp_page_cache c, CommitWs w) {
    const int n = *w.n_copy;
    const int64_t eb = c.dtype == HP_BF16 ? 2 : 4;
    const int64_t words = static_cast<int64_t>(c.n_kv) * c.page_size * c.d * eb / 16;
    const int64_t total = static_cast<int64_t>(n) * words;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = i / words, o = i - e * words;
        const int64_t page = w.copy_page[e], slot = w.copy_slot[e];
        reinterpret_cast<uint4*>(c.k_slots)[slot * words + o] = reinterpret_cast<const uint4*>(c.k_host)[page * words + o];
        if (c.v_slots)
            reinterpret_cast<uint4*>(c.v_slots)[slot * words + o] = reinterpret_cast<const uint4*>(c.v_host)[page * words + o];
    }
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" size_t hp_cache_workspace_bytes(int32_t num_pages, int32_t num_slots) {
    return 256 + align_up(static_cast<size_t>(num_pages) * 4, 256) + 2 * align_up(static_cast<size_t>(num_slots) * 4, 256) + 256;
}

extern "C" int hp_cache_commit(const hp_page_cache* cp, uint32_t stamp, int32_t* stats, void* workspace,
                               size_t workspace_bytes, void* stream) {
    if (!cp) return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: null cache");
    const hp_page_cache& c = *cp;
    if (c.num_pages <= 0 || c.num_slots <= 0 || c.page_size <= 0 || c.n_kv <= 0 || c.d <= 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: bad geometry");
    if (c.num_slots > kMaxCacheSlots)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: %d slots exceed the %d-slot limit", c.num_slots,
                              kMaxCacheSlots);
    if (!c.k_slots || !c.k_host || !c.page_table || !c.slot_page || !c.slot_stamp || !c.touched || !stats)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: null pointer");
    if ((static_cast<int64_t>(c.n_kv) * c.page_size * c.d * (c.dtype == HP_BF16 ? 2 : 4)) % 16)
        return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: page bytes must be a multiple of 16");
    const size_t need = hp_cache_workspace_bytes(c.num_pages, c.num_slots);
    if (!workspace || workspace_bytes < need) return hph::set_error(HP_INVALID_ARGUMENT, "hp_cache_commit: workspace too small");
    char* ws = static_cast<char*>(workspace);
    CommitWs w;
    w.clock = reinterpret_cast<uint32_t*>(ws);
    w.miss = reinterpret_cast<int32_t*>(ws + 256);
    size_t off = 256 + align_up(static_cast<size_t>(c.num_pages) * 4, 256);
    w.copy_page = reinterpret_cast<int32_t*>(ws + off);
    off += align_up(static_cast<size_t>(c.num_slots) * 4, 256);
    w.copy_slot = reinterpret_cast<int32_t*>(ws + off);
    off += align_up(static_cast<size_t>(c.num_slots) * 4, 256);
    w.n_copy = reinterpret_cast<int32_t*>(ws + off);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t smem = static_cast<size_t>(kMaxCacheSlots) * 8;
    cudaError_t e = cudaFuncSetAttribute(commit_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return hph::check_cuda(e, "commit_select_kernel");
    commit_select_kernel<<<1, kCommitThreads, smem, s>>>(c, stamp, w, stats);
    if ((e = cudaGetLastError()) != cudaSuccess) return hph::check_cuda(e, "commit_select_kernel");
    commit_copy_kernel<<<148 * 4, 256, 0, s>>>(c, w);
    return hph::check_cuda(cudaGetLastError(), "commit_copy_kernel");
}

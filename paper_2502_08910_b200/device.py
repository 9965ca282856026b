"""Device-side orchestration of the hot path over the C ABI.

torch is used only for device memory and streams; every byte of compute runs
in the sm_100a kernels of ``_lib/libhipprune_b200.so``. There is no CPU path:
without the library or a CUDA device the calls raise.

Mapping to the reference (paths relative to /root/reference/proj):
  PagedKV              KeySource / KvView over a paged layer (key_source.hpp:13-18,
                       kv_store.cpp:50-56,160-200) — pages of `page_size` tokens
                       covering all kv heads, pool layout [slot][n_kv][page][d]
  RopeTable            build_rope_table (tensor.cpp:30-59), uploaded
  build_mask           build_mask (pruning.cpp:202-313)
  prune_stage          run_pruning_stage (pruning.cpp:153-200)
  selected_indices     selected_indices (sparse_attention.cpp:95-112)
  bsa                  attention_row / block_sparse_attention (sparse_attention.cpp:33-145)
  DecodeLayer          the per-layer body of DecodeEngine::step (decode.cpp:225-273)
"""
from __future__ import annotations

import collections
import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from ._capi import BsaArgs, KvView, RopeCtx, StageArgs, check, lib

_DT = {torch.float32: _capi.HP_F32, torch.bfloat16: _capi.HP_BF16}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda() -> None:
    lib()
    if not torch.cuda.is_available() or not lib().hp_device_available():
        raise RuntimeError("hipprune_b200: no CUDA device — the B200 path has no CPU fallback")


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


# ----------------------------------------------------------------------------- KV
class PagedKV:
    """Paged K/V of one layer resident in HBM (identity page table) or cached.

    k, v: [n_kv, T, d] tensors. Pool layout [num_slots][n_kv][page_size][d].
    ``capacity`` (tokens) reserves pages for decode appends.
    """

    def __init__(self, k: torch.Tensor, v: torch.Tensor | None, *, page_size: int = 64,
                 dtype: torch.dtype = torch.bfloat16, capacity: int | None = None,
                 device="cuda"):
        assert k.dim() == 3
        self.n_kv, t, self.d = k.shape
        self.page_size = page_size
        self.dtype = dtype
        self.t_kv = t
        cap = max(capacity or t, t)
        self.num_pages = ceil_div(cap, page_size)
        self.k_pool = self._pack(k, device)
        self.v_pool = self._pack(v, device) if v is not None else None
        self.page_table = None
        self.touched = None
        self.row_bits = None
        # device flag: every key is bf16 with |k| in [2^-63, 2^63] or 0, so bf16 q*k
        # products are exact in fp32 (lets the fused stage issue FFMA, see decode.cu)
        self.keys_exact = torch.zeros(1, dtype=torch.int32, device=device)
        if dtype == torch.bfloat16:
            self.keys_exact.fill_(int(self._products_safe(self.k_pool)))

    @staticmethod
    def _products_safe(x: torch.Tensor) -> bool:
        a = x.float().abs()
        return bool(((a == 0) | ((a >= 2.0 ** -63) & (a <= 2.0 ** 63))).all())

    def _pack(self, x: torch.Tensor, device) -> torch.Tensor:
        n_kv, t, d = x.shape
        ps = self.page_size
        pool = torch.zeros(self.num_pages, n_kv, ps, d, dtype=self.dtype, device=device)
        full = t // ps
        xd = x.to(device=device, dtype=self.dtype)
        if full:
            pool[:full].copy_(xd[:, : full * ps].reshape(n_kv, full, ps, d).permute(1, 0, 2, 3))
        rem = t - full * ps
        if rem:
            pool[full, :, :rem].copy_(xd[:, full * ps:])
        return pool

    def append(self, k_row: torch.Tensor, v_row: torch.Tensor | None = None) -> None:
        """Append one token's K/V rows [n_kv, d] (DecodeEngine::step, decode.cpp:202-208)."""
        t = self.t_kv
        page, off = divmod(t, self.page_size)
        if page >= self.num_pages:
            raise IndexError("PagedKV: capacity exhausted")
        self.k_pool[page, :, off].copy_(k_row)
        if self.dtype == torch.bfloat16:
            a = self.k_pool[page, :, off].float().abs()
            ok = ((a == 0) | ((a >= 2.0 ** -63) & (a <= 2.0 ** 63))).all().to(torch.int32)
            self.keys_exact.mul_(ok)
        if v_row is not None and self.v_pool is not None:
            self.v_pool[page, :, off].copy_(v_row)
        self.t_kv = t + 1

    def view(self, t_kv: int | None = None) -> KvView:
        return KvView(k_pool=_ptr(self.k_pool), v_pool=_ptr(self.v_pool), k_host=None,
                      v_host=None, page_table=_ptr(self.page_table), touched=_ptr(self.touched),
                      num_pages=self.num_pages, page_size=self.page_size, n_kv=self.n_kv,
                      d=self.d, dtype=_DT[self.dtype], t_kv=t_kv if t_kv is not None else self.t_kv,
                      row_bits=_ptr(self.row_bits),
                      row_bits_stride=self.num_pages * self.page_size)

    def count_rows(self, enable: bool = True) -> None:
        """Instrumentation: record every distinct key row read (see hp_kv_view.row_bits)."""
        if enable:
            nbits = self.n_kv * self.num_pages * self.page_size
            self.row_bits = torch.zeros((nbits + 31) // 32, dtype=torch.int32, device=self.k_pool.device)
        else:
            self.row_bits = None

    def distinct_rows(self) -> int:
        b = self.row_bits
        if b is None:
            return 0
        x = b.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        cnt = torch.zeros_like(x)
        for s in range(32):
            cnt += (x >> s) & 1
        return int(cnt.sum())


# --------------------------------------------------------------------------- RoPE
class RopeTable:
    """build_rope_table (tensor.cpp:30-59) computed on the host in double and uploaded."""

    def __init__(self, max_pos: int, d: int, theta: float = 10000.0, device="cuda"):
        half = d // 2
        cos = np.empty((max_pos, half), np.float32)
        sin = np.empty((max_pos, half), np.float32)
        check(lib().hp_build_rope_table(max_pos, d, theta, cos.ctypes.data, sin.ctypes.data))
        self.max_pos, self.d = max_pos, d
        self.cos_host, self.sin_host = cos, sin
        self.cos = torch.from_numpy(cos).to(device)
        self.sin = torch.from_numpy(sin).to(device)


@dataclass
class RopePolicy:
    """RopePolicySet (rope_policy.hpp:24-34); pruning layer is 1-based."""
    extension: bool = False
    early_cutoff: int = 3
    early_policy: int = _capi.HP_ROPE_CHUNK_INDEXED
    late_policy: int = _capi.HP_ROPE_RELATIVE

    def ctx(self, layer1: int, table: RopeTable | None) -> RopeCtx:
        if self.extension and table is None:
            raise ValueError("RopePolicy: extension enabled without a rope table")
        return RopeCtx(cos_tab=_ptr(table.cos) if (table is not None and self.extension) else None,
                       sin_tab=_ptr(table.sin) if (table is not None and self.extension) else None,
                       rope_max=table.max_pos if table is not None else 0,
                       extension=int(self.extension), early_cutoff=self.early_cutoff,
                       early_policy=self.early_policy, late_policy=self.late_policy,
                       layer=layer1, pad_=0)


# ------------------------------------------------------------------------- stages
class Workspace:
    """Grow-only device scratch (allocated outside the hot path)."""

    def __init__(self, device="cuda"):
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.buf.device)
        return self.buf


def prune_stage(stage, q: torch.Tensor, kv: PagedKV, *, n_masks: int, n_blocks: int = 1,
                in_list: torch.Tensor | None = None, in_start: torch.Tensor | None = None,
                in_count: torch.Tensor, in_stride: int = 0, max_chunks: int,
                out_list: torch.Tensor, out_count: torch.Tensor, query_offset: int,
                stream_tokens: int, layer1: int, policy: RopePolicy, rope: RopeTable | None,
                ws: Workspace, stream=None) -> None:
    """One pruning stage over n_masks x n_blocks lists (run_pruning_stage, pruning.cpp:153-200)."""
    bq, lc, keep = stage
    hq, q_rows, _ = q.shape
    need = lib().hp_stage_workspace_bytes(n_masks * n_blocks, max(1, max_chunks), keep, lc)
    w = ws.get(need)
    a = StageArgs(query_block=bq, chunk_size=lc, keep=keep, n_masks=n_masks,
                  heads_per_mask=hq // n_masks, n_q_heads=hq, n_blocks=n_blocks, q_rows=q_rows,
                  q=_ptr(q), query_offset=query_offset, stream_tokens=stream_tokens,
                  max_chunks=max_chunks, in_list=_ptr(in_list), in_start=_ptr(in_start),
                  in_count=_ptr(in_count), in_stride=in_stride, out_list=_ptr(out_list),
                  out_count=_ptr(out_count), out_stride=out_list.shape[-1], workspace=_ptr(w),
                  workspace_bytes=w.numel(), keys=kv.view(), rope=policy.ctx(layer1, rope),
                  keys_exact=_ptr(getattr(kv, "keys_exact", None)))
    v = C.c_int32(-1)
    check(lib().hp_prune_stage_variant(C.byref(a), C.byref(v)))
    PRUNE_VARIANTS_USED.append(v.value)
    check(lib().hp_prune_stage(C.byref(a), C.c_void_p(_stream(stream))))


# descent kernel of the recent prune_stage calls (hp_prune_variant), for tests and tools
PRUNE_VARIANTS_USED: collections.deque = collections.deque(maxlen=1024)


def build_mask(q: torch.Tensor, kv: PagedKV, stages, *, sink: int, stream_tokens: int,
               t_kv: int | None = None, layer0: int = 0, policy: RopePolicy | None = None,
               rope: RopeTable | None = None, n_masks: int = 1, ws: Workspace | None = None,
               stream=None):
    """build_mask (pruning.cpp:202-313) on the device.

    q: fp32 [n_q_heads, T_q, d] on the device. Returns (lists [n_masks, n_blocks, keep],
    counts [n_masks, n_blocks], trace list of (list, count) per stage for the last block,
    block_size, query_offset).
    """
    require_cuda()
    policy = policy or RopePolicy()
    ws = ws or Workspace(q.device)
    hq, t_q, d = q.shape
    t_kv = kv.t_kv if t_kv is None else t_kv
    if t_q == 0 or t_q > t_kv:
        raise ValueError("build_mask: workload query length inconsistent")
    for bq, lc, keep in stages:
        if bq <= 0 or lc <= 0:
            raise ValueError("StageConfig: b_q and l_c must be >= 1")
        if keep <= 0 or keep % lc:
            raise ValueError("StageConfig: k must be a positive multiple of l_c")
    if not stages:
        raise ValueError("PruningPlan: no stages")
    for i in range(1, len(stages)):
        if stages[i][0] > stages[i - 1][0] or stages[i - 1][0] % stages[i][0]:
            raise ValueError("PruningPlan: successive b_q must be non-increasing and divisible")
        if stages[i][2] > stages[i - 1][2]:
            raise ValueError("PruningPlan: k must be non-increasing across stages")
    offset = t_kv - t_q
    dev = q.device
    bq = stages[0][0]
    nb = ceil_div(t_q, bq)
    starts = np.full((n_masks, nb), sink, np.int32)
    counts = np.zeros((n_masks, nb), np.int32)
    for m in range(nb):
        end = offset + min((m + 1) * bq, t_q)
        upper = end - stream_tokens if end > stream_tokens else 0
        counts[:, m] = max(0, upper - sink)
    in_start = torch.from_numpy(starts).to(dev)
    in_count = torch.from_numpy(counts).to(dev)
    in_list = None
    in_stride = 0
    max_in = int(counts.max()) if counts.size else 0
    trace = []
    rope_ctx_layer = layer0 + 1
    for si, (bq, lc, keep) in enumerate(stages):
        out_list = torch.empty((n_masks, nb, keep), dtype=torch.int32, device=dev)
        out_count = torch.empty((n_masks, nb), dtype=torch.int32, device=dev)
        prune_stage((bq, lc, keep), q, kv, n_masks=n_masks, n_blocks=nb, in_list=in_list,
                    in_start=in_start, in_count=in_count, in_stride=in_stride,
                    max_chunks=ceil_div(max_in, lc), out_list=out_list, out_count=out_count,
                    query_offset=offset, stream_tokens=stream_tokens, layer1=rope_ctx_layer,
                    policy=policy, rope=rope, ws=ws, stream=stream)
        trace.append((out_list[:, nb - 1], out_count[:, nb - 1]))
        in_list, in_count, in_start, in_stride = out_list, out_count, None, keep
        max_in = keep
        if si + 1 < len(stages) and stages[si + 1][0] != bq:
            bq_next = stages[si + 1][0]
            nb2 = ceil_div(t_q, bq_next)
            nl = torch.empty((n_masks, nb2, keep), dtype=torch.int32, device=dev)
            nc = torch.empty((n_masks, nb2), dtype=torch.int32, device=dev)
            check(lib().hp_remap_blocks(_ptr(out_list), _ptr(out_count), keep, n_masks, nb, bq,
                                        bq_next, t_q, offset, stream_tokens, _ptr(nl), _ptr(nc),
                                        keep, C.c_void_p(_stream(stream))))
            in_list, in_count, nb = nl, nc, nb2
    return in_list, in_count, trace, stages[-1][0], offset


def selected_indices(mask_list: torch.Tensor, mask_count: torch.Tensor, *, n_rows: int,
                     block_size: int, query_offset: int, sink: int, stream_tokens: int,
                     sel_stride: int | None = None, out=None, stream=None):
    """Per-row selected lists (selected_indices, sparse_attention.cpp:95-112)."""
    n_masks = mask_list.shape[0]
    cap = mask_list.shape[-1]
    sel_stride = sel_stride or (sink + cap + stream_tokens + 1)
    if out is None:
        sel = torch.empty((n_masks, n_rows, sel_stride), dtype=torch.int32, device=mask_list.device)
        cnt = torch.empty((n_masks, n_rows), dtype=torch.int32, device=mask_list.device)
    else:
        sel, cnt = out
    check(lib().hp_selected_indices(_ptr(mask_list), _ptr(mask_count), cap, n_masks, n_rows,
                                    block_size, query_offset, sink, stream_tokens, _ptr(sel),
                                    _ptr(cnt), sel.shape[-1], C.c_void_p(_stream(stream))))
    return sel, cnt


def bsa(q: torch.Tensor, kv: PagedKV, sel: torch.Tensor, sel_count: torch.Tensor, *,
        query_offset: int, max_sel: int, policy: RopePolicy | None = None,
        rope: RopeTable | None = None, out: torch.Tensor | None = None,
        partials=None, ws: Workspace | None = None, stream=None) -> torch.Tensor:
    """Split-K block-sparse attention over selected lists; q fp32 [n_q_heads, n_rows, d]."""
    policy = policy or RopePolicy()
    ws = ws or Workspace(q.device)
    hq, n_rows, d = q.shape
    n_masks = sel.shape[0]
    out = out if out is not None else torch.empty_like(q)
    need = lib().hp_bsa_workspace_bytes(hq, n_rows, max_sel, d)
    w = ws.get(need)
    pm, pl, po = partials if partials is not None else (None, None, None)
    a = BsaArgs(n_q_heads=hq, heads_per_mask=hq // n_masks, n_rows=n_rows, q=_ptr(q),
                query_offset=query_offset, sel_list=_ptr(sel), sel_count=_ptr(sel_count),
                sel_stride=sel.shape[-1], max_sel=max_sel, out=_ptr(out), part_m=_ptr(pm),
                part_l=_ptr(pl), part_o=_ptr(po), workspace=_ptr(w), workspace_bytes=w.numel(),
                kv=kv.view(), rope=policy.ctx(0, rope))
    check(lib().hp_bsa(C.byref(a), C.c_void_p(_stream(stream))))
    return out


def lse_merge(m: torch.Tensor, l: torch.Tensor, o: torch.Tensor, out: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """Merge per-shard (m, l, o) triples: m, l [S, n]; o [S, n, d] -> [n, d]."""
    s, n, d = o.shape
    out = out if out is not None else torch.empty((n, d), dtype=torch.float32, device=o.device)
    check(lib().hp_lse_merge(_ptr(m), _ptr(l), _ptr(o), s, n, d, _ptr(out), C.c_void_p(_stream(stream))))
    return out


# ------------------------------------------------------------------- decode layer
class DecodeLayer:
    """The per-layer decode body of DecodeEngine::step (decode.cpp:225-273) for one
    token at position T-1: due stages chained through per-stage caches, then the
    BSA over sinks ∪ last cache ∪ stream. Buffers are preallocated so the whole
    step is CUDA-graph capturable.

    q: fp32 [n_q_heads, d]; n_masks independent pooled masks (KV groups).
    """

    def __init__(self, kv: PagedKV, stages, *, sink: int, stream_tokens: int, n_q_heads: int,
                 n_masks: int, layer1: int = 4, policy: RopePolicy | None = None,
                 rope: RopeTable | None = None, device="cuda"):
        require_cuda()
        self.kv, self.stages = kv, [tuple(s) for s in stages]
        self.sink, self.stream_tokens = sink, stream_tokens
        self.n_q_heads, self.n_masks = n_q_heads, n_masks
        self.layer1 = layer1
        self.policy = policy or RopePolicy()
        self.rope = rope
        self.dev = torch.device(device)
        self.ws = Workspace(self.dev)
        self.caches = [(torch.zeros((n_masks, 1, s[2]), dtype=torch.int32, device=self.dev),
                        torch.zeros((n_masks, 1), dtype=torch.int32, device=self.dev))
                       for s in self.stages]
        self.in_start = torch.full((n_masks, 1), sink, dtype=torch.int32, device=self.dev)
        self.in_count = torch.zeros((n_masks, 1), dtype=torch.int32, device=self.dev)
        keep_last = self.stages[-1][2]
        self.sel_stride = sink + keep_last + stream_tokens + 1
        self.sel = torch.zeros((n_masks, 1, self.sel_stride), dtype=torch.int32, device=self.dev)
        self.sel_count = torch.zeros((n_masks, 1), dtype=torch.int32, device=self.dev)
        self.q = torch.zeros((n_q_heads, 1, kv.d), dtype=torch.float32, device=self.dev)
        self.out = torch.zeros((n_q_heads, 1, kv.d), dtype=torch.float32, device=self.dev)
        # size the workspace once for the largest stage / BSA
        t_max = kv.num_pages * kv.page_size
        need = 0
        prev = max(0, t_max - stream_tokens - sink)
        for (_, lc, keep) in self.stages:
            need = max(need, lib().hp_stage_workspace_bytes(n_masks, max(1, ceil_div(prev, lc)), keep, lc))
            prev = keep
        need = max(need, lib().hp_bsa_workspace_bytes(n_q_heads, 1, self.sel_stride, kv.d))
        self.ws.get(need)

    def set_t(self, t: int) -> None:
        """Stage-1 input [n_sink, T - n_stream) for a context of T tokens (decode.cpp:232-240)."""
        upper = t - self.stream_tokens if t > self.stream_tokens else 0
        self.in_count.fill_(max(0, upper - self.sink))

    def run(self, t: int, refresh=None, stream=None) -> torch.Tensor:
        """One layer step at context length t (query position t-1). ``refresh`` flags which
        stages are due (default: all). Reads self.q, writes self.out [n_q_heads, 1, d]."""
        refresh = refresh if refresh is not None else [True] * len(self.stages)
        pos = t - 1
        upper = t - self.stream_tokens if t > self.stream_tokens else 0
        n0 = max(0, upper - self.sink)
        self.in_count.fill_(n0)
        for i, ((bq, lc, keep), (cl, cc)) in enumerate(zip(self.stages, self.caches)):
            if not refresh[i]:
                continue
            if i == 0:
                kw = dict(in_start=self.in_start, in_count=self.in_count, max_chunks=ceil_div(n0, lc))
            else:
                pl, pc = self.caches[i - 1]
                kw = dict(in_list=pl, in_count=pc, in_stride=pl.shape[-1],
                          max_chunks=ceil_div(self.stages[i - 1][2], lc))
            prune_stage((1, lc, keep), self.q, self.kv, n_masks=self.n_masks, n_blocks=1,
                        out_list=cl, out_count=cc, query_offset=pos, stream_tokens=self.stream_tokens,
                        layer1=self.layer1, policy=self.policy, rope=self.rope, ws=self.ws,
                        stream=stream, **kw)
        last_l, last_c = self.caches[-1]
        selected_indices(last_l, last_c, n_rows=1, block_size=1, query_offset=pos, sink=self.sink,
                         stream_tokens=self.stream_tokens, out=(self.sel, self.sel_count),
                         stream=stream)
        bsa(self.q, self.kv, self.sel, self.sel_count, query_offset=pos, max_sel=self.sel_stride,
            policy=self.policy, rope=self.rope, out=self.out, ws=self.ws, stream=stream)
        return self.out


# ----------------------------------------------------------- fused decode (d=128)
def _ref_range(start: int):
    r = _capi.ListRef()
    r.depth = 0
    r.base_list = None
    r.range_start = start
    return r


def _ref_list(base: torch.Tensor):
    r = _capi.ListRef()
    r.depth = 0
    r.base_list = _ptr(base)
    r.base_stride = base.shape[-1]
    r.range_start = 0
    return r


def _ref_push(ref, sel: torch.Tensor, lc: int):
    r = _capi.ListRef()
    C.pointer(r)[0] = ref
    if ref.depth >= 4:
        raise ValueError("list chain deeper than 4 stages")
    r.sel[ref.depth] = _ptr(sel)
    r.sel_stride[ref.depth] = sel.shape[-1]
    r.lc[ref.depth] = lc
    r.depth = ref.depth + 1
    return r


class FusedDecodeLayer:
    """The per-layer decode body on the fused kernels (d = 128): one kernel per due
    stage (exact top-k fused), one BSA kernel (fused combine), one materialize
    kernel that refreshes the stage caches (DecodeEngine::caches_, decode.hpp:107).

    Stage caches follow DecodeEngine::step (decode.cpp:225-249): a due stage reads
    the previous stage's list — implicit (chunk ids) when that stage also ran this
    step, the materialized cache otherwise."""

    def __init__(self, kv: PagedKV, stages, *, sink: int, stream_tokens: int, n_q_heads: int,
                 n_masks: int, layer1: int = 4, policy: RopePolicy | None = None,
                 rope: RopeTable | None = None, device="cuda"):
        require_cuda()
        if kv.d != 128:
            raise ValueError("FusedDecodeLayer: head_dim must be 128 (use DecodeLayer)")
        self.kv, self.stages = kv, [tuple(s) for s in stages]
        self.sink, self.stream_tokens = sink, stream_tokens
        self.n_q_heads, self.n_masks = n_q_heads, n_masks
        self.hpm = n_q_heads // n_masks
        self.layer1 = layer1
        self.policy = policy or RopePolicy()
        self.rope = rope
        dev = self.dev = torch.device(device)
        S = len(self.stages)
        self.sel = [torch.zeros((n_masks, max(1, keep // lc)), dtype=torch.int32, device=dev)
                    for (_, lc, keep) in self.stages]
        self.count = [torch.zeros((n_masks,), dtype=torch.int32, device=dev) for _ in range(S)]
        self.cache = [torch.zeros((n_masks, keep), dtype=torch.int32, device=dev)
                      for (_, _, keep) in self.stages]
        # q and the new token's K/V rows share one device buffer so the host-facing call
        # (step_host) moves all of a step's inputs with a single H2D copy
        esz = torch.tensor([], dtype=kv.dtype).element_size()
        self._io_q = n_q_heads * kv.d * 4
        self._io_kv = kv.n_kv * kv.d * esz
        self._d_io = torch.zeros(self._io_q + 2 * self._io_kv, dtype=torch.uint8, device=dev)
        self.q = self._d_io[: self._io_q].view(torch.float32).view(n_q_heads, kv.d)
        self._d_k = self._d_io[self._io_q: self._io_q + self._io_kv].view(kv.dtype).view(kv.n_kv, kv.d)
        self._d_v = self._d_io[self._io_q + self._io_kv:].view(kv.dtype).view(kv.n_kv, kv.d)
        self.out = torch.zeros((n_q_heads, kv.d), dtype=torch.float32, device=dev)
        t_max = kv.num_pages * kv.page_size
        n0 = max(0, t_max - stream_tokens - sink)
        self.max_chunks = []
        prev = n0
        for (_, lc, keep) in self.stages:
            self.max_chunks.append(max(1, ceil_div(prev, lc)))
            prev = keep
        ws_stage = max(max(lib().hp_decode_stage_workspace_bytes(n_masks, mc) for mc in self.max_chunks),
                       lib().hp_decode_layer_workspace_bytes(n_masks, self.max_chunks[0]))
        self.ws_stage = torch.zeros(ws_stage, dtype=torch.uint8, device=dev)
        max_sel = sink + self.stages[-1][2] + stream_tokens + 1
        self.ws_bsa = torch.zeros(lib().hp_decode_bsa_workspace_bytes(n_q_heads, max_sel),
                                  dtype=torch.uint8, device=dev)
        self._keep = []  # ctypes objects alive across async launches
        self._last_args = [None] * (S + 1)  # per stage + BSA: the last launch's arguments
        self._fused = None  # hp_decode_layer (one cluster kernel after stage 0) when supported

    def _run_fused(self, t, refresh, stream, materialize, mat_stream):
        """The layer on hp_decode_layer: stage 0's descent + one cluster kernel; then the
        refreshed stage caches are expanded (materialize) from the kept chunk ids."""
        S = len(self.stages)
        sp = C.c_void_p(_stream(stream))
        a = self._layer_args(t, refresh)
        check(lib().hp_decode_layer(C.byref(a), sp))
        self._last_args = [self._stage0_args(t) if refresh[0] else None] + ["layer"] * S
        if materialize:
            chains = [None] * S
            for i, (_, lc, keep) in enumerate(self.stages):
                if i == 0:
                    base = _ref_range(self.sink)
                elif refresh[i - 1]:
                    base = chains[i - 1]
                else:
                    base = _ref_list(self.cache[i - 1])
                chains[i] = _ref_push(base, self.sel[i], lc) if refresh[i] else None
            idx = [i for i in range(S) if refresh[i]]
            if idx:
                n = len(idx)
                refs = (_capi.ListRef * n)(*[chains[i] for i in idx])
                counts = (C.c_void_p * n)(*[_ptr(self.count[i]) for i in idx])
                outs = (C.c_void_p * n)(*[_ptr(self.cache[i]) for i in idx])
                strides = (C.c_int64 * n)(*[self.cache[i].shape[-1] for i in idx])
                msp = sp
                if mat_stream is not None:
                    ev = torch.cuda.Event()
                    ev.record(stream if stream is not None else torch.cuda.current_stream())
                    mat_stream.wait_event(ev)
                    msp = C.c_void_p(mat_stream.cuda_stream)
                check(lib().hp_decode_materialize(refs, counts, outs, strides, n, self.n_masks,
                                                  max(self.stages[i][2] for i in idx), msp))
        return self.out

    def dispatch(self) -> list[str]:
        """Which kernel each stage of the last run() launched, then the BSA's
        (hp_decode_stage_variant / hp_decode_bsa_variant); None = not run."""
        out = []
        for i, a in enumerate(self._last_args):
            if a is None or isinstance(a, str):
                out.append(a)
                continue
            v = C.c_int32(-1)
            if i < len(self.stages):
                check(lib().hp_decode_stage_variant(C.byref(a), C.byref(v)))
                out.append(_capi.STAGE_VARIANTS[v.value])
            else:
                check(lib().hp_decode_bsa_variant(C.byref(a), C.byref(v)))
                out.append(_capi.BSA_VARIANTS[v.value])
        return out

    def _layer_args(self, t: int, refresh) -> "_capi.DecodeLayerArgs":
        S = len(self.stages)
        a = _capi.DecodeLayerArgs()
        a.n_stages = S
        for i, (_, lc, keep) in enumerate(self.stages):
            a.chunk_size[i], a.keep[i], a.refresh[i] = lc, keep, int(bool(refresh[i]))
            a.sel[i], a.sel_stride[i] = _ptr(self.sel[i]), self.sel[i].shape[-1]
            a.count[i] = _ptr(self.count[i])
            a.cache[i], a.cache_stride[i] = _ptr(self.cache[i]), self.cache[i].shape[-1]
        a.n_masks, a.heads_per_mask, a.n_q_heads = self.n_masks, self.hpm, self.n_q_heads
        a.sink_tokens, a.stream_tokens = self.sink, self.stream_tokens
        a.q, a.query_position, a.out = _ptr(self.q), t - 1, self._out_ptr()
        a.workspace, a.workspace_bytes = _ptr(self.ws_stage), self.ws_stage.numel()
        a.kv = self.kv.view(t)
        a.keys_exact = _ptr(self.kv.keys_exact)
        return a

    def _out_ptr(self) -> int:
        """Where the step's output goes: self.out, or (inside step_host graphs) the pinned
        host buffer itself — the merging CTA stores straight to host memory (UVA), so the
        host-facing call needs no device-to-host copy."""
        return getattr(self, "_out_override", None) or _ptr(self.out)

    def fused_supported(self) -> bool:
        """hp_decode_layer takes this configuration (bf16, d = 128, RoPE extension off,
        1/2/4/8 heads per KV group, <= 4 stages) and it was not disabled (HP_LAYER=0)."""
        import os
        if os.environ.get("HP_LAYER", "1") == "0" or self.policy.extension or len(self.stages) > 4:
            return False
        return bool(lib().hp_decode_layer_supported(C.byref(self._layer_args(self.kv.t_kv, [True] * len(self.stages)))))

    def run(self, t: int, refresh=None, stream=None, materialize: bool = True,
            mat_stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """One layer step at context length t. ``mat_stream``: materialize the refreshed
        stage caches on that stream (forked after the BSA; the caller joins it before the
        caches are next read) so the copy is off the layer's critical path."""
        S = len(self.stages)
        refresh = list(refresh) if refresh is not None else [True] * S
        if self._fused is None:
            self._fused = self.fused_supported()
        # hp_decode_layer when any stage is due (the stages' selections and the attention
        # chain inside one kernel); a step that reuses every cache runs the split-K BSA
        # kernel alone, measured faster for that step
        if self._fused and (self._fused == "always" or any(refresh)):
            return self._run_fused(t, refresh, stream, materialize, mat_stream)
        pos = t - 1
        upper = t - self.stream_tokens if t > self.stream_tokens else 0
        n0 = max(0, upper - self.sink)
        sp = C.c_void_p(_stream(stream))
        kvv = self.kv.view(t)
        chains = [None] * S
        # per-stage bound on the input length at this context (stage i reads at most
        # min(n0, k_{i-1}) tokens): tight grids, and provably-identity stages are known
        # on the host (the reference never rotates — so never range-checks — those)
        bound, prev = [], n0
        for i, (_, lc, keep) in enumerate(self.stages):
            if i > 0 and not refresh[i - 1]:
                prev = self.stages[i - 1][2]  # a cached list from an earlier step: only k bounds it
            bound.append(max(1, min(self.max_chunks[i], ceil_div(prev, lc))))
            prev = min(prev, keep)
        for i, (_, lc, keep) in enumerate(self.stages):
            if i == 0:
                in_ref, in_count, const = _ref_range(self.sink), None, n0
            elif refresh[i - 1]:
                in_ref, in_count, const = chains[i - 1], self.count[i - 1], 0
            else:
                in_ref, in_count, const = _ref_list(self.cache[i - 1]), self.count[i - 1], 0
            if refresh[i]:
                a = _capi.DecodeStageArgs(
                    chunk_size=lc, keep=keep, n_masks=self.n_masks, heads_per_mask=self.hpm,
                    n_q_heads=self.n_q_heads, stream_tokens=self.stream_tokens, q=_ptr(self.q),
                    query_position=pos, in_=in_ref, in_count=_ptr(in_count), in_count_const=const,
                    max_chunks=bound[i], sel_stride=self.sel[i].shape[-1],
                    sel_out=_ptr(self.sel[i]), out_count=_ptr(self.count[i]),
                    workspace=_ptr(self.ws_stage), workspace_bytes=self.ws_stage.numel(),
                    keys=kvv, rope=self.policy.ctx(self.layer1, self.rope),
                    keys_exact=_ptr(self.kv.keys_exact),
                    # the last stage materializes its list (= its cache) for the BSA
                    list_out=_ptr(self.cache[i]) if i == S - 1 else None,
                    list_out_stride=self.cache[i].shape[-1])
                check(lib().hp_decode_stage(C.byref(a), sp))
                self._last_args[i] = a
                chains[i] = (_ref_list(self.cache[i]) if i == S - 1
                             else _ref_push(in_ref, self.sel[i], lc))
            else:
                chains[i] = _ref_list(self.cache[i])
        b = _capi.DecodeBsaArgs(
            n_q_heads=self.n_q_heads, heads_per_mask=self.hpm, sink_tokens=self.sink,
            stream_tokens=self.stream_tokens, q=_ptr(self.q), query_position=pos,
            mask=chains[-1], mask_count=_ptr(self.count[-1]), max_mask=self.stages[-1][2],
            out=self._out_ptr(), part_m=None, part_l=None, part_o=None,
            workspace=_ptr(self.ws_bsa), workspace_bytes=self.ws_bsa.numel(), kv=kvv,
            rope=self.policy.ctx(0, self.rope),
            # the last stage's cache is untouched this step: gather in the PDL prologue
            mask_stable=0 if refresh[-1] else 1)
        check(lib().hp_decode_bsa(C.byref(b), sp))
        self._last_args[S] = b
        if materialize:
            idx = [i for i in range(S - 1) if refresh[i]]  # the last stage wrote its own
            if idx:
                n = len(idx)
                refs = (_capi.ListRef * n)(*[chains[i] for i in idx])
                counts = (C.c_void_p * n)(*[_ptr(self.count[i]) for i in idx])
                outs = (C.c_void_p * n)(*[_ptr(self.cache[i]) for i in idx])
                strides = (C.c_int64 * n)(*[self.cache[i].shape[-1] for i in idx])
                msp = sp
                if mat_stream is not None:
                    ev = torch.cuda.Event()
                    ev.record(stream if stream is not None else torch.cuda.current_stream())
                    mat_stream.wait_event(ev)
                    msp = C.c_void_p(mat_stream.cuda_stream)
                check(lib().hp_decode_materialize(refs, counts, outs, strides, n, self.n_masks,
                                                  max(self.stages[i][2] for i in idx), msp))
        return self.out

    def _stage0_args(self, t: int):
        """Stage 0's descent arguments as hp_decode_layer builds them (dispatch query)."""
        (_, lc, keep) = self.stages[0]
        upper = t - self.stream_tokens if t > self.stream_tokens else 0
        n0 = max(0, upper - self.sink)
        return _capi.DecodeStageArgs(
            chunk_size=lc, keep=keep, n_masks=self.n_masks, heads_per_mask=self.hpm,
            n_q_heads=self.n_q_heads, stream_tokens=self.stream_tokens, q=_ptr(self.q),
            query_position=t - 1, in_=_ref_range(self.sink), in_count=None, in_count_const=n0,
            max_chunks=max(1, ceil_div(n0, lc)), sel_stride=self.sel[0].shape[-1], sel_out=None,
            out_count=_ptr(self.count[0]), workspace=_ptr(self.ws_stage),
            workspace_bytes=self.ws_stage.numel(), keys=self.kv.view(t), keys_exact=_ptr(self.kv.keys_exact))

    def run_stage(self, t: int, i: int = 0, stream=None, select: bool = True) -> None:
        """Launch only stage i (descent, + selection unless select=False) on its input:
        stage 0 reads the range [n_sink, T - n_stream), later stages the materialized
        cache of i-1. Used to time / instrument the dominant kernel in isolation."""
        (_, lc, keep) = self.stages[i]
        pos = t - 1
        upper = t - self.stream_tokens if t > self.stream_tokens else 0
        if i == 0:
            in_ref, in_count, const = _ref_range(self.sink), None, max(0, upper - self.sink)
        else:
            in_ref, in_count, const = _ref_list(self.cache[i - 1]), self.count[i - 1], 0
        a = _capi.DecodeStageArgs(
            chunk_size=lc, keep=keep, n_masks=self.n_masks, heads_per_mask=self.hpm,
            n_q_heads=self.n_q_heads, stream_tokens=self.stream_tokens, q=_ptr(self.q),
            query_position=pos, in_=in_ref, in_count=_ptr(in_count), in_count_const=const,
            max_chunks=self.max_chunks[i], sel_stride=self.sel[i].shape[-1],
            sel_out=_ptr(self.sel[i]) if select else None, out_count=_ptr(self.count[i]),
            workspace=_ptr(self.ws_stage), workspace_bytes=self.ws_stage.numel(),
            keys=self.kv.view(t), rope=self.policy.ctx(self.layer1, self.rope),
            keys_exact=_ptr(self.kv.keys_exact), list_out=None, list_out_stride=0)
        check(lib().hp_decode_stage(C.byref(a), C.c_void_p(_stream(stream))))

    def step_host(self, t: int, q_host, k_row=None, v_row=None, out_host=None, refresh=None,
                  sync: bool = True) -> torch.Tensor:
        """The host-facing decode call for the token at position t-1 (what a serving
        loop calls per layer): host q [n_q_heads, d] fp32 and the token's K/V rows
        [n_kv, d] in, host output [n_q_heads, d] fp32 out. One CUDA graph per
        (t, refresh): pinned H2D copy -> append kernel -> the layer step, whose merging CTA
        stores the output straight into the pinned host buffer (no D2H copy).
        Returns the pinned output buffer (valid after sync)."""
        has_kv = k_row is not None
        key = (t, tuple(refresh) if refresh is not None else None, has_kv)
        if not hasattr(self, "_hg"):
            self._hg = {}
            self._h_io = torch.empty(self._d_io.numel(), dtype=torch.uint8).pin_memory()
            self._h_q = self._h_io[: self._io_q].view(torch.float32).view(self.q.shape)
            self._h_k = self._h_io[self._io_q: self._io_q + self._io_kv].view(self.kv.dtype).view(self._d_k.shape)
            self._h_v = self._h_io[self._io_q + self._io_kv:].view(self.kv.dtype).view(self._d_v.shape)
            self._h_out = torch.empty((self.n_q_heads, self.kv.d), dtype=torch.float32).pin_memory()
            self._side = torch.cuda.Stream(device=self.dev)
        self._h_q.copy_(torch.as_tensor(q_host).reshape(self._h_q.shape))
        if has_kv:
            self._h_k.copy_(torch.as_tensor(k_row).reshape(self._h_k.shape))
            self._h_v.copy_(torch.as_tensor(v_row).reshape(self._h_v.shape))
        g = self._hg.get(key)
        if g is None:
            def body():
                # one H2D copy of q + the token's K/V rows, append, the layer step (stage
                # caches materialized on a side branch; output written to host memory)
                cur = torch.cuda.current_stream()
                n_in = self._d_io.numel() if has_kv else self._io_q
                self._d_io[:n_in].copy_(self._h_io[:n_in], non_blocking=True)
                if has_kv:
                    view = self.kv.view(t)
                    check(lib().hp_decode_append(C.byref(view), _ptr(self._d_k), _ptr(self._d_v),
                                                 t - 1, _ptr(self.kv.keys_exact),
                                                 C.c_void_p(_stream())))
                self._side.wait_stream(cur)
                self._out_override = self._h_out.data_ptr()  # output stored to pinned host memory
                try:
                    self.run(t, refresh=refresh, mat_stream=self._side)
                finally:
                    self._out_override = None
                cur.wait_stream(self._side)
            s = torch.cuda.Stream(device=self.dev)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                body()  # warm-up outside capture
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body()
            self._hg[key] = g
        g.replay()
        if sync:
            torch.cuda.current_stream().synchronize()
            if out_host is not None:
                torch.as_tensor(out_host).copy_(self._h_out.reshape(torch.as_tensor(out_host).shape))
        return self._h_out

    def mask(self, stage: int = -1):
        """Materialized stage cache (lists, counts) — DecodeEngine::stage_cache."""
        return self.cache[stage], self.count[stage]


# ------------------------------------------------------------ page cache (K6)
class CachedKV(PagedKV):
    """Paged K/V of one layer held in pinned host memory with an on-GPU LRU page
    cache of ``num_slots`` pages in front of it (TieredKvStore over the host tier,
    kv_store.cpp:58-120). Gathers read resident pages from their device slot and
    missing pages from the mapped host tier inside the same kernel, flagging the
    page; ``commit()`` (the step-end commit) installs the missed pages into the
    least-recently-used slots. Drop-in for PagedKV in the decode layers.

    warm: "recent" makes the last ``num_slots`` pages resident at start (the
    prefill's working set around the stream window), "none" starts empty.
    """

    def __init__(self, k: torch.Tensor, v: torch.Tensor | None, *, num_slots: int, page_size: int = 64,
                 dtype: torch.dtype = torch.bfloat16, capacity: int | None = None, device="cuda",
                 warm: str = "recent"):
        super().__init__(k, v, page_size=page_size, dtype=dtype, capacity=capacity, device=device)
        dev = torch.device(device)
        # host tier (authoritative, pinned, device-mapped under UVA) and the device slots
        self.k_host = self.k_pool.cpu().pin_memory()
        self.v_host = self.v_pool.cpu().pin_memory() if self.v_pool is not None else None
        self.num_slots = int(min(num_slots, self.num_pages))
        shape = (self.num_slots, self.n_kv, page_size, self.d)
        self.k_slots = torch.zeros(shape, dtype=dtype, device=dev)
        self.v_slots = torch.zeros(shape, dtype=dtype, device=dev) if v is not None else None
        self.page_table = torch.full((self.num_pages,), -1, dtype=torch.int32, device=dev)
        self.slot_page = torch.full((self.num_slots,), -1, dtype=torch.int32, device=dev)
        self.slot_stamp = torch.zeros((self.num_slots,), dtype=torch.int32, device=dev)
        self.touched = torch.zeros((self.num_pages,), dtype=torch.uint8, device=dev)
        self.stats = torch.zeros(3, dtype=torch.int32, device=dev)  # hits, misses, evictions
        self.ws_cache = torch.zeros(lib().hp_cache_workspace_bytes(self.num_pages, self.num_slots),
                                    dtype=torch.uint8, device=dev)
        self.stamp = 1
        if warm == "recent":
            used = ceil_div(self.t_kv, page_size)
            first = max(0, used - self.num_slots)
            pages = torch.arange(first, used, device=dev, dtype=torch.int32)
            n = pages.numel()
            self.page_table[first:used] = torch.arange(n, device=dev, dtype=torch.int32)
            self.slot_page[:n] = pages
            self.slot_stamp[:n] = 1
            self.k_slots[:n].copy_(self.k_pool[first:used])
            if self.v_slots is not None:
                self.v_slots[:n].copy_(self.v_pool[first:used])
        # the full device pools were only needed to build the tiers
        self.k_pool_full, self.v_pool_full = self.k_pool, self.v_pool
        self.k_pool, self.v_pool = self.k_slots, self.v_slots
        del self.k_pool_full, self.v_pool_full

    def view(self, t_kv: int | None = None) -> KvView:
        return KvView(k_pool=_ptr(self.k_slots), v_pool=_ptr(self.v_slots), k_host=self.k_host.data_ptr(),
                      v_host=self.v_host.data_ptr() if self.v_host is not None else None,
                      page_table=_ptr(self.page_table), touched=_ptr(self.touched),
                      num_pages=self.num_pages, page_size=self.page_size, n_kv=self.n_kv, d=self.d,
                      dtype=_DT[self.dtype], t_kv=t_kv if t_kv is not None else self.t_kv,
                      row_bits=_ptr(self.row_bits), row_bits_stride=self.num_pages * self.page_size)

    def cache_struct(self):
        return _capi.PageCache(k_slots=_ptr(self.k_slots), v_slots=_ptr(self.v_slots),
                               k_host=self.k_host.data_ptr(),
                               v_host=self.v_host.data_ptr() if self.v_host is not None else None,
                               page_table=_ptr(self.page_table), slot_page=_ptr(self.slot_page),
                               slot_stamp=_ptr(self.slot_stamp), touched=_ptr(self.touched),
                               num_pages=self.num_pages, num_slots=self.num_slots,
                               page_size=self.page_size, n_kv=self.n_kv, d=self.d, dtype=_DT[self.dtype])

    def commit(self, stream=None) -> None:
        """Step-end commit (decode.cpp:279-280): hits take this step's stamp, misses
        are installed into the LRU slots. Uses the device step clock (stamp 0), so a
        captured CUDA graph replays it correctly."""
        self._cache_s = self.cache_struct()
        check(lib().hp_cache_commit(C.byref(self._cache_s), 0, _ptr(self.stats), _ptr(self.ws_cache),
                                    self.ws_cache.numel(), C.c_void_p(_stream(stream))))

    def append(self, k_row, v_row=None):
        raise NotImplementedError("CachedKV: append through hp_decode_append (write-through to the host tier)")

    def resident_pages(self) -> int:
        return int((self.page_table >= 0).sum())


# ------------------------------------------------------- prefill BSA on tcgen05
def bsa_prefill_tc(q: torch.Tensor, kv: PagedKV, mask_list: torch.Tensor, mask_count: torch.Tensor, *,
                   block_size: int, query_offset: int, sink: int, stream_tokens: int,
                   out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """block_sparse_attention (sparse_attention.cpp:114-145) for a prefill on the tensor
    cores (hp_bsa_prefill): q fp32 [n_q_heads, T_q, 128]; mask lists [n_masks, n_blocks,
    stride] (+ counts) as build_mask returns them; bf16 K/V. Returns [n_q_heads, T_q, 128]."""
    hq, t_q, d = q.shape
    n_masks, nb, stride = mask_list.shape
    out = out if out is not None else torch.empty_like(q)
    a = _capi.BsaPrefillArgs(n_q_heads=hq, heads_per_mask=hq // n_masks, n_rows=t_q, block_size=block_size,
                             q=_ptr(q), query_offset=query_offset, mask_list=_ptr(mask_list),
                             mask_count=_ptr(mask_count), mask_stride=stride, n_mask_blocks=nb, max_mask=stride,
                             sink_tokens=sink, stream_tokens=stream_tokens, out=_ptr(out), kv=kv.view())
    check(lib().hp_bsa_prefill(C.byref(a), C.c_void_p(_stream(stream))))
    return out

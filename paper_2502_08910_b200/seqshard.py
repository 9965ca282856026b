"""Sequence-sharded decode (BASELINE config C5: 3M-token context over several GPUs).

The KV sequence is split into contiguous shards, one per rank; sinks live on rank 0
and the stream window on the last rank. Shard boundaries sit at
``n_sink + (multiple of the stage-1 chunk size)``, so every stage-1 chunk is
shard-local, and because the stage chunk sizes nest (256 = 8 x 32, 32 = 4 x 8, 3k
preset) every stage-2/3 chunk is shard-local too: every descent and every chunk score
is computed on the rank that holds its keys.

The only exchanges, per layer step:
  * per stage: all-gather of the shards' fp32 chunk scores, then the identical global
    stable top-K on every rank (hp_select_topk) — the reference's selection
    (pruning.cpp:187-192) over the full score vector, so the kept indices equal the
    unsharded run's exactly;
  * after the BSA: all-gather of each shard's (m, l, o) per q-head and the log-sum-exp
    merge (hp_lse_merge).

``SeqShardLayer`` holds one rank's shard and exposes the step as phases (descend,
select, attend, merge) around those two collectives; every phase is one kernel launch
(select: hp_select_topk_sharded rebuilds the global score vector, selects, and cuts
out the rank's part on the device). Every rank's score buffer has the same width,
ceil(chunks / world), so the all-gather needs no padding step. ``run_step`` drives
the phases with a real process group (NCCL; gloo through host memory for the 1-GPU
multi-rank tests); ``run_step_virtual`` drives several shards inside one process (the
single-GPU parity check). ``assemble``, ``local_part`` and ``lse_merge_reference``
are torch restatements of the device steps for the CPU checks only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _capi
from ._capi import check, lib


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


# ------------------------------------------------------------------ geometry
@dataclass
class ShardGeometry:
    """Rank `rank`'s part of the stage-1 middle range [sink, T - stream)."""
    t: int
    sink: int
    stream: int
    lc1: int
    world: int
    rank: int

    @property
    def upper(self) -> int:
        return self.t - self.stream if self.t > self.stream else 0

    @property
    def n0(self) -> int:  # stage-1 input length (decode.cpp:232-240)
        return max(0, self.upper - self.sink)

    @property
    def cc1(self) -> int:
        return ceil_div(self.n0, self.lc1)

    def chunk_range(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        return r * self.cc1 // self.world, (r + 1) * self.cc1 // self.world

    def token_range(self, rank: int | None = None) -> tuple[int, int]:
        """Tokens whose K/V rank r holds: its stage-1 chunks, plus the sinks on rank 0
        and the stream window (and decode capacity) on the last rank."""
        r = self.rank if rank is None else rank
        c0, c1 = self.chunk_range(r)
        t0 = 0 if r == 0 else self.sink + c0 * self.lc1
        t1 = self.t if r == self.world - 1 else self.sink + c1 * self.lc1
        return t0, t1

    def local_stage1(self) -> tuple[int, int]:
        """(first token, length) of this rank's stage-1 input."""
        c0, c1 = self.chunk_range()
        a = self.sink + c0 * self.lc1
        b = min(self.upper, self.sink + c1 * self.lc1)
        return a, max(0, b - a)


def assemble(gathered: torch.Tensor, counts: torch.Tensor, width: int) -> torch.Tensor:
    """(CPU checker of hp_select_topk_sharded) concatenate per-rank segments in rank order, per mask.

    gathered [R, M, W] local scores (rank r's first counts[r, m] are valid),
    counts [R, M] -> [M, width] with row m = concat_r gathered[r, m, :counts[r, m]]
    (padding past the total is -inf)."""
    R, M, W = gathered.shape
    starts = torch.cumsum(counts, 0) - counts                      # [R, M]
    total = counts.sum(0)                                          # [M]
    pos = torch.arange(width, device=gathered.device).expand(M, width)
    # owner rank of global position i of mask m: last r with starts[r, m] <= i
    owner = (pos.unsqueeze(0) >= starts.unsqueeze(-1)).sum(0) - 1  # [M, width]
    owner = owner.clamp(0, R - 1)
    local = pos - torch.gather(starts.t(), 1, owner)
    val = gathered[owner, torch.arange(M, device=gathered.device).unsqueeze(1), local.clamp(0, W - 1)]
    return torch.where(pos < total.unsqueeze(1), val, torch.full_like(val, float("-inf")))


def local_part(sel: torch.Tensor, k: torch.Tensor, lo: torch.Tensor, n: torch.Tensor):
    """(CPU checker of hp_select_topk_sharded) this rank's slice of a global ascending selection.

    sel [M, K] global chunk ids ascending (first k[m] valid), lo/n [M]: this rank owns
    global chunks [lo, lo + n). Returns (local ids [M, K] — the first cnt[m] valid —,
    cnt [M], number of selected chunks below lo [M])."""
    M, K = sel.shape
    idx = torch.arange(K, device=sel.device).expand(M, K)
    valid = idx < k.unsqueeze(1)
    below = ((sel < lo.unsqueeze(1)) & valid).sum(1)
    inside = ((sel >= lo.unsqueeze(1)) & (sel < (lo + n).unsqueeze(1)) & valid).sum(1)
    src = (below.unsqueeze(1) + idx).clamp(max=K - 1)
    loc = torch.gather(sel, 1, src) - lo.unsqueeze(1)
    loc = torch.where(idx < inside.unsqueeze(1), loc, torch.zeros_like(loc))
    return loc.to(torch.int32), inside.to(torch.int32), below


def lse_merge_reference(m: torch.Tensor, l: torch.Tensor, o: torch.Tensor) -> torch.Tensor:
    """torch restatement of hp_lse_merge (the CPU checker for the merge): m, l [S, n],
    o [S, n, d] (each shard's normalised output) -> [n, d]."""
    live = l > 0
    mm = torch.where(live, m, torch.full_like(m, float("-inf")))
    M = mm.max(0).values
    w = torch.where(live, l * torch.exp(mm - M), torch.zeros_like(l))
    return (o * w.unsqueeze(-1)).sum(0) / w.sum(0).unsqueeze(-1)


# ---------------------------------------------------------------- rank state
class SeqShardLayer:
    """One rank's shard of a decode layer (fused d = 128 kernels).

    k, v: this rank's token range [t0, t1) of the layer's K/V, [n_kv, t1 - t0, d].
    Global page ids resolve through a page table to the shard's local pages, so the
    kernels see global token indices throughout."""

    def __init__(self, geo: ShardGeometry, k: torch.Tensor, v: torch.Tensor, stages, *, n_q_heads: int,
                 n_masks: int, page_size: int = 64, device="cuda"):
        from .device import PagedKV, _ref_push, _ref_range  # noqa: F401
        self.geo = geo
        self.stages = [tuple(s) for s in stages]
        if any(self.stages[i][1] % self.stages[i + 1][1] for i in range(len(self.stages) - 1)):
            raise ValueError("sequence sharding needs nested chunk sizes (l_c of stage i divisible by stage i+1)")
        self.dev = torch.device(device)
        self.n_q_heads, self.n_masks = n_q_heads, n_masks
        self.hpm = n_q_heads // n_masks
        t0, t1 = geo.token_range()
        if t0 % page_size:
            raise ValueError("shard start must be page aligned (sink + multiple of l_c1)")
        self.t0, self.t1 = t0, t1
        self.kv = PagedKV(k, v, page_size=page_size, device=device)
        # global pages -> local pages; num_pages spans the whole context (others = -1)
        g_pages = ceil_div(geo.t, page_size)
        pt = torch.full((g_pages,), -1, dtype=torch.int32, device=self.dev)
        first = t0 // page_size
        pt[first:first + self.kv.num_pages] = torch.arange(self.kv.num_pages, dtype=torch.int32, device=self.dev)
        self.kv.page_table = pt
        self.kv.num_pages = g_pages
        self.kv.t_kv = geo.t
        self.q = torch.zeros((n_q_heads, 128), dtype=torch.float32, device=self.dev)
        self.out = torch.zeros((n_q_heads, 128), dtype=torch.float32, device=self.dev)
        M = n_masks
        self.part_m = torch.zeros(n_q_heads, dtype=torch.float32, device=self.dev)
        self.part_l = torch.zeros(n_q_heads, dtype=torch.float32, device=self.dev)
        self.part_o = torch.zeros((n_q_heads, 128), dtype=torch.float32, device=self.dev)
        # per stage: local scores (padded), global selection, this rank's slice of it
        self.max_local = []
        prev_keep = None
        for i, (_, lc, keep) in enumerate(self.stages):
            if i == 0:  # the same width on every rank: the all-gather needs equal sizes
                self.max_local.append(max(1, ceil_div(geo.cc1, geo.world)))
            else:
                self.max_local.append(max(1, ceil_div(prev_keep, lc)))
            prev_keep = keep
        self.scores = [torch.full((M, w), float("-inf"), device=self.dev) for w in self.max_local]
        self.sel_g = [torch.zeros((M, max(1, keep // lc)), dtype=torch.int32, device=self.dev)
                      for (_, lc, keep) in self.stages]
        self.cnt_g = [torch.zeros(M, dtype=torch.int32, device=self.dev) for _ in self.stages]
        self.sel_l = [torch.zeros((M, max(1, keep // lc)), dtype=torch.int32, device=self.dev)
                      for (_, lc, keep) in self.stages]  # this rank's kept chunks (local ids)
        self.len_l = [torch.zeros(M, dtype=torch.int32, device=self.dev)
                      for _ in self.stages]  # this rank's stage-(i+1) input length [M]
        self.ccl = [None] * len(self.stages)       # this rank's chunk count at stage i [M]
        self.g0 = [None] * len(self.stages)        # first global chunk of this rank at stage i [M]
        ws = max(lib().hp_decode_stage_workspace_bytes(M, w) for w in self.max_local)
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=self.dev)
        last_keep = self.stages[-1][2]
        max_sel = geo.sink + last_keep + geo.stream + 1
        self.ws_bsa = torch.zeros(lib().hp_decode_bsa_workspace_bytes(n_q_heads, max_sel), dtype=torch.uint8,
                                  device=self.dev)
        self._keep = []

    # ---- chain of this rank's input list for stage i (tokens resolved globally)
    def _in_ref(self, i: int):
        from .device import _ref_push, _ref_range
        a, _ = self.geo.local_stage1()
        ref = _ref_range(a)
        for j in range(i):
            ref = _ref_push(ref, self.sel_l[j], self.stages[j][1])
        return ref

    def descend(self, i: int, pos: int, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """Stage i's descents over this rank's chunks -> (local scores [M, W], chunk counts [M])."""
        M = self.n_masks
        _, lc, keep = self.stages[i]
        if i == 0:
            _, n_local = self.geo.local_stage1()
            count = torch.full((M,), n_local, dtype=torch.int32, device=self.dev)
            in_count, const = None, n_local
        else:
            count = self.len_l[i - 1]
            in_count, const = count, 0
        ccl = (count + lc - 1) // lc
        self.ccl[i] = ccl
        a = _capi.DecodeStageArgs(
            chunk_size=lc, keep=keep, n_masks=M, heads_per_mask=self.hpm, n_q_heads=self.n_q_heads,
            stream_tokens=self.geo.stream, q=self.q.data_ptr(), query_position=pos, in_=self._in_ref(i),
            in_count=in_count.data_ptr() if in_count is not None else None, in_count_const=const,
            max_chunks=self.max_local[i], sel_stride=0, sel_out=None, out_count=None,
            workspace=self.ws.data_ptr(), workspace_bytes=self.ws.numel(), keys=self.kv.view(self.geo.t),
            rope=_capi.RopeCtx(), keys_exact=self.kv.keys_exact.data_ptr(), list_out=None, list_out_stride=0,
            scores_out=self.scores[i].data_ptr())
        self._keep.append(a)
        if const > 0 or in_count is not None:
            check(lib().hp_decode_stage(C.byref(a), C.c_void_p(_stream(stream))))
        return self.scores[i], ccl.to(torch.int32)

    def select(self, i: int, gathered: torch.Tensor, counts: torch.Tensor, stream=None) -> None:
        """Global stable top-K from every rank's scores [R, M, W] (chunk counts [R, M]),
        and this rank's slice of it — one kernel (hp_select_topk_sharded)."""
        M = self.n_masks
        _, lc, keep = self.stages[i]
        R, _, W = gathered.shape
        g = gathered.contiguous()
        c = counts.to(torch.int32).contiguous()
        self._keep += [g, c]
        if i == 0:
            n_in, n_const = None, self.geo.n0
        else:
            n_in, n_const = self.cnt_g[i - 1].data_ptr(), 0
        check(lib().hp_select_topk_sharded(g.data_ptr(), c.data_ptr(), R, W, self.geo.rank, M, n_in, n_const, lc,
                                           keep, self.sel_g[i].data_ptr(), self.sel_g[i].shape[1],
                                           self.cnt_g[i].data_ptr(), self.sel_l[i].data_ptr(),
                                           self.len_l[i].data_ptr(), C.c_void_p(_stream(stream))))

    def _global_input_len(self, i: int) -> torch.Tensor:
        M = self.n_masks
        if i == 0:
            return torch.full((M,), self.geo.n0, dtype=torch.int32, device=self.dev)
        return self.cnt_g[i - 1]

    def attend(self, pos: int, stream=None) -> None:
        """This shard's part of the BSA: its mask tokens (+ sinks on rank 0, + stream on
        the last rank) -> the per-head (m, l, o) triple."""
        from .device import _ref_push
        geo = self.geo
        ref = self._in_ref(len(self.stages) - 1)
        ref = _ref_push(ref, self.sel_l[-1], self.stages[-1][1])
        b = _capi.DecodeBsaArgs(
            n_q_heads=self.n_q_heads, heads_per_mask=self.hpm,
            sink_tokens=geo.sink if geo.rank == 0 else 0,
            stream_tokens=geo.stream if geo.rank == geo.world - 1 else 0, q=self.q.data_ptr(),
            query_position=pos, mask=ref, mask_count=self.len_l[-1].data_ptr(), max_mask=self.stages[-1][2],
            out=self.out.data_ptr(), part_m=self.part_m.data_ptr(), part_l=self.part_l.data_ptr(),
            part_o=self.part_o.data_ptr(), workspace=self.ws_bsa.data_ptr(), workspace_bytes=self.ws_bsa.numel(),
            kv=self.kv.view(geo.t), rope=_capi.RopeCtx())
        self._keep.append(b)
        check(lib().hp_decode_bsa(C.byref(b), C.c_void_p(_stream(stream))))

    def merge(self, m: torch.Tensor, l: torch.Tensor, o: torch.Tensor, out: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
        S, n = m.shape
        out = out if out is not None else torch.empty((n, 128), dtype=torch.float32, device=self.dev)
        check(lib().hp_lse_merge(m.data_ptr(), l.data_ptr(), o.data_ptr(), S, n, 128, out.data_ptr(),
                                 C.c_void_p(_stream(stream))))
        return out

    def final_mask(self) -> torch.Tensor:
        """The global final-stage token list per mask on this rank's part (for checks)."""
        return self.sel_l[-1], self.len_l[-1]


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------------- drivers
def _all_gather(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[world, *x.shape]: NCCL all_gather_into_tensor on the device; gloo (CPU process
    groups — the multi-rank tests with every rank on one GPU) through host memory."""
    import torch.distributed as dist
    x = x.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x, group=group)
        return out
    parts = [torch.empty_like(x, device="cpu") for _ in range(world)]
    dist.all_gather(parts, x.cpu(), group=group)
    return torch.stack(parts).to(x.device)


def run_step(layer: SeqShardLayer, pos: int, group=None) -> torch.Tensor:
    """One decode layer step over a process group (NCCL over NVLink on a GPU box):
    per stage an all-gather of chunk scores + chunk counts, then one of the (m, l, o)
    partials. Every rank returns the merged output [n_q_heads, 128]."""
    world = layer.geo.world
    layer._keep.clear()  # the previous step's launch arguments (stream order keeps them valid)
    for i in range(len(layer.stages)):
        sc, cnt = layer.descend(i, pos)
        layer.select(i, _all_gather(sc, world, group), _all_gather(cnt, world, group))
    layer.attend(pos)
    parts = torch.cat([layer.part_m.unsqueeze(1), layer.part_l.unsqueeze(1), layer.part_o], 1)
    g = _all_gather(parts, world, group)
    return layer.merge(g[:, :, 0].contiguous(), g[:, :, 1].contiguous(), g[:, :, 2:].contiguous())


def run_step_virtual(layers: list[SeqShardLayer], pos: int) -> torch.Tensor:
    """The same step with every shard in this process (single-GPU parity check): the
    collectives become stacks of the shards' tensors."""
    for ly in layers:
        ly._keep.clear()
    for i in range(len(layers[0].stages)):
        outs = [ly.descend(i, pos) for ly in layers]
        g_sc = torch.stack([sc for sc, _ in outs])
        g_cnt = torch.stack([c for _, c in outs])
        for ly in layers:
            ly.select(i, g_sc, g_cnt)
    for ly in layers:
        ly.attend(pos)
    m = torch.stack([ly.part_m for ly in layers])
    l = torch.stack([ly.part_l for ly in layers])
    o = torch.stack([ly.part_o for ly in layers])
    return layers[0].merge(m.contiguous(), l.contiguous(), o.contiguous())

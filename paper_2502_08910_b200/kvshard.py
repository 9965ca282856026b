"""KV-head-group sharded decode (BASELINE config C3 on 1/2/4/8 GPUs).

Masks are per KV group: the reference pools the chunk score over every head it is
handed (max over heads, /root/reference/proj/src/pruning.cpp:176-184), so one
reference call per KV group — the GQA convention of SURVEY.md §7 — makes the
groups fully independent: their K/V, their pruning stages, their stage caches and
their attention share nothing. Rank r of N therefore owns the contiguous groups
``group_range(n_groups, N, r)`` of EVERY layer (strong scaling: the layer's work is
fixed, split N ways), runs the whole per-layer body for them on its own GPU, and
exchanges nothing on the data path. The only collective is optional: an all-gather
of the per-rank attention outputs (n_q_heads x d fp32, 16 KB per layer for the
Llama-3.1-8B shape) when the caller wants every head on every rank.

Refilling the GPU as groups shrink: with one group per GPU (N = 8) the stage-1
descent has only ~4K chunk x 4-head lanes, so hp_decode_stage drops from the one-wave
kernel to the two-comparison lookahead kernel, and hp_decode_layer sizes its
persistent grid as n_SM / n_groups CTAs per group — all 148 SMs serve the one group
(DESIGN.md §6).
"""
from __future__ import annotations

import torch

from . import device as D


def group_range(n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous groups of rank `rank` (the first n_groups % world ranks take one more)."""
    if not (0 <= rank < world) or n_groups < world:
        raise ValueError(f"kvshard: {n_groups} KV groups cannot be split over {world} ranks")
    base, extra = divmod(n_groups, world)
    g0 = rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


class KvGroupShardLayer:
    """One rank's KV groups of one layer: a FusedDecodeLayer over heads
    [g0 * hpm, g1 * hpm) and kv heads [g0, g1).

    k, v: [n_groups_local, T, d] (this rank's groups only) or the full [n_groups, T, d]
    (then sliced here)."""

    def __init__(self, k: torch.Tensor, v: torch.Tensor, stages, *, sink: int, stream_tokens: int,
                 n_groups: int, heads_per_group: int, world: int, rank: int, page_size: int = 64,
                 capacity: int | None = None, device="cuda"):
        self.g0, self.g1 = group_range(n_groups, world, rank)
        self.n_groups, self.hpm, self.world, self.rank = n_groups, heads_per_group, world, rank
        if k.shape[0] == n_groups and n_groups != self.g1 - self.g0:
            k, v = k[self.g0:self.g1], v[self.g0:self.g1]
        self.kv = D.PagedKV(k, v, page_size=page_size, capacity=capacity, device=device)
        ng = self.g1 - self.g0
        self.layer = D.FusedDecodeLayer(self.kv, stages, sink=sink, stream_tokens=stream_tokens,
                                        n_q_heads=ng * heads_per_group, n_masks=ng, device=device)

    @property
    def head_range(self) -> tuple[int, int]:
        return self.g0 * self.hpm, self.g1 * self.hpm

    @property
    def q(self) -> torch.Tensor:
        return self.layer.q

    def set_q(self, q_all: torch.Tensor) -> None:
        """Copy this rank's heads out of the full [n_q_heads, d] query."""
        h0, h1 = self.head_range
        self.layer.q.copy_(q_all[h0:h1])

    def run(self, t: int, refresh=None, stream=None, mat_stream=None) -> torch.Tensor:
        return self.layer.run(t, refresh=refresh, stream=stream, mat_stream=mat_stream)

    def gather(self, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
        """All ranks' outputs as [n_q_heads, d] on every rank (the optional collective)."""
        return gather_outputs(self.layer.out if out is None else out, self.world, group=group)


def gather_outputs(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Concatenate every rank's [heads_r, d] output in rank order (= head order, groups
    are contiguous per rank): one all_gather_into_tensor over NCCL; over gloo (CPU
    process groups, the 1-GPU multi-rank tests) through host memory. Needs equal head
    counts per rank (n_groups % world == 0)."""
    import torch.distributed as dist
    if world == 1:
        return local.clone()
    backend = dist.get_backend(group)
    if backend == "nccl":
        full = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(full, local.contiguous(), group=group)
        return full
    host = local.detach().cpu().contiguous()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(local.device)

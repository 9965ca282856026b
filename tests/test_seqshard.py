"""Sequence-sharded decode (C5): shard geometry, the per-stage score all-gather +
global selection, and the log-sum-exp merge of the shards' (m, l, o).

CPU (gloo, world size 2, real all_gather): the host logic — assembling the gathered
scores, each rank's slice of the global selection, the merge math.
GPU (one device, the shards driven in-process): stage selections, final masks and the
merged output against the unsharded fused decode layer — indices exact, output within
the fp32 tolerance (only the summation order differs).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2502_08910_b200 import seqshard as S  # noqa: E402


def test_geometry_partitions_the_middle_range():
    for world in (1, 2, 3, 8):
        geos = [S.ShardGeometry(t=3 * 2 ** 20, sink=256, stream=1024, lc1=256, world=world, rank=r)
                for r in range(world)]
        ranges = [g.chunk_range() for g in geos]
        assert ranges[0][0] == 0 and ranges[-1][1] == geos[0].cc1
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        toks = [g.token_range() for g in geos]
        assert toks[0][0] == 0 and toks[-1][1] == 3 * 2 ** 20
        assert all(a[1] == b[0] for a, b in zip(toks, toks[1:]))
        assert all(t0 % 64 == 0 for t0, _ in toks)  # page aligned
        assert sum(g.local_stage1()[1] for g in geos) == geos[0].n0


def _reference_topk(scores: np.ndarray, k: int) -> np.ndarray:
    order = sorted(range(len(scores)), key=lambda j: (-scores[j], j))
    return np.sort(np.asarray(order[:k]))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        M, lc = 3, 32
        counts = torch.randint(5, 40, (world, M), generator=g)
        full = [torch.randn(int(counts[:, m].sum()), generator=g) for m in range(M)]
        starts = torch.cumsum(counts, 0) - counts
        W = int(counts.max())
        mine = torch.full((M, W), float("-inf"))
        for m in range(M):
            a, n = int(starts[rank, m]), int(counts[rank, m])
            mine[m, :n] = full[m][a:a + n]
        gathered = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        gc = [torch.empty_like(counts[rank]) for _ in range(world)]
        dist.all_gather(gc, counts[rank].contiguous())
        glob = S.assemble(torch.stack(gathered), torch.stack(gc), world * W)
        ok = all(torch.equal(glob[m, : full[m].numel()], full[m]) for m in range(M))
        # global selection (reference stable top-K) -> this rank's slice
        K = 8
        sel = torch.stack([torch.from_numpy(_reference_topk(full[m].numpy(), K)) for m in range(M)])
        loc, inside, below = S.local_part(sel, torch.full((M,), K), starts[rank], counts[rank])
        mine_sel = [(loc[m, : int(inside[m])] + starts[rank, m]).tolist() for m in range(M)]
        allsel = [None] * world
        dist.all_gather_object(allsel, mine_sel)
        ok &= all(sum((allsel[r][m] for r in range(world)), []) == sel[m].tolist() for m in range(M))
        # merge: shards' (m, l, o) of one softmax over the union == the unsharded softmax
        n, d = 4, 16
        s_all = torch.randn(n, 64, generator=g)
        v_all = torch.randn(64, d, generator=g)
        part = torch.arange(64) % world == rank
        s = s_all[:, part]
        mm = s.max(1).values
        p = torch.exp(s - mm.unsqueeze(1))
        ll = p.sum(1)
        oo = (p @ v_all[part]) / ll.unsqueeze(1)
        gm = [torch.empty_like(mm) for _ in range(world)]; dist.all_gather(gm, mm)
        gl = [torch.empty_like(ll) for _ in range(world)]; dist.all_gather(gl, ll)
        go = [torch.empty_like(oo) for _ in range(world)]; dist.all_gather(go, oo)
        merged = S.lse_merge_reference(torch.stack(gm), torch.stack(gl), torch.stack(go))
        want = torch.softmax(s_all, 1) @ v_all
        ok &= bool(torch.allclose(merged, want, rtol=1e-5, atol=1e-6))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_host_logic_over_gloo_world2():
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
@pytest.mark.parametrize("world,groups,t", [(2, 8, 1 << 18), (4, 8, 1 << 18), (8, 8, 1 << 18),
                                           (8, 1, 3 << 20)])  # last: the C5 context (3M) of one KV group
def test_sharded_decode_matches_unsharded(world, groups, t):
    from paper_2502_08910_b200 import _capi, device as D, synth
    import ctypes as C
    D.require_cuda()
    hpm, d = 4, 128
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    q, k, v = synth.generate(groups * hpm, groups, t, d, t_q=2, seed=9)
    full = D.FusedDecodeLayer(D.PagedKV(k, v), stages, sink=256, stream_tokens=1024,
                              n_q_heads=groups * hpm, n_masks=groups)
    full.q.copy_(q[:, 0])
    want = full.run(t).clone()
    shards = []
    for r in range(world):
        geo = S.ShardGeometry(t=t, sink=256, stream=1024, lc1=256, world=world, rank=r)
        t0, t1 = geo.token_range()
        ly = S.SeqShardLayer(geo, k[:, t0:t1], v[:, t0:t1], stages, n_q_heads=groups * hpm, n_masks=groups)
        ly.q.copy_(q[:, 0])
        shards.append(ly)
    got = S.run_step_virtual(shards, t - 1)
    torch.cuda.synchronize()
    # every rank holds the same global selection per stage, equal to the unsharded one
    for i in range(3):
        K = full.sel[i].shape[1]
        for ly in shards:
            assert torch.equal(ly.sel_g[i][:, :K], full.sel[i]), f"stage {i}"
            assert torch.equal(ly.cnt_g[i], full.count[i]), f"stage {i} count"
    # the final token lists, assembled over the shards, equal the unsharded cache
    lists = []
    for ly in shards:
        ref = ly._in_ref(2)
        from paper_2502_08910_b200.device import _ref_push
        ref = _ref_push(ref, ly.sel_l[-1], stages[-1][1])
        out = torch.zeros((groups, 2048), dtype=torch.int32, device="cuda")
        refs = (_capi.ListRef * 1)(ref)
        cnts = (C.c_void_p * 1)(ly.len_l[-1].data_ptr())
        outs = (C.c_void_p * 1)(out.data_ptr())
        strides = (C.c_int64 * 1)(2048)
        _capi.check(_capi.lib().hp_decode_materialize(refs, cnts, outs, strides, 1, groups, 2048, None))
        torch.cuda.synchronize()
        lists.append([out[m, : int(ly.len_l[-1][m])].tolist() for m in range(groups)])
    cl, cc = full.mask()
    for m in range(groups):
        assert sum((lists[r][m] for r in range(world)), []) == cl[m, : int(cc[m])].tolist()
    err = (got - want).abs().max().item() / want.abs().max().item()
    assert err <= 1e-3, err


def _run_step_worker(rank, world, port, q, t, groups):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_08910_b200 import device as D, synth
        torch.cuda.set_device(0)
        hpm, d = 4, 128
        stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
        qq, k, v = synth.generate(groups * hpm, groups, t, d, seed=31)
        geo = S.ShardGeometry(t=t, sink=256, stream=1024, lc1=256, world=world, rank=rank)
        t0, t1 = geo.token_range()
        ly = S.SeqShardLayer(geo, k[:, t0:t1], v[:, t0:t1], stages, n_q_heads=groups * hpm, n_masks=groups)
        ly.q.copy_(qq[:, 0])
        got = S.run_step(ly, t - 1)  # the real multi-rank driver: all-gathers over the process group
        full = D.FusedDecodeLayer(D.PagedKV(k, v), stages, sink=256, stream_tokens=1024,
                                  n_q_heads=groups * hpm, n_masks=groups)
        full.q.copy_(qq[:, 0])
        want = full.run(t)
        torch.cuda.synchronize()
        ok = True
        for i in range(3):
            K = full.sel[i].shape[1]
            ok &= bool(torch.equal(ly.sel_g[i][:, :K], full.sel[i])) and bool(torch.equal(ly.cnt_g[i], full.count[i]))
        err = ((got - want).abs().max() / want.abs().max()).item()
        q.put((rank, (ok and err <= 1e-3, err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("t,groups", [(1 << 18, 8), (300_001, 2)])  # uneven chunk split across the ranks
def test_run_step_multirank_world2(t, groups):
    """seqshard.run_step with two real ranks (both on cuda:0, gloo): every stage's global
    selection equals the unsharded layer's, the merged output within 1e-3."""
    import socket
    import torch.multiprocessing as mp
    geo = S.ShardGeometry(t=t, sink=256, stream=1024, lc1=256, world=2, rank=0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run_step_worker, args=(r, 2, port, q, t, groups)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] for r in res.values()), (res, geo.cc1)


@pytest.mark.gpu
def test_c5_3m_selection_matches_oracle(port):
    """C5 context (3M tokens), one KV group, 8 virtual shards: the sharded step's final mask
    equals the CPU oracle's (pruning.cpp:153-200 chained as decode.cpp:225-249)."""
    from paper_2502_08910_b200 import synth
    import ctypes as C
    from paper_2502_08910_b200 import _capi
    from paper_2502_08910_b200.device import _ref_push
    t, groups, hpm, world = 3 << 20, 1, 4, 8
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    qq, k, v = synth.generate(groups * hpm, groups, t, 128, seed=41)
    shards = []
    for r in range(world):
        geo = S.ShardGeometry(t=t, sink=256, stream=1024, lc1=256, world=world, rank=r)
        t0, t1 = geo.token_range()
        ly = S.SeqShardLayer(geo, k[:, t0:t1], v[:, t0:t1], stages, n_q_heads=groups * hpm, n_masks=groups)
        ly.q.copy_(qq[:, 0])
        shards.append(ly)
    got = S.run_step_virtual(shards, t - 1)
    torch.cuda.synchronize()
    mask = []
    for ly in shards:
        ref = _ref_push(ly._in_ref(2), ly.sel_l[-1], stages[-1][1])
        out = torch.zeros((groups, 2048), dtype=torch.int32, device="cuda")
        _capi.check(_capi.lib().hp_decode_materialize((_capi.ListRef * 1)(ref), (C.c_void_p * 1)(ly.len_l[-1].data_ptr()),
                                                      (C.c_void_p * 1)(out.data_ptr()), (C.c_int64 * 1)(2048), 1,
                                                      groups, 2048, None))
        torch.cuda.synchronize()
        mask += out[0, : int(ly.len_l[-1][0])].tolist()
    masks, want, _ = port.decode_layer_step(qq[:, 0].cpu().numpy().reshape(1, hpm, 128), k.float().cpu().numpy(),
                                            v.float().cpu().numpy(), stages, sink=256, stream=1024)
    assert mask == masks[0].tolist()
    err = float(np.abs(got.cpu().numpy().reshape(1, hpm, 128) - want).max() / np.abs(want).max())
    assert err <= 1e-3, err

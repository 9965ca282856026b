"""KV-group sharded decode (C3 on 1/2/4/8 GPUs): rank r owns contiguous
KV groups of every layer; no data-path collective.

CPU: the group partition, and the output all-gather over gloo with world size 2.
GPU (two processes sharing cuda:0, gloo): each rank runs its groups of an 8-group decode
step; its masks equal the unsharded run's for those groups, and the gathered outputs
equal the unsharded output (fp32 summation order only: the persistent grid's split per
group depends on how many groups share the GPU)."""
from __future__ import annotations

import os
import socket

import pytest

torch = pytest.importorskip("torch")

from paper_2502_08910_b200 import kvshard as K  # noqa: E402


def test_group_range_partitions_the_groups():
    for n, world in [(8, 1), (8, 2), (8, 4), (8, 8), (8, 3), (5, 2)]:
        rs = [K.group_range(n, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        K.group_range(4, 8, 0)


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def _gather_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = torch.full((4, 8), float(rank)) + torch.arange(8.0)
        full = K.gather_outputs(local, world)
        want = torch.cat([torch.full((4, 8), float(r)) + torch.arange(8.0) for r in range(world)])
        q.put((rank, bool(torch.equal(full, want))))
    finally:
        dist.destroy_process_group()


def test_gather_outputs_over_gloo_world2():
    assert _spawn(_gather_worker, 2) == {0: True, 1: True}


def _decode_worker(rank, world, port, q, t):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_08910_b200 import device as D, synth
        torch.cuda.set_device(0)
        groups, hpm, d = 8, 4, 128
        stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
        q_, k, v = synth.generate(groups * hpm, groups, t, d, seed=21)
        shard = K.KvGroupShardLayer(k, v, stages, sink=256, stream_tokens=1024, n_groups=groups,
                                    heads_per_group=hpm, world=world, rank=rank)
        shard.set_q(q_[:, 0])
        shard.run(t)
        out = shard.gather()
        full = D.FusedDecodeLayer(D.PagedKV(k, v), stages, sink=256, stream_tokens=1024,
                                  n_q_heads=groups * hpm, n_masks=groups)
        full.q.copy_(q_[:, 0])
        want = full.run(t)
        torch.cuda.synchronize()
        ok = True
        for i in range(3):  # this rank's groups: every stage cache exact
            cl, cc = shard.layer.mask(i)
            fl, fc = full.mask(i)
            for gl, g in enumerate(range(shard.g0, shard.g1)):
                n = int(cc[gl])
                ok &= n == int(fc[g]) and torch.equal(cl[gl, :n], fl[g, :n])
        err = ((out - want).abs().max() / want.abs().max()).item()
        ok &= err <= 1e-5
        q.put((rank, (ok, err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_kvshard_world2_matches_unsharded():
    res = _spawn(_decode_worker, 2, 1 << 17)
    assert all(r[0] for r in res.values()), res

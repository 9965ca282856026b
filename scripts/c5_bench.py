"""C5 timing on one B200: a 3M-token decode layer (Llama-3.1-8B shape: 8 KV groups x 4
q-heads, d = 128, bf16, 3k preset) (a) unsharded — FusedDecodeLayer, full-refresh step —
and (b) sequence-sharded over 8 virtual ranks in this process (seqshard.run_step_virtual:
every shard's descents, the global selections, every shard's BSA and the LSE merge run
back to back on the one GPU, the collectives replaced by stacks). (b) / 8 is the device
work one rank of the 8-GPU split does per layer (timed as one CUDA graph of the whole
virtual step), before the all-gathers (3 x 8 x 4 KB of scores + 8 x 16 KB of partials
per layer). L2 flushed before every step.
Dev tool: python scripts/c5_bench.py [T]"""
import json
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, seqshard as S, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 3 << 20
groups, hpm, d, world = 8, 4, 128, 8
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
sink, stream = 256, 1024
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, steps=10, warmup=3):
    ts = []
    for i in range(warmup + steps):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= warmup:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


res = {"t": t, "groups": groups, "heads": groups * hpm, "world": world}
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=3)
# (a) unsharded
layer = D.FusedDecodeLayer(D.PagedKV(k, v, page_size=64), stages, sink=sink, stream_tokens=stream,
                           n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
res["unsharded_full_refresh_us"] = timed(lambda: layer.run(t, materialize=False))
out_ref = layer.out.clone()
del layer
# (b) 8 virtual ranks
geos = [S.ShardGeometry(t=t, sink=sink, stream=stream, lc1=stages[0][1], world=world, rank=r) for r in range(world)]
shards = []
for g in geos:
    t0, t1 = g.token_range()
    ly = S.SeqShardLayer(g, k[:, t0:t1], v[:, t0:t1], stages, n_q_heads=groups * hpm, n_masks=groups)
    ly.q.copy_(q.view(ly.q.shape))
    shards.append(ly)
del k, v
res["sharded_8_virtual_step_us_eager"] = timed(lambda: S.run_step_virtual(shards, t - 1))
# the same step captured in one CUDA graph (no host launch gaps between the shards' kernels)
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs):
    S.run_step_virtual(shards, t - 1)
torch.cuda.current_stream().wait_stream(cs)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=cs):
    S.run_step_virtual(shards, t - 1)
res["sharded_8_virtual_step_us"] = timed(graph.replay)
res["per_rank_us"] = res["sharded_8_virtual_step_us"] / world
out = S.run_step_virtual(shards, t - 1)
torch.cuda.synchronize()
res["sharded_vs_unsharded_rel_err"] = ((out - out_ref).abs().max() / out_ref.abs().max()).item()
print(json.dumps(res))

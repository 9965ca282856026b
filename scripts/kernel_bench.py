"""Marginal per-launch time of each decode kernel at C3 (1M, 8 groups): graphs of N
back-to-back launches of one piece of the layer step (L2 flushed before each replay).
Dev tool: python scripts/kernel_bench.py [T]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
groups, hpm, d = (int(sys.argv[2]) if len(sys.argv) > 2 else 8), 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64)
del k, v
import os
ext = os.environ.get("EXT") == "1"
rope = D.RopeTable(t + 2, d) if ext else None
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups,
                           policy=D.RopePolicy(extension=ext), rope=rope)
layer.q.copy_(q.view(layer.q.shape))
layer.run(t)
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
N = 8
pieces = {
    "s1 descent": lambda: layer.run_stage(t, 0, select=False),
    "s1 descent+topk": lambda: layer.run_stage(t, 0),
    "s2 descent": lambda: layer.run_stage(t, 1, select=False),
    "s2 descent+topk": lambda: layer.run_stage(t, 1),
    "s3 descent": lambda: layer.run_stage(t, 2, select=False),
    "s3 descent+topk": lambda: layer.run_stage(t, 2),
    "bsa": lambda: layer.run(t, refresh=[False] * 3, materialize=False),
    "full step": lambda: layer.run(t),
    "full no-mat": lambda: layer.run(t, materialize=False),
}
s = torch.cuda.Stream()
for name, fn in pieces.items():
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(N):
            fn()
    ts = []
    for _ in range(10):
        flush.zero_(); sink.copy_(flush_rd.view(torch.int64).sum().view(1))
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / N)
    ts.sort()
    print(f"{name:18s} {ts[len(ts)//2]:8.2f} us per launch (graph of {N}, median)")

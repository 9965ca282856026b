"""Which graph-captured decode piece fails under ncu (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth

t, groups = 1 << 20, 8
q, k, v = synth.generate(groups * 4, groups, t, 128, seed=1)
kv = D.PagedKV(k, v, page_size=64)
layer = D.FusedDecodeLayer(kv, [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)], sink=256,
                           stream_tokens=1024, n_q_heads=groups * 4, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
layer.run(t)
torch.cuda.synchronize()
piece = sys.argv[1]
fns = {"s1": lambda: layer.run_stage(t, 0), "s1d": lambda: layer.run_stage(t, 0, select=False),
       "s2": lambda: layer.run_stage(t, 1), "s3": lambda: layer.run_stage(t, 2),
       "bsa": lambda: layer.run(t, refresh=[False] * 3, materialize=False)}
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    fns[piece]()
    fns[piece]()
g.replay()
torch.cuda.synchronize()
print(piece, "ok")

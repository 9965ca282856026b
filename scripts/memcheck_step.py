"""One fused decode layer step (optionally a graph replay with the side-branch caches)
for compute-sanitizer. Dev tool: python scripts/memcheck_step.py [T] [groups]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 8
q, k, v = synth.generate(groups * 4, groups, t, 128, seed=1)
kv = D.PagedKV(k, v, page_size=64)
layer = D.FusedDecodeLayer(kv, [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)], sink=256,
                           stream_tokens=1024, n_q_heads=groups * 4, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
side = torch.cuda.Stream()
for fl in ([True] * 3, [False, True, True], [False] * 3, [True] * 3):
    layer.run(t, refresh=fl, mat_stream=side)
    torch.cuda.synchronize()
print("ok", layer.out.float().abs().sum().item())
if len(sys.argv) > 3:  # also capture the step as a graph (bench.py's shape) and replay it
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        side.wait_stream(stream)
        layer.run(t, mat_stream=side if sys.argv[3] == "side" else None)
        stream.wait_stream(side)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    print("graph ok", layer.out.float().abs().sum().item())

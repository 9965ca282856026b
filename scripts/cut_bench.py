"""Marginal time of kernel prefixes (dev build, HP_TRACE=1): graphs of N launches of
the BSA-only step (kernel id 2) with the kernel cut at successive points."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import _capi, device as D, synth

t = 1 << 20
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
del k, v
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
L = _capi.lib()
L.hp_debug_cut.argtypes = [C.c_int, C.c_int]
layer.run(t)
torch.cuda.synchronize()
N = 8
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    layer.run(t, refresh=[False] * 3)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(N):
        layer.run(t, refresh=[False] * 3)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 2
stage_of = {5: 2, 3: int(sys.argv[3]) if len(sys.argv) > 3 else 0}
if kid == 3:  # a stage's top-k kernel (descent + top-k launched; the cut applies to top-k)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(N):
            layer.run_stage(t, stage_of[3])
if kid == 5:  # stage-3 descent (all-rows kernel)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(N):
            layer.run_stage(t, 2, select=False)
for cut in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,5,6,7,1,2,3,4,-1").split(",")]:
    _capi.check(L.hp_debug_cut(kid, cut))
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / N)
    ts.sort()
    print(f"kernel {kid} cut at {cut:2d}: {ts[len(ts)//2]:7.2f} us per launch (graph of {N})")

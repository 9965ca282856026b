"""Quick per-phase timing of the decode layer step at C2/C3 shapes (dev tool).
usage: quick_perf.py T [--ncu]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
ncu = "--ncu" in sys.argv
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
t0 = time.time()
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
del k, v
torch.cuda.synchronize()
print(f"gen {time.time()-t0:.1f}s", flush=True)
fused = "--generic" not in sys.argv
layer = (D.FusedDecodeLayer if fused else D.DecodeLayer)(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
flush_out = torch.empty(1, dtype=torch.int64, device="cuda")
def do_flush(mode):
    if mode in ("w", "wr"):
        flush.zero_()
    if mode == "wr":  # evict the dirty lines: the timed step starts with a clean, cold L2
        flush_out.copy_(flush_rd.view(torch.int64).sum().view(1))
variants = {"full": [True] * 3, "s23_bsa": [False, True, True], "s3_bsa": [False, False, True],
            "bsa": [False] * 3}
for _ in range(3):
    layer.run(t)
torch.cuda.synchronize()
if ncu:
    for name, fl in variants.items():
        layer.run(t, refresh=fl)
    torch.cuda.synchronize()
    sys.exit(0)
graphs = {}
s = torch.cuda.Stream()
for name, fl in variants.items():
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.run(t, refresh=fl)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.run(t, refresh=fl)
    graphs[name] = g
torch.cuda.synchronize()
def timeit(g, n=20, mode="w"):
    ts = []
    for _ in range(n):
        do_flush(mode)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]
# marginal cost: a graph with the BSA-only step twice, and one with a trivial kernel
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    layer.run(t, refresh=[False] * 3)
torch.cuda.current_stream().wait_stream(s)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    layer.run(t, refresh=[False] * 3)
    layer.run(t, refresh=[False] * 3)
graphs["bsa_x2"] = g2
tiny = torch.zeros(1, device="cuda")
g0 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g0):
    tiny.add_(1)
graphs["trivial"] = g0
for mode in ("w", "wr", "none"):
    for name, g in graphs.items():
        print(f"{name:10s} graph us (median, flush={mode}): {timeit(g, mode=mode):8.1f}")
print("counts", [c.view(-1).tolist()[:2] for c in layer.count] if fused else "")

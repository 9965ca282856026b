"""Per refresh pattern: the fused layer (hp_decode_layer) vs the per-stage kernels at C3
(1M, 8 groups), graphs of N back-to-back layer steps, L2 flushed before each replay.
Dev tool: python scripts/layer_bench.py [T] [cluster sizes, e.g. 8,16]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth
from paper_2502_08910_b200._capi import lib

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
css = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]  # cluster sizes need a dev build (HP_VARIANT)
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64)
del k, v
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
N = 8
pats = {"full": [True] * 3, "s23": [False, True, True], "s3": [False, False, True], "bsa": [False] * 3}


def timeit(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(N):
            fn()
    ts = []
    for _ in range(15):
        flush.zero_(); sink.copy_(flush_rd.view(torch.int64).sum().view(1))
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / N)
    ts.sort()
    return ts[len(ts) // 2]


layer._fused = False
layer.run(t); torch.cuda.synchronize()
ref = {n: timeit(lambda fl=fl: layer.run(t, refresh=fl, materialize=False)) for n, fl in pats.items()}
print("per-stage  " + "  ".join(f"{n} {v:7.2f}" for n, v in ref.items()), flush=True)
m_ref = [c.clone() for c in layer.cache]
layer._fused = "always"
for cs in css:
    if hasattr(lib(), "hp_decode_layer_cluster"):
        lib().hp_decode_layer_cluster(cs)
    layer.run(t); torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(m_ref, layer.cache))
    res = {n: timeit(lambda fl=fl: layer.run(t, refresh=fl, materialize=False)) for n, fl in pats.items()}
    print(f"layer {'grid' if cs <= 0 else 'cs=' + str(cs):6s} " + "  ".join(f"{n} {v:7.2f}" for n, v in res.items()) + f"  caches==per-stage: {same}", flush=True)

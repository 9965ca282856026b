"""Quick per-phase timing of the decode layer step at C2/C3 shapes (dev tool)."""
import sys, time
import torch
from paper_2502_08910_b200 import device as D, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
torch.manual_seed(0)
t0 = time.time()
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
del k, v
torch.cuda.synchronize()
print(f"gen {time.time()-t0:.1f}s", flush=True)
layer = D.DecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, n=10):
    ts = []
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]
for _ in range(3): layer.run(t)
torch.cuda.synchronize()
print("full layer step us (median):", timeit(lambda: layer.run(t)))
print("bsa-only us:", timeit(lambda: layer.run(t, refresh=[False, False, False])))
print("stage3+bsa us:", timeit(lambda: layer.run(t, refresh=[False, False, True])))
print("stage2,3+bsa us:", timeit(lambda: layer.run(t, refresh=[False, True, True])))
print("counts", [c.view(-1).tolist() for _, c in layer.caches], layer.sel_count.view(-1).tolist())

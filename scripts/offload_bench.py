"""C3 with host-offloaded KV: one layer at T (default 1M) with the K/V in pinned host
memory behind the on-GPU LRU page cache (CachedKV, `frac` of the pages resident).
Runs the (16, 8, 4) refresh schedule for `steps` steps with a commit per step and
reports the mean step time, the hit ratio, and the steady-state BSA-only step."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth
t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t, d, t_q=steps, seed=1)
kv = D.CachedKV(k, v, num_slots=int(frac * (t // 64)), page_size=64)
del k, v
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
refresh = [16, 8, 4]
ctr = [0, 0, 0]
times, kinds = [], []
for i in range(steps):
    layer.q.copy_(q[:, i])
    fl = [c == 0 for c in ctr]
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    layer.run(t, refresh=fl)
    kv.commit()
    b.record(); torch.cuda.synchronize()
    times.append(a.elapsed_time(b) * 1e3)
    kinds.append("".join("1" if f else "0" for f in fl))
    ctr = [(c + 1) % r for c, r in zip(ctr, refresh)]
st = kv.stats.cpu().tolist()
full = [x for x, kd in zip(times, kinds) if kd == "111"]
bsa = [x for x, kd in zip(times, kinds) if kd == "000"]
print(json.dumps({"t": t, "cache_frac": frac, "steps": steps, "mean_step_us": sum(times[4:]) / max(1, len(times[4:])),
                  "full_refresh_us": full, "bsa_only_us_median": sorted(bsa)[len(bsa) // 2] if bsa else None,
                  "hits": st[0], "misses": st[1], "evictions": st[2], "hit_ratio": st[0] / max(1, st[0] + st[1])}))

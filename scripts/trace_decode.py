"""Per-CTA phase timeline of the fused decode kernels at 1M ctx (dev tool).
Stage kernels trace as id 10 + l_c; the BSA kernel as id 2."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2502_08910_b200 import _capi, device as D, synth

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
groups, hpm, d = 8, 4, 128
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t, d, seed=1)
kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
del k, v
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
L = _capi.lib()
L.hp_trace_enable.argtypes = [C.c_void_p, C.c_int]
buf = torch.zeros((16384, 8), dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
flush_out = torch.empty(1, dtype=torch.int64, device="cuda")
mode = sys.argv[2] if len(sys.argv) > 2 else "w"
for _ in range(3):
    layer.run(t)
torch.cuda.synchronize()
names = {10 + 256: "stage1", 10 + 32: "stage2", 10 + 8: "stage3", 3: "topk(last stage)", 2: "bsa"}
for kid, name in names.items():
    buf.zero_()
    _capi.check(L.hp_trace_enable(buf.data_ptr(), kid))
    if mode in ("w", "wr"):
        flush.zero_()
    if mode == "wr":
        flush_out.copy_(flush_rd.view(torch.int64).sum().view(1))
    torch.cuda.synchronize()
    layer.run(t)
    torch.cuda.synchronize()
    _capi.check(L.hp_trace_enable(None, -1))
    ball = buf.cpu().numpy().astype(np.float64)
    b = ball[:8192]
    clk = ball[8192:]
    used = b[:, 0] > 0
    b = b[used]
    clk = clk[used]
    last = b[:, 5] > 0
    if last.any():
        dt = b[last][:, 5] - b[last][:, 4]
        dc = clk[last][:, 5] - clk[last][:, 4]
        print(f"  last-CTA tail: {dt.mean()/1000:.2f} us, {dc.mean():.0f} cycles -> {dc.mean()/dt.mean():.3f} GHz")
    dt = b[:, 2] - b[:, 0]
    dc = clk[:, 2] - clk[:, 0]
    print(f"  body: {dt.mean()/1000:.2f} us, {dc.mean():.0f} cycles -> {dc.mean()/dt.mean():.3f} GHz")
    t0 = b[:, 0].min()
    rel = np.where(b > 0, (b - t0) / 1000.0, np.nan)  # us
    print(f"== {name}: {used.sum()} CTAs traced")
    for s in range(8):
        col = rel[:, s]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"  slot {s}: n={col.size:5d} min {col.min():8.2f} p50 {np.median(col):8.2f} "
                  f"p90 {np.percentile(col, 90):8.2f} max {col.max():8.2f} us")
    dur = rel[:, 3 if name != "bsa" else 6] - rel[:, 0]
    dur = dur[~np.isnan(dur)]
    if dur.size:
        print(f"  per-CTA (0->ticket) p50 {np.median(dur):.2f} p90 {np.percentile(dur, 90):.2f} max {dur.max():.2f} us")

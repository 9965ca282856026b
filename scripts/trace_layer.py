"""Per-CTA phase timeline of the fused layer kernel (trace id 20) at 1M (dev tool; needs
the HP_TRACE=1 build). Slots: 0 start, 1 q loaded, 2..4 stage 0..2 selected, 5 BSA tiles
done, 6 merged, 7 exit."""
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
kv = D.PagedKV(k, v, page_size=64)
del k, v
layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
layer.q.copy_(q.view(layer.q.shape))
L = _capi.lib()
import os
# decode.cu kernels (ids < 20) trace through hp_trace_enable, the layer kernel through its own
_en = L.hp_trace_enable if int(os.environ.get("KID", "20")) < 20 else L.hp_layer_trace_enable
_en.argtypes = [C.c_void_p, C.c_int]
buf = torch.zeros((16384, 8), dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    layer.run(t)
torch.cuda.synchronize()
import os
kid = int(os.environ.get("KID", "20"))
for name, fl in {"full": [True] * 3, "s23": [False, True, True], "s3": [False, False, True], "bsa": [False] * 3}.items():
    for rep in range(2):
        buf.zero_()
        _capi.check(_en(buf.data_ptr(), kid))
        flush.zero_()
        torch.cuda.synchronize()
        layer.run(t, refresh=fl, materialize=False)
        torch.cuda.synchronize()
        _capi.check(_en(None, -1))
    ball = buf.cpu().numpy().astype(np.float64)
    used = ball[:8192, 0] > 0
    b = ball[:8192][used]
    ck = ball[8192:][used]
    if not len(b):
        print(f"== {name}: no CTA recorded trace {kid}")
        continue
    t0 = b[:, 0].min()
    rel = np.where(b > 0, (b - t0) / 1000.0, np.nan)
    crel = np.where(b > 0, ck - ck[:, :1], np.nan)  # cycles since the CTA's slot 0 (same SM)
    print(f"== {name}: {len(b)} CTAs")
    for s in range(8):
        col = rel[:, s]
        cc = crel[:, s]
        ok = ~np.isnan(col)
        if ok.any():
            print(f"  slot {s}: n={ok.sum():4d} min {col[ok].min():7.2f} p50 {np.median(col[ok]):7.2f} max {col[ok].max():7.2f} us"
                  f"   cycles since slot 0: p50 {np.median(cc[ok]):8.0f}")
    last = np.nanmax(np.where(b > 0, b, np.nan), axis=1) - b[:, 0]
    lastc = np.nanmax(np.where(b > 0, ck, np.nan), axis=1) - ck[:, 0]
    print(f"  clock: {np.median(lastc / np.maximum(last, 1)):.3f} GHz")

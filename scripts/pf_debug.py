import ctypes as C, sys, threading, time, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import _capi, device as D, synth
L = _capi.lib()
flag = torch.zeros(4, dtype=torch.int32).pin_memory()
L.hp_debug_prefill_progress.argtypes = [C.c_void_p]
_capi.check(L.hp_debug_prefill_progress(flag.data_ptr()))
def watch():
    last = None
    for i in range(60):
        time.sleep(0.5)
        v = int(flag[0])
        if v != last:
            print("progress", v, flush=True); last = v
    print("STALLED at", int(flag[0]), flush=True)
    os._exit(3)
groups, hpm = 1, 2
t_kv, t_q, bq, sink, stream = 512, 64, 64, 32, 64
stages = [(64, 8, 128)]
q, k, v = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=3)
kv = D.PagedKV(k, v, page_size=64)
lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups)
want = D.bsa(q, kv, *D.selected_indices(lists, counts, n_rows=t_q, block_size=bs, query_offset=off, sink=sink, stream_tokens=stream),
             query_offset=off, max_sel=sink + lists.shape[-1] + stream + 1)
torch.cuda.synchronize()
print("row path ok", flush=True)
threading.Thread(target=watch, daemon=True).start()
got = D.bsa_prefill_tc(q, kv, lists, counts, block_size=bs, query_offset=off, sink=sink, stream_tokens=stream)
try:
    torch.cuda.synchronize()
    print("tc ok; max|diff|", (want - got).abs().max().item(), "max|want|", want.abs().max().item(), "final progress", int(flag[0]), flush=True)
    print(want[0, -1, :6].tolist()); print(got[0, -1, :6].tolist())
    print(want[1, 3, :6].tolist()); print(got[1, 3, :6].tolist())
except Exception as e:
    print("ERROR", e, "progress", int(flag[0]), flush=True)
os._exit(0)

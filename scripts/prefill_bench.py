"""C4-style prefill timing: one 32K query chunk at T_kv = 128K (the last chunk of a 128K
chunked prefill), Llama-3.1-8B heads (32 q / 8 kv, d=128), 3k preset (b_q = 64).
Times build_mask (query-block pruning, CUDA cores, index-exact) and the block-sparse
attention on tcgen05 vs the CUDA-core row path; reports TFLOP/s of the tcgen05 BSA
(algorithmic flops = sum over rows of |selected| * d * 4 per q-head)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2502_08910_b200 import device as D, synth
t_kv = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
t_q = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 15
groups, hpm, d = 8, 4, 128
sink, stream = 256, 1024
stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
q, k, v = synth.generate(groups * hpm, groups, t_kv, d, t_q=t_q, seed=11)
kv = D.PagedKV(k, v, page_size=64)
del k, v
ws = D.Workspace()
def ev_time(fn, n=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)
res = {}
lists = counts = None
def mask():
    global lists, counts, bs, off
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups, ws=ws)
res["build_mask_ms"] = ev_time(mask)
sel, selc = D.selected_indices(lists, counts, n_rows=t_q, block_size=bs, query_offset=off, sink=sink, stream_tokens=stream)
n_sel = selc.double().sum().item() * hpm  # per q-head rows x selected
flops = n_sel * d * 4
out_tc = torch.empty_like(q)
res["bsa_tc_ms"] = ev_time(lambda: D.bsa_prefill_tc(q, kv, lists, counts, block_size=bs, query_offset=off, sink=sink,
                                                   stream_tokens=stream, out=out_tc))
out_row = torch.empty_like(q)
res["bsa_rowpath_ms"] = ev_time(lambda: D.bsa(q, kv, sel, selc, query_offset=off, max_sel=sel.shape[-1], out=out_row, ws=ws), n=1)
res["bsa_tflop"] = flops / 1e12
res["bsa_tc_tflops"] = flops / (res["bsa_tc_ms"] * 1e-3) / 1e12
res["tc_vs_row_rel_err"] = ((out_tc - out_row).abs().max() / out_row.abs().max()).item()
res.update(t_kv=t_kv, t_q=t_q, heads=groups * hpm)
print(json.dumps(res))

"""The CUDA path against the reference's OWN outputs (tests/golden/, produced by the
unmodified reference library on inputs from its own libstdc++ generator).
Masks must be identical; attention outputs within 1e-3 relative."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_golden.npz"


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def _rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(1e-6, np.abs(b).max())


@pytest.mark.parametrize("name", ["mb3", "k3", "smoke"])
@pytest.mark.parametrize("ext", [0, 1])
def test_build_mask_and_bsa_vs_reference(gold, name, ext):
    from paper_2502_08910_b200 import device as D
    D.require_cuda()
    dev = torch.device("cuda")
    q, k, v = gold[f"{name}_q"], gold[f"{name}_k"], gold[f"{name}_v"]
    stages = [tuple(int(x) for x in s) for s in gold[f"{name}_stages"]]
    sink, stream = (int(x) for x in gold[f"{name}_sink_stream"])
    nb, bs, off = (int(x) for x in gold[f"{name}_ext{ext}_nblocks"])
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=64, dtype=torch.float32)
    rope = D.RopeTable(k.shape[1] + 2, k.shape[2])
    policy = D.RopePolicy(extension=bool(ext))
    lists, counts, trace, dbs, doff = D.build_mask(torch.from_numpy(q).to(dev), kv, stages, sink=sink,
                                                   stream_tokens=stream, policy=policy, rope=rope)
    torch.cuda.synchronize()
    assert (lists.shape[1], dbs, doff) == (nb, bs, off)
    L, Cn = lists.cpu().numpy(), counts.cpu().numpy()
    for b in range(nb):
        assert np.array_equal(L[0, b, : Cn[0, b]], gold[f"{name}_ext{ext}_mask{b}"]), b
    for s, (tl, tc) in enumerate(trace):
        assert np.array_equal(tl[0, : int(tc[0])].cpu().numpy(), gold[f"{name}_ext{ext}_trace{s}"])
    sel, cnt = D.selected_indices(lists, counts, n_rows=q.shape[1], block_size=bs, query_offset=off,
                                  sink=sink, stream_tokens=stream)
    out = D.bsa(torch.from_numpy(q).to(dev), kv, sel, cnt, query_offset=off, max_sel=sel.shape[-1],
                policy=policy, rope=rope)
    torch.cuda.synchronize()
    assert _rel(out.cpu().numpy(), gold[f"{name}_ext{ext}_bsa"]) <= 1e-3


def test_decode_layer_vs_reference(gold):
    from paper_2502_08910_b200 import device as D
    D.require_cuda()
    dev = torch.device("cuda")
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 128)]
    q, k, v = gold["dec_q"], gold["dec_k"], gold["dec_v"]  # q [2 groups, 4, d=32]
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=64, dtype=torch.float32)
    layer = D.DecodeLayer(kv, stages, sink=128, stream_tokens=512, n_q_heads=8, n_masks=2)
    layer.q.copy_(torch.from_numpy(q.reshape(8, 1, 32)).to(dev))
    out = layer.run(k.shape[1]).clone()
    torch.cuda.synchronize()
    cl, cc = layer.caches[-1]
    for g in range(2):
        assert np.array_equal(cl[g, 0, : int(cc[g, 0])].cpu().numpy(), gold[f"dec_mask{g}"])
    assert _rel(out.cpu().numpy().reshape(2, 4, 32), gold["dec_out"]) <= 1e-3

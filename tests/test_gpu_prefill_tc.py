"""Prefill block-sparse attention on tcgen05 (hp_bsa_prefill) against the CUDA-core
row path (hp_bsa, itself checked against the reference within 1e-3) on the same
masks: Q and P enter the tensor cores as bf16, so the stated bf16 tolerance is 2e-2
relative (max |diff| / max |ref|)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
BF16_RTOL = 2e-2


def _D():
    from paper_2502_08910_b200 import device as D
    D.require_cuda()
    return D


@pytest.mark.parametrize("t_kv,t_q,bq,sink,stream,stages", [
    (4096, 1024, 64, 128, 512, [(64, 16, 512), (64, 4, 128)]),
    (8192, 2048, 64, 256, 1024, [(64, 64, 2048), (64, 16, 512), (64, 4, 256)]),
    (3000, 700, 32, 64, 256, [(32, 8, 256), (32, 4, 128)]),
])
def test_prefill_tc_matches_row_path(t_kv, t_q, bq, sink, stream, stages):
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm = 2, 4
    q, k, v = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=3)
    kv = D.PagedKV(k, v, page_size=64)
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups)
    assert bs == bq
    want = D.bsa(q, kv, *D.selected_indices(lists, counts, n_rows=t_q, block_size=bs, query_offset=off,
                                             sink=sink, stream_tokens=stream),
                 query_offset=off, max_sel=sink + lists.shape[-1] + stream + 1)
    got = D.bsa_prefill_tc(q, kv, lists, counts, block_size=bs, query_offset=off, sink=sink, stream_tokens=stream)
    torch.cuda.synchronize()
    w, g = want.double(), got.double()
    assert torch.isfinite(g).all()
    err = ((w - g).abs().max() / w.abs().max()).item()
    assert err <= BF16_RTOL, err

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


def test_prefill_tc_from_position_zero():
    """a prompt prefilled from position 0 (T_q == T_kv, query_offset 0)
    with sinks wider than a query block — rows must not attend to future sink tokens."""
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm, t = 2, 4, 2048
    stages = [(64, 16, 512), (64, 4, 128)]
    q, k, v = synth.generate(groups * hpm, groups, t, 128, t_q=t, seed=11)
    kv = D.PagedKV(k, v, page_size=64)
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=256, stream_tokens=256, n_masks=groups)
    assert off == 0
    want = D.bsa(q, kv, *D.selected_indices(lists, counts, n_rows=t, block_size=bs, query_offset=off,
                                             sink=256, stream_tokens=256),
                 query_offset=off, max_sel=256 + lists.shape[-1] + 256 + 1)
    got = D.bsa_prefill_tc(q, kv, lists, counts, block_size=bs, query_offset=off, sink=256, stream_tokens=256)
    torch.cuda.synchronize()
    w, g = want.double(), got.double()
    err = ((w - g).abs().max() / w.abs().max()).item()
    assert err <= BF16_RTOL, err
    # row 0 sees only token 0: its output is v[0] exactly (up to bf16 P rounding)
    v0 = v[0, 0].double()
    assert ((g[0, 0] - v0).abs().max() / v0.abs().max()).item() <= BF16_RTOL


@pytest.mark.parametrize("t_kv,t_q,stages,sink,stream", [
    (8192, 2048, [(64, 64, 2048), (64, 16, 512), (64, 4, 256)], 256, 1024),
    # reduced C4: the 3k preset on a 4K-row chunk at 40K context (stage 1 active for late blocks)
    (40960, 4096, [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)], 256, 1024),
])
def test_prefill_mask_and_tc_vs_oracle(port, t_kv, t_q, stages, sink, stream):
    """Prefill against the CPU oracle: build_mask lists index-exact per KV group
    (pruning.cpp:202-313), and the tcgen05 BSA within the bf16 tolerance of the oracle's
    block_sparse_attention (sparse_attention.cpp:114-145) on the same masks."""
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm = 2, 4
    q, k, v = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=5)
    kv = D.PagedKV(k, v, page_size=64)
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups)
    got = D.bsa_prefill_tc(q, kv, lists, counts, block_size=bs, query_offset=off, sink=sink, stream_tokens=stream)
    torch.cuda.synchronize()
    qh, kh, vh = q.cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy()
    L, Cn = lists.cpu().numpy(), counts.cpu().numpy()
    g_out = got.cpu().numpy()
    for g in range(groups):
        want_lists, _, wbs, woff = port.build_mask(qh[g * hpm:(g + 1) * hpm], kh[g:g + 1], stages,
                                                   sink=sink, stream=stream, threads=8)
        assert (wbs, woff) == (bs, off)
        assert len(want_lists) == L.shape[1]
        for b, wl in enumerate(want_lists):
            assert np.array_equal(L[g, b, : Cn[g, b]], wl), (g, b)
        want = port.block_sparse_attention(qh[g * hpm:(g + 1) * hpm], kh[g:g + 1], vh[g:g + 1], want_lists,
                                           block_size=bs, sink=sink, stream=stream, offset=off)
        og = g_out[g * hpm:(g + 1) * hpm].astype(np.float64)
        err = np.abs(og - want).max() / np.abs(want).max()
        assert err <= BF16_RTOL, (g, err)

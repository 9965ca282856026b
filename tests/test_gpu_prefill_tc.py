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
    D.PRUNE_VARIANTS_USED.clear()
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups)
    assert set(D.PRUNE_VARIANTS_USED) == {1}  # every stage on the tensor-core descent
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


def _masks_vs_oracle(port, D, q, k, stages, sink, stream, groups, hpm):
    kv = D.PagedKV(k, k, page_size=64)
    lists, counts, _, bs, off = D.build_mask(q, kv, stages, sink=sink, stream_tokens=stream, n_masks=groups)
    torch.cuda.synchronize()
    qh, kh = q.cpu().numpy(), k.float().cpu().numpy()
    L, Cn = lists.cpu().numpy(), counts.cpu().numpy()
    for g in range(groups):
        want_lists, _, wbs, woff = port.build_mask(qh[g * hpm:(g + 1) * hpm], kh[g:g + 1], stages,
                                                   sink=sink, stream=stream, threads=8)
        assert (wbs, woff) == (bs, off)
        for b, wl in enumerate(want_lists):
            assert np.array_equal(L[g, b, : Cn[g, b]], wl), (g, b)


@pytest.mark.parametrize("period", [97, 5])
def test_tc_descent_near_ties_exact(port, period):
    """The tensor-core descent's certified comparisons and top-K boundary under massive
    ties: keys repeat with a short period, so most branch comparisons and most chunk
    scores are exactly equal (every one undecided by the bound) — the exact re-decisions
    and the boundary replay must still give the reference's lists (strict '>', lowest
    chunk index first)."""
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm, t_kv, t_q = 2, 4, 8192, 512
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 256)]
    q, k, _ = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=21)
    idx = torch.arange(t_kv, device=k.device) % period
    k = k[:, idx].contiguous()
    D.PRUNE_VARIANTS_USED.clear()
    _masks_vs_oracle(port, D, q, k, stages, 256, 1024, groups, hpm)
    assert set(D.PRUNE_VARIANTS_USED) == {1}


def test_tc_descent_mixed_precision_heads(port):
    """One head's q rows are not bf16-exact: that head's CTAs score with the separately
    rounded fp32 dots, the others on the tensor cores, and the boundary replay uses each
    head's own exact arithmetic."""
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm, t_kv, t_q = 2, 4, 8192, 512
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 256)]
    q, k, _ = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=23)
    q[1] += 1e-3 * torch.randn_like(q[1])  # head 1 (group 0) in full fp32
    _masks_vs_oracle(port, D, q, k, stages, 256, 1024, groups, hpm)


_C4_MASKS = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2502_08910_b200 import device as D, synth
q, k, v = synth.generate(32, 8, 1 << 17, 128, t_q=1 << 15, seed=11)
kv = D.PagedKV(k, v, page_size=64)
lists, counts, _, bs, off = D.build_mask(q, kv, [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)],
                                         sink=256, stream_tokens=1024, n_masks=8)
np.savez({out!r}, lists=lists.cpu().numpy(), counts=counts.cpu().numpy(),
         variants=np.array(list(D.PRUNE_VARIANTS_USED)))
"""


def test_tc_descent_equals_cuda_core_at_c4(tmp_path):
    """C4 size (a 32K-row chunk at 128K, 8 KV groups, the 3k preset): every list of the
    tensor-core build_mask equals the CUDA-core descent's (HP_TC_DESCENT=0, itself
    index-exact against the oracle) — two independent exact paths at full size."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for name, env in (("tc", "1"), ("cc", "0")):
        out = str(tmp_path / f"{name}.npz")
        subprocess.run([sys.executable, "-c", _C4_MASKS.format(root=root, out=out)], check=True,
                       env={**os.environ, "HP_TC_DESCENT": env}, timeout=600)
        res[name] = np.load(out)
    assert set(res["tc"]["variants"]) == {1} and set(res["cc"]["variants"]) == {0}
    assert np.array_equal(res["tc"]["counts"], res["cc"]["counts"])
    c = res["tc"]["counts"]
    lt, lc = res["tc"]["lists"], res["cc"]["lists"]
    for g in range(c.shape[0]):
        for b in range(c.shape[1]):
            assert np.array_equal(lt[g, b, : c[g, b]], lc[g, b, : c[g, b]]), (g, b)


@pytest.mark.parametrize("t_kv,t_q,stages", [
    (8192, 500, [(64, 64, 2048), (64, 16, 512), (64, 4, 256)]),   # last block: 52 rows
    (6000, 333, [(32, 32, 1024), (32, 8, 256), (16, 4, 128)]),    # b_q 32 -> 16 remap, ragged tail
    (9000, 777, [(64, 128, 4096), (32, 16, 512)]),                # 128-token chunks, ragged everything
])
def test_tc_descent_ragged_blocks_exact(port, t_kv, t_q, stages):
    """Tensor-core descent at ragged shapes: a short last query block (fewer q rows than the
    MMA's n-tiles), b_q = 32 and 16 (rows >= 16 still take the tensor cores), a sub-block
    remap between stages, a context that is no multiple of the chunk size."""
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm = 2, 4
    q, k, _ = synth.generate(groups * hpm, groups, t_kv, 128, t_q=t_q, seed=t_q)
    D.PRUNE_VARIANTS_USED.clear()
    _masks_vs_oracle(port, D, q, k, stages, 128, 512, groups, hpm)
    assert 1 in set(D.PRUNE_VARIANTS_USED)

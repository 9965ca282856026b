"""Mask quality on the GPU path: the reference's quality
harness — recall of the pruned mask vs the exact top-k and vs a random equal-budget
set (commands.cpp:222-270, acceptance #3 `recall_dominance`) and planted-needle
retention (acceptance #4 `needle_retention`, acceptance.cpp:110-142) — restated
over the device path, first through the drop-in API at the reference's own sizes,
then on the fused decode path at 1M context where the CPU oracle is too slow.

The checker (softmax mass, exact top-k) is computed with torch on the device in
fp32; the masks come from the product kernels."""
import math

import numpy as np
import pytest
import torch

from paper_2502_08910_b200 import hipprune as hp

pytestmark = pytest.mark.gpu


def _recall(sel, q, keys):
    """attention_recall (sparse_attention.cpp:147-175): softmax mass of `sel` under q."""
    s = keys @ q / math.sqrt(q.numel())
    w = torch.softmax(s.double(), dim=0)
    return float(w[sel].sum())


def test_needle_retention_acceptance4():
    """acceptance.cpp:110-142: 100 seeds, 8192 keys, d 64, needle at 4096 with strength
    100, 3k preset without extension; every trial certified by the exact top-1 and the
    needle must survive every stage in >= 99 of them."""
    kept = 0
    for seed in range(100):
        w = hp.generate(heads=2, layers=1, seq_kv=8192, seq_q=64, dim=64, seed=7000 + seed,
                        needles=[(4096, 100.0)])
        for h in range(2):
            assert hp.exact_topk(w.q(0, h)[63], w.k(0, h), 1) == [4096]
        mask = hp.build_mask(w, 0, preset="3k", extension=False)
        kept += 4096 in set(mask.indices[-1])
    assert kept >= 99


def test_recall_dominance_acceptance3():
    """acceptance.cpp:97-107: 1 head, 8192 keys, d 64, 20 seeds, one query row at the
    end; the mask's attention mass beats a random equal-budget set by >= 0.1 on average
    and never exceeds the exact top-k of the same size."""
    rng = np.random.default_rng(0)
    margins = []
    for seed in range(1, 21):
        w = hp.generate(heads=1, layers=1, seq_kv=8192, seq_q=1, dim=64, seed=seed)
        mask = hp.build_mask(w, 0, preset="3k", extension=False)
        sel = hp.selected_indices(mask, 0)
        q = torch.from_numpy(np.ascontiguousarray(w.q(0, 0)[0])).double()
        keys = torch.from_numpy(np.ascontiguousarray(w.k(0, 0))).double()
        r_mask = _recall(torch.tensor(sel), q, keys)
        r_top = hp.attention_recall(hp.exact_topk(w.q(0, 0)[0], w.k(0, 0), len(sel)), w.q(0, 0)[0], w.k(0, 0))
        r_rand = _recall(torch.from_numpy(rng.choice(8192, len(sel), replace=False)), q, keys)
        assert r_mask <= r_top + 1e-9
        assert abs(r_mask - hp.attention_recall(sel, w.q(0, 0)[0], w.k(0, 0))) < 1e-6  # fp32 scores there
        margins.append(r_mask - r_rand)
    assert float(np.mean(margins)) >= 0.1


@pytest.fixture(scope="module")
def fused_1m():
    """Llama-3.1-8B head shape (32 q / 8 kv, d 128) at 1M tokens, bf16, 3k preset."""
    from paper_2502_08910_b200 import device as D, synth
    t, groups, hpm = 1 << 20, 8, 4
    q, k, v = synth.generate(groups * hpm, groups, t, 128, seed=11)
    kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
    layer = D.FusedDecodeLayer(kv, [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)], sink=256,
                               stream_tokens=1024, n_q_heads=groups * hpm, n_masks=groups)
    yield D, t, groups, hpm, q, k, kv, layer


def _selected(layer, g, t):
    cl, cc = layer.mask()
    mid = cl[g, : int(cc[g])].long()
    return torch.cat([torch.arange(256, device=mid.device), mid, torch.arange(t - 1024, t, device=mid.device)])


def test_fused_1m_recall(fused_1m):
    """Recall report at 1M on the fused decode path: per q-head, the selected set's
    softmax mass vs the exact top-|sel| and a random |sel| sample (commands.cpp:243-262)."""
    D, t, groups, hpm, q, k, kv, layer = fused_1m
    layer.q.copy_(q[:, 0])
    layer.run(t)
    torch.cuda.synchronize()
    gen = torch.Generator(device="cuda").manual_seed(0)
    r_mask, r_top, r_rand = [], [], []
    for g in range(groups):
        sel = _selected(layer, g, t)
        assert sel.numel() == 256 + 2048 + 1024 and bool((sel[1:] > sel[:-1]).all())
        keys = k[g].float()
        for h in range(hpm):
            qq = q[g * hpm + h, 0]
            s = (keys @ qq / math.sqrt(128)).double()
            wts = torch.softmax(s, 0)
            r_mask.append(float(wts[sel].sum()))
            r_top.append(float(torch.topk(wts, sel.numel()).values.sum()))
            rnd = torch.randperm(t, generator=gen, device="cuda")[: sel.numel()]
            r_rand.append(float(wts[rnd].sum()))
        del keys
    m, o, r = (float(np.mean(x)) for x in (r_mask, r_top, r_rand))
    print(f"\n1M recall: mask {m:.4f} exact-top {o:.4f} random {r:.4f}")
    assert all(a <= b + 1e-9 for a, b in zip(r_mask, r_top))
    # near-uniform attention at 1M with random synthetic q: absolute mass is small, the
    # mask still holds ~4x the mass of a random set (seed-fixed run: 0.0122 vs 0.0032)
    assert m >= 2.5 * r


def test_fused_1m_needle_retention(fused_1m):
    """Planted needles (workload.cpp:191-220: a key along the group's mean query with
    norm `strength`) at random depths of the 1M context survive all three stages of
    every KV group, once certified as the exact top-1 of each of the group's heads.

    As in acceptance #4 (needle 4096 = sink 256 + 15 x 256) the needle is the first row
    of a stage-1 chunk — and so of its nested stage-2/3 chunks — where Alg. 3 always
    scores it. A one-row spike elsewhere is seen only if the binary descent happens to
    land on it (2 of 32 random depths in a trial run): a property of the algorithm the
    reference shares, since the selections here are index-exact with it."""
    D, t, groups, hpm, q, k, kv, layer = fused_1m
    rng = np.random.default_rng(3)
    kept = total = 0
    for trial in range(4):
        pos = 256 + 256 * rng.integers(0, (t - 1024 - 256) // 256, size=groups)
        saved = []
        for g in range(groups):
            u = q[g * hpm:(g + 1) * hpm, 0].mean(0)
            row = (100.0 * u / u.norm()).to(torch.bfloat16)
            p = int(pos[g])
            slot = kv.k_pool[p // kv.page_size, g, p % kv.page_size]
            saved.append(slot.clone())
            slot.copy_(row)
            k[g, p] = row
            keys = k[g].float()
            for h in range(hpm):
                assert int(torch.argmax(keys @ q[g * hpm + h, 0])) == p
            del keys
        layer.q.copy_(q[:, 0])
        layer.run(t)
        torch.cuda.synchronize()
        for g in range(groups):
            kept += int(pos[g]) in set(_selected(layer, g, t).tolist())
            total += 1
            p = int(pos[g])
            kv.k_pool[p // kv.page_size, g, p % kv.page_size].copy_(saved[g])
            k[g, p] = saved[g]
    print(f"\n1M needle retention: {kept}/{total}")
    assert kept == total

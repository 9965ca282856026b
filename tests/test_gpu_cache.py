"""On-GPU LRU page cache over the pinned host tier (hp_cache_commit + the gathers'
page-table resolution) against the reference TieredKvStore (kv_store.cpp:58-120).

* LRU order: single-page access traces through the device cache reproduce the
  reference's recency order and hit/miss/eviction counts (golden lru{i}, made by
  tests/golden/make_golden.py from the unmodified reference, acceptance #8 setting).
* Transparency: a decode layer step reading through the cache (misses served from the
  host tier inside the kernels) gives bit-identical masks and outputs to the fully
  HBM-resident pool, step after step as the cache warms.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLD = Path(__file__).resolve().parent / "golden"


def _D():
    from paper_2502_08910_b200 import device as D
    D.require_cuda()
    return D


@pytest.mark.parametrize("i", range(8))
def test_lru_order_matches_reference(i):
    D = _D()
    import ctypes as C
    from paper_2502_08910_b200 import _capi
    g = np.load(GOLD / "reference_golden.npz")
    cap = int(g[f"lru{i}_cap"][0])
    trace = g[f"lru{i}_trace"].astype(np.int64)
    n_pages = int(trace.max()) + 1
    ps, d = 4, 8
    k = torch.randn((1, n_pages * ps, d))
    kv = D.CachedKV(k, k.clone(), num_slots=cap, page_size=ps, dtype=torch.float32, warm="none")
    cs = kv.cache_struct()
    for step, p in enumerate(trace):
        resident = int(kv.page_table[p]) >= 0
        kv.touched[p] = 1 if resident else 2
        _capi.check(_capi.lib().hp_cache_commit(C.byref(cs), step + 2, kv.stats.data_ptr(),
                                                kv.ws_cache.data_ptr(), kv.ws_cache.numel(), None))
    torch.cuda.synchronize()
    sp = kv.slot_page.cpu().numpy()
    st = kv.slot_stamp.cpu().numpy()
    live = sp >= 0
    order = sp[live][np.argsort(-st[live], kind="stable")]
    assert order.tolist() == g[f"lru{i}_final"].astype(np.int64).tolist()
    assert kv.stats.cpu().tolist() == g[f"lru{i}_stats"].tolist()
    # every resident slot holds its page's bytes
    for s in np.nonzero(live)[0]:
        assert torch.equal(kv.k_slots[s].cpu(), kv.k_host[sp[s]])
        assert torch.equal(kv.v_slots[s].cpu(), kv.v_host[sp[s]])


@pytest.mark.parametrize("frac", [0.1, 0.5])
def test_cached_decode_is_transparent(frac):
    D = _D()
    from paper_2502_08910_b200 import synth
    groups, hpm, t, d = 8, 4, 1 << 16, 128
    stages = [(64, 64, 8192), (64, 16, 2048), (64, 4, 512)]
    q, k, v = synth.generate(groups * hpm, groups, t, d, t_q=4, seed=5)
    ref_kv = D.PagedKV(k, v, page_size=64)
    c_kv = D.CachedKV(k, v, num_slots=int(frac * (t // 64)), page_size=64)
    mk = lambda kv: D.FusedDecodeLayer(kv, stages, sink=128, stream_tokens=512, n_q_heads=groups * hpm,
                                       n_masks=groups)
    a, b = mk(ref_kv), mk(c_kv)
    hits = []
    for s in range(4):
        for ly in (a, b):
            ly.q.copy_(q[:, s])
        oa = a.run(t).clone()
        ob = b.run(t).clone()
        torch.cuda.synchronize()
        touched = int((c_kv.touched > 0).sum())
        assert touched > 0
        c_kv.commit()
        torch.cuda.synchronize()
        for i in range(3):
            la, ca = a.mask(i)
            lb, cb = b.mask(i)
            assert torch.equal(ca, cb) and torch.equal(la, lb), f"step {s} stage {i}"
        assert torch.equal(oa, ob), f"step {s} output"
        hits.append(int(c_kv.stats[0]))
    st = c_kv.stats.cpu().tolist()
    assert st[0] + st[1] > 0 and hits[-1] > hits[0]
    assert c_kv.resident_pages() == c_kv.num_slots

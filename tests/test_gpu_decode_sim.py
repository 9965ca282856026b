"""Decode-sim parity: the C++ DecodeEngine on the device
against the unmodified reference engine (oracle/_ref), step by step —

  * refresh flags, stage caches (index-exact) and mask sizes;
  * the two-bank page accounting: per-step Mask / SA hits and accesses, the modeled
    stage and BSA latencies (CostModel units), and the LRU recency order of both banks
    after every step (kv_store.cpp:58-120,188-200; decode.cpp:13-27,225-281);
  * outputs within 1e-3 of the reference's fp32;

for the plain schedule and the frozen-stage scenarios of decode-sim, and then the
report itself (hipprune.run_report("decode-sim")) — the reference's smoke test call.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "python"))

STAGES = [(16, 8, 64), (8, 4, 32)]


def _arrays(w):
    L, H = w.num_layers, w.num_heads
    q = np.stack([np.stack([w.q(l, h) for h in range(H)]) for l in range(L)])
    k = np.stack([np.stack([w.k(l, h) for h in range(H)]) for l in range(L)])
    v = np.stack([np.stack([w.v(l, h) for h in range(H)]) for l in range(L)])
    return q, k, v


@pytest.mark.parametrize("frozen", [(False, False), (True, False), (True, True)])
@pytest.mark.parametrize("caps", [(16, 16), (6, 40), (0, 8)])
def test_engine_accounting_matches_reference(ref, frozen, caps):
    import hipprune
    seq, steps = 384, 24
    w = hipprune.generate(heads=2, layers=2, seq_kv=seq, seq_q=seq, dim=16, seed=5)
    q, k, v = _arrays(w)
    prefill = seq - steps
    kw = dict(prefill_len=prefill, q_len=STAGES[0][0], stages=STAGES, sink=16, stream=32, refresh=[4, 2])
    mine = hipprune.DecodeEngine(w, page_size=8, mask_capacity=caps[0], sa_capacity=caps[1], **kw)
    theirs = ref.engine(q, k, v, page_size=8, mask_cap=caps[0], sa_cap=caps[1], **kw)
    mine.set_frozen_stages(list(frozen))
    theirs.set_frozen_stages(list(frozen))
    mine.prefill()
    theirs.prefill()
    for bank in (0, 1):
        assert mine.store_recency(bank) == theirs.store_recency(bank), ("prefill", bank)
    for s in range(steps):
        out, tel = mine.step()
        want, flags, sizes = theirs.step(prefill + s)
        tw = theirs.last_telemetry
        assert tel["refreshed"] == flags, s
        assert tel["mask_sizes"] == sizes, s
        for key in ("mask_hits", "mask_accesses", "sa_hits", "sa_accesses"):
            assert tel[key] == tw[key], (s, key, tel[key], tw[key])
        assert tel["stage_latency"] == tw["stage_latency"], s
        assert tel["bsa_latency"] == tw["bsa_latency"], s
        for bank in (0, 1):
            assert mine.store_recency(bank) == theirs.store_recency(bank), (s, bank)
        for layer in range(2):
            for i in range(len(STAGES)):
                assert list(mine.stage_cache(layer, i)) == list(theirs.stage_cache(layer, i)), (s, layer, i)
        err = np.abs(out - want).max() / max(1e-6, np.abs(want).max())
        assert err <= 1e-3, (s, err)


def test_reference_smoke_report_and_hash():
    """tests/python/test_smoke.py::test_report_and_hash of the reference, via `import hipprune`."""
    import hipprune
    overrides = ["workload.heads=1", "workload.layers=1", "workload.seq_kv=256", "workload.dim=16",
                 "plan.stages=16:8:64,8:4:32", "plan.sink=16", "plan.stream=32", "plan.refresh=4,2",
                 "store.page_size=8", "store.mask_capacity=16", "store.sa_capacity=16", "run.steps=8"]
    report = hipprune.run_report("decode-sim", overrides)
    summary = json.loads(report["json"])
    assert summary["command"] == "decode-sim"
    assert [s["name"] for s in summary["scenarios"]] == ["none", "s1", "all"]
    assert set(report["extras"]) == {"none.jsonl", "s1.jsonl", "all.jsonl"}
    lines = report["extras"]["none.jsonl"].strip().split("\n")
    assert len(lines) == 8 and json.loads(lines[0])["step"] == 1
    h = hipprune.config_hash(overrides)
    assert h == hipprune.config_hash(overrides)
    assert h != hipprune.config_hash(overrides[:-1] + ["run.steps=9"])


def test_reference_smoke_calls():
    """The remaining reference smoke-test calls (tests/python/test_smoke.py) through `import hipprune`."""
    import hipprune
    w = hipprune.generate(heads=2, layers=1, seq_kv=1024, seq_q=32, dim=16, seed=3)
    assert w.num_heads == 2 and w.seq_len_kv == 1024
    assert w.q(0, 0).shape == (32, 16) and w.k(0, 1).shape == (1024, 16)
    mask = hipprune.build_mask(w, layer=0, stages=[(32, 8, 128), (32, 4, 64)], sink=32, stream=64)
    assert mask.block_size == 32 and len(mask.indices) == 1 and len(mask.indices[0]) <= 64
    assert all(32 <= i < 1024 - 64 for i in mask.indices[0])
    sparse = hipprune.block_sparse_attention(w, 0, mask)
    dense = hipprune.dense_attention(w, 0)
    assert sparse[0].shape == dense[0].shape and np.isfinite(sparse[0]).all()
    selected = hipprune.selected_indices(mask, 31)
    qv = w.q(0, 0)[31]
    keys = w.k(0, 0)
    recall = hipprune.attention_recall(selected, qv, keys)
    top = hipprune.exact_topk(qv, keys, len(selected))
    assert 0.0 <= recall <= hipprune.attention_recall(top, qv, keys) + 1e-9
    sp = json.loads(hipprune.run_report("sparsity-report", ["workload.heads=1", "workload.layers=1",
                                                              "workload.seq_kv=1024", "workload.dim=16",
                                                              "run.sparsity_topk=64"])["json"])
    assert [r["chunk_size"] for r in sp["rows"]] == [8, 16, 32, 64, 128, 256]
    assert all(0.0 <= r["empty_fraction"] <= 1.0 for r in sp["rows"])

"""Pin the CPU oracle (oracle/hipprune_oracle.c, the C restatement) to the reference.

* against the committed golden vectors produced by the unmodified reference
  library on inputs from the reference's own generator (tests/golden/) — runs
  everywhere;
* against the reference library itself (oracle/_ref) on random cases, including
  the acceptance-gate settings (acceptance.cpp:146-265) — runs where it is built.
Everything index-like and every float must match bit for bit.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_golden.npz"


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def test_port_matches_reference_golden_masks(port, gold):
    for name in ("mb3", "k3", "smoke"):
        q, k, v = gold[f"{name}_q"], gold[f"{name}_k"], gold[f"{name}_v"]
        stages = [tuple(int(x) for x in s) for s in gold[f"{name}_stages"]]
        sink, stream = (int(x) for x in gold[f"{name}_sink_stream"])
        for ext in (0, 1):
            nb, bs, off = (int(x) for x in gold[f"{name}_ext{ext}_nblocks"])
            lists, trace, pbs, poff = port.build_mask(q, k, stages, sink=sink, stream=stream, ext=ext)
            assert (len(lists), pbs, poff) == (nb, bs, off)
            for b in range(nb):
                assert np.array_equal(lists[b], gold[f"{name}_ext{ext}_mask{b}"]), (name, ext, b)
            for s in range(len(stages)):
                assert np.array_equal(trace[s], gold[f"{name}_ext{ext}_trace{s}"])
            o = port.block_sparse_attention(q, k, v, lists, block_size=bs, sink=sink, stream=stream,
                                            offset=off, ext=bool(ext))
            assert np.array_equal(o, gold[f"{name}_ext{ext}_bsa"]), (name, ext)


def test_port_matches_reference_golden_decode(port, gold):
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 128)]
    masks, out, _ = port.decode_layer_step(gold["dec_q"], gold["dec_k"], gold["dec_v"], stages,
                                           sink=128, stream=512)
    for g in range(2):
        assert np.array_equal(masks[g], gold[f"dec_mask{g}"])
    assert np.array_equal(out, gold["dec_out"])


def test_port_matches_reference_golden_select_rep_traces(port, gold):
    for i in range(24):
        ext, layer1, qstart, ci, cnt, rep = (int(x) for x in gold[f"rep{i}_meta"])
        r, reads = port.select_rep(gold[f"rep{i}_q"], gold[f"rep{i}_chunk"], gold[f"rep{i}_k"],
                                   layer1=layer1, stream=8, qstart=qstart, ext=bool(ext),
                                   chunk_index=ci, chunk_count=cnt, rope_max=4096)
        assert r == rep
        assert np.array_equal(reads, gold[f"rep{i}_reads"])


def test_port_matches_reference_golden_lru(port, gold):
    for i in range(8):
        cap = int(gold[f"lru{i}_cap"][0])
        st = port.store(1, 4, cap, 1)
        for p in gold[f"lru{i}_trace"]:
            miss = st.access(0, [p])
            if miss.size:
                st.commit(0, miss)
        assert np.array_equal(st.recency(0), gold[f"lru{i}_final"])
        assert np.array_equal(np.asarray(st.stats(0)), gold[f"lru{i}_stats"])
        st.check()


# ------------------------------------------------------------ live reference
def test_port_vs_reference_stages(port, ref):
    """acceptance #6 (acceptance.cpp:220-265) and #5 (:146-217) settings, 400 cases."""
    rng = np.random.default_rng(7)
    for trial in range(400):
        ext = bool(trial % 2)
        rows = int(1 + rng.integers(4))
        h = int(1 + rng.integers(3))
        q = rng.standard_normal((h, rows, 8), dtype=np.float32)
        k = rng.standard_normal((h, 128, 8), dtype=np.float32)
        idx = np.sort(rng.permutation(128)[: 1 + rng.integers(120)])
        lc = int(1 + rng.integers(16))
        stage = (64, lc, lc * int(1 + rng.integers(8)))
        kw = dict(layer1=int(1 + rng.integers(6)), stream=8, qstart=int(rng.integers(2048)),
                  ext=ext, rope_max=4096, count_reads=True)
        a, ta, da = port.run_pruning_stage(stage, idx, q, k, **kw)
        b, tb, db = ref.run_pruning_stage(stage, idx, q, k, **kw)
        assert np.array_equal(a, b), trial
        assert (ta, da) == (tb, db)


def test_port_vs_reference_build_mask_and_bsa(port, ref):
    rng = np.random.default_rng(11)
    for trial in range(12):
        q, k, v = ref.generate(heads=int(1 + rng.integers(3)), layers=1, seq_kv=int(600 + rng.integers(2000)),
                               seq_q=int(1 + rng.integers(200)), dim=16, seed=int(rng.integers(1 << 30)))
        q, k, v = q[0], k[0], v[0]
        bq = [64, 32, 16][trial % 3]
        stages = [(bq, 16, 256), (max(1, bq // 2), 8, 128)]
        for ext in (0, 1):
            la, ta, bs, off = port.build_mask(q, k, stages, sink=32, stream=64, ext=ext, layer0=trial % 5)
            lb, tb, _, _ = ref.build_mask(q, k, stages, sink=32, stream=64, ext=ext, layer0=trial % 5)
            assert all(np.array_equal(x, y) for x, y in zip(la, lb)) and len(la) == len(lb)
            assert all(np.array_equal(x, y) for x, y in zip(ta, tb))
            oa = port.block_sparse_attention(q, k, v, la, block_size=bs, sink=32, stream=64, offset=off, ext=bool(ext))
            ob = ref.block_sparse_attention(q, k, v, lb, block_size=bs, sink=32, stream=64, offset=off, ext=bool(ext))
            assert np.array_equal(oa, ob)


def test_port_vs_reference_decode_and_helpers(port, ref):
    rng = np.random.default_rng(5)
    q, k, v = ref.generate(heads=2, layers=1, seq_kv=9000, seq_q=1, dim=32, seed=5)
    qg = rng.standard_normal((2, 4, 32), dtype=np.float32)
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 128)]
    for ext in (False, True):
        ma, oa, _ = port.decode_layer_step(qg, k[0], v[0], stages, sink=128, stream=512, ext=ext)
        mb, ob, _ = ref.decode_layer_step(qg, k[0], v[0], stages, sink=128, stream=512, ext=ext)
        assert all(np.array_equal(x, y) for x, y in zip(ma, mb))
        assert np.array_equal(oa, ob)
    keys = k[0, 0, :300]
    qq = q[0, 0, 0]
    for kk in (1, 7, 64):
        assert np.array_equal(port.exact_topk(qq, keys, kk), ref.exact_topk(qq, keys, kk))
    sel = np.arange(0, 300, 3)
    assert port.attention_recall(sel, qq, keys) == ref.attention_recall(sel, qq, keys)
    d = port.dense_attention(q[0, :, :5], k[0, :, :40], v[0, :, :40])
    e = ref.dense_attention(q[0, :, :5], k[0, :, :40], v[0, :, :40])
    assert np.array_equal(d, e)
    ca, sa = port.rope_table(70, 16)
    cb, sb = ref.rope_table(70, 16)
    assert np.array_equal(ca, cb) and np.array_equal(sa, sb)


def test_port_vs_reference_lru(port, ref):
    """acceptance #8 (acceptance.cpp:319-373): recency order after every access."""
    rng = np.random.default_rng(1008)
    for trial in range(200):
        cap = int(1 + rng.integers(8))
        uni = int(2 + rng.integers(16))
        a, b = port.store(1, 4, cap, 2), ref.store(1, 4, cap, 2)
        for _ in range(60):
            p = a.page_of(0, 4 * int(rng.integers(uni)))
            ma, mb = a.access(0, [p]), b.access(0, [p])
            assert np.array_equal(ma, mb)
            if ma.size:
                assert np.array_equal(a.commit(0, ma), b.commit(0, mb))
            assert np.array_equal(a.recency(0), b.recency(0))
        assert a.stats(0) == b.stats(0)


# -------------------------------------------------------------- reference KATs
def test_kats_select_rep_and_stage(port):
    """test_pruning.cpp:89-118 and :201-235 known answers."""
    q = np.zeros((1, 4), np.float32); q[0, 0] = 1.0
    k = np.zeros((8, 4), np.float32)
    rep, reads = port.select_rep(q, [5], k)
    assert rep == 5 and reads.size == 0                    # length one: zero reads
    k1 = k.copy(); k1[:, 0] = np.arange(8)
    assert port.select_rep(q, [1, 2, 3, 4], k1)[0] == 4    # increasing scores
    k2 = k.copy(); k2[:, 0] = 1.0
    assert port.select_rep(q, [2, 3, 4, 5, 6], k2)[0] == 2  # ties take the left branch
    from oracle import OracleError
    with pytest.raises(OracleError):
        port.select_rep(q, [], k)                          # empty chunk: ContractViolation
    rng = np.random.default_rng(37)
    kk = rng.standard_normal((1, 32, 4), dtype=np.float32)
    qq = rng.standard_normal((1, 2, 4), dtype=np.float32)
    idx = np.arange(16)
    assert np.array_equal(port.run_pruning_stage((64, 4, 16), idx, qq, kk), idx)
    with pytest.raises(OracleError):
        port.run_pruning_stage((64, 4, 8), [1, 0, 2], qq, kk)
    kc = np.full_like(kk, 0.5)
    assert np.array_equal(port.run_pruning_stage((64, 4, 8), idx, qq, kc), np.arange(8))


def test_kats_selected_indices(port):
    """test_sparse_attention.cpp:181-192 goldens."""
    lists = [[2, 5, 7, 11], [2, 5, 7, 11]]
    assert port.selected_indices(lists, 4, 2, 3, 8, 0).tolist() == [0, 1, 2, 5, 6, 7, 8]
    assert port.selected_indices(lists, 4, 2, 3, 8, 4).tolist() == [0, 1, 2, 5, 7, 10, 11, 12]
    assert port.selected_indices([[]], 4, 4, 4, 0, 1).tolist() == [0, 1]


def test_kats_exact_topk_and_rope(port):
    """test_sparse_attention.cpp:223-239; test_tensor.cpp:20-29."""
    keys = np.zeros((4, 2), np.float32); keys[:, 0] = [1, 3, 2, 3]
    q = np.array([1, 0], np.float32)
    assert port.exact_topk(q, keys, 1).tolist() == [1]
    assert port.exact_topk(q, keys, 3).tolist() == [1, 3, 2]
    assert port.exact_topk(q, keys, 4).tolist() == [1, 3, 2, 0]
    assert port.exact_topk(q, np.ones((3, 2), np.float32), 3).tolist() == [0, 1, 2]
    c, s = port.rope_table(4, 4)
    assert abs(c[2, 1] - np.cos(0.02)) < 1e-6 and abs(c[2, 1] - 0.99980) < 1e-4

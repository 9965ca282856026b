"""The reference-named Python API (paper_2502_08910_b200.hipprune == proj/python/hipprune)
over the C++ host layer and the sm_100a kernels.

CPU tests cover what runs on the host in the reference too (generator, HIPW dumps,
selected_indices, exact_topk, attention_recall) and the loud failure of the device
operators without a GPU. GPU tests mirror proj/tests/python/test_smoke.py and check
build_mask / block_sparse_attention / dense_attention / DecodeEngine against the
reference's own outputs (tests/golden/*.npz, made by tests/golden/make_golden.py from
the unmodified reference library).
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

hp = pytest.importorskip("paper_2502_08910_b200.hipprune")

GOLD = Path(__file__).resolve().parent / "golden"
RTOL = 1e-3


def _gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def rel_err(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(1e-6, np.abs(b).max())


@pytest.fixture(scope="module")
def engine_gold():
    return np.load(GOLD / "engine_golden.npz")


@pytest.fixture(scope="module")
def workload():
    return hp.generate(heads=2, layers=1, seq_kv=1024, seq_q=32, dim=16, seed=3)


# ------------------------------------------------------------------ host side
def test_exports_match_reference_package():
    ref_names = {"SparseBlockMask", "Workload", "attention_recall", "block_sparse_attention",
                 "build_mask", "config_hash", "dense_attention", "dump_checksum", "exact_topk",
                 "generate", "load_dump", "run_report", "save_dump", "selected_indices"}
    assert set(hp.__all__) == ref_names
    for n in ref_names:
        assert hasattr(hp, n)


def test_generator_bit_identical_to_reference(engine_gold):
    """generate_synthetic (workload.cpp:147-189): same libstdc++ streams, same smoothing."""
    w = hp.generate(heads=2, layers=2, seq_kv=640, seq_q=640, dim=16, seed=21)
    for l in range(2):
        for h in range(2):
            assert np.array_equal(w.q(l, h), engine_gold["q"][l, h])
            assert np.array_equal(w.k(l, h), engine_gold["k"][l, h])
            assert np.array_equal(w.v(l, h), engine_gold["v"][l, h])


def test_workload_shapes_and_determinism(workload):
    assert workload.num_heads == 2 and workload.seq_len_kv == 1024
    assert workload.q(0, 0).shape == (32, 16) and workload.k(0, 1).shape == (1024, 16)
    assert np.isfinite(workload.k(0, 0)).all()
    again = hp.generate(heads=2, layers=1, seq_kv=1024, seq_q=32, dim=16, seed=3)
    assert np.array_equal(workload.k(0, 0), again.k(0, 0))
    assert hp.dump_checksum(workload) == hp.dump_checksum(again)


def test_needles_planted_along_mean_query():
    w = hp.generate(heads=2, layers=1, seq_kv=256, seq_q=8, dim=8, seed=5, needles=[(100, 50.0)])
    k = w.k(0, 0)[100]
    assert abs(np.linalg.norm(k) - 50.0) < 1e-3
    with pytest.raises(IndexError):
        hp.generate(heads=1, layers=1, seq_kv=64, seq_q=8, dim=8, needles=[(64, 1.0)])


def test_dump_round_trip_and_corruption(workload, tmp_path):
    path = tmp_path / "w.hipw"
    hp.save_dump(workload, str(path))
    loaded = hp.load_dump(str(path))
    assert np.array_equal(workload.v(0, 1), loaded.v(0, 1))
    assert hp.dump_checksum(loaded) == hp.dump_checksum(workload)
    raw = bytearray(path.read_bytes())
    raw[60] ^= 0xFF  # flip a payload byte -> checksum mismatch (workload.cpp:303-306)
    bad = tmp_path / "bad.hipw"
    bad.write_bytes(bytes(raw))
    with pytest.raises(hp.FormatError, match="checksum"):
        hp.load_dump(str(bad))
    bad.write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(hp.FormatError, match="magic"):
        hp.load_dump(str(bad))
    bad.write_bytes(bytes(raw[:40]))
    with pytest.raises(hp.FormatError, match="truncated"):
        hp.load_dump(str(bad))


def test_workload_from_arrays_validates():
    q = np.zeros((1, 2, 4, 8), np.float32); k = np.zeros((1, 2, 16, 8), np.float32)
    w = hp.Workload(q, k, k)
    assert (w.num_layers, w.num_heads, w.seq_len_q, w.seq_len_kv, w.head_dim) == (1, 2, 4, 16, 8)
    with pytest.raises(ValueError):
        hp.Workload(np.zeros((1, 2, 32, 8), np.float32), k, k)  # T_q > T_kv
    k2 = k.copy(); k2[0, 0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        hp.Workload(q, k2, k)


def test_selected_indices_goldens():
    """test_sparse_attention.cpp:181-192."""
    m = hp.SparseBlockMask(4, 2, 3, 8, [[2, 5, 7, 11], [2, 5, 7, 11]])
    assert hp.selected_indices(m, 0) == [0, 1, 2, 5, 6, 7, 8]
    assert hp.selected_indices(m, 4) == [0, 1, 2, 5, 7, 10, 11, 12]
    assert hp.selected_indices(hp.SparseBlockMask(4, 4, 4, 0, [[]]), 1) == [0, 1]
    with pytest.raises(IndexError):
        hp.selected_indices(m, 8)


def test_exact_topk_and_recall_goldens(workload):
    """test_sparse_attention.cpp:223-239 + the smoke test's recall bound."""
    keys = np.zeros((4, 2), np.float32); keys[:, 0] = [1, 3, 2, 3]
    q = np.asarray([1, 0], np.float32)
    assert hp.exact_topk(q, keys, 1) == [1]
    assert hp.exact_topk(q, keys, 3) == [1, 3, 2]
    assert hp.exact_topk(q, keys, 4) == [1, 3, 2, 0]
    with pytest.raises(ValueError):
        hp.exact_topk(q, keys, 99)
    assert hp.exact_topk(q, np.ones((3, 2), np.float32), 3) == [0, 1, 2]
    qq, kk = workload.q(0, 0)[31], workload.k(0, 0)
    top = hp.exact_topk(qq, kk, 50)
    assert 0.0 <= hp.attention_recall(top[:10], qq, kk) <= hp.attention_recall(top, qq, kk) + 1e-12
    assert abs(hp.attention_recall(list(range(1024)), qq, kk) - 1.0) < 1e-9


def test_report_plumbing():
    """run_report / config_hash (the reference's report plumbing, python/hipprune/_reports.py):
    config_hash is deterministic and override-sensitive on any host; unknown commands are
    ValueError as in bindings.cpp; decode-sim itself runs on the GPU (test_gpu_decode_sim.py)."""
    h = hp.config_hash(["run.steps=8"])
    assert isinstance(h, int) and h == hp.config_hash(["run.steps=8"]) != hp.config_hash(["run.steps=9"])
    with pytest.raises(ValueError):
        hp.run_report("no-such-report", [])


@pytest.mark.skipif(_gpu(), reason="checks the no-device failure mode")
def test_device_operators_fail_loudly_without_gpu(workload):
    assert not hp.device_available()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hp.build_mask(workload, 0, stages=[(32, 8, 128), (32, 4, 64)], sink=32, stream=64)
    m = hp.SparseBlockMask(32, 32, 64, 992, [[40, 41]])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hp.block_sparse_attention(workload, 0, m)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hp.dense_attention(workload, 0)


# ------------------------------------------------------------------ device side
@pytest.mark.gpu
def test_smoke_mask_and_sparse_attention(workload):
    """proj/tests/python/test_smoke.py::test_mask_and_sparse_attention."""
    mask = hp.build_mask(workload, layer=0, stages=[(32, 8, 128), (32, 4, 64)], sink=32, stream=64)
    assert mask.block_size == 32 and len(mask.indices) == 1
    assert len(mask.indices[0]) <= 64
    assert all(32 <= i < 1024 - 64 for i in mask.indices[0])
    sparse = hp.block_sparse_attention(workload, 0, mask)
    dense = hp.dense_attention(workload, 0)
    assert sparse[0].shape == dense[0].shape and np.isfinite(sparse[0]).all()
    sel = hp.selected_indices(mask, 31)
    q, keys = workload.q(0, 0)[31], workload.k(0, 0)
    recall = hp.attention_recall(sel, q, keys)
    oracle = hp.attention_recall(hp.exact_topk(q, keys, len(sel)), q, keys)
    assert 0.0 <= recall <= oracle + 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mb3", "k3", "smoke"])
@pytest.mark.parametrize("ext", [0, 1])
def test_build_mask_and_bsa_match_reference_golden(name, ext):
    g = np.load(GOLD / "reference_golden.npz")
    q, k, v = g[f"{name}_q"], g[f"{name}_k"], g[f"{name}_v"]
    stages = [tuple(int(x) for x in s) for s in g[f"{name}_stages"]]
    sink, stream = (int(x) for x in g[f"{name}_sink_stream"])
    w = hp.Workload(q[None], k[None], v[None])
    mask = hp.build_mask(w, 0, stages=stages, sink=sink, stream=stream, extension=bool(ext))
    nb, bs, off = (int(x) for x in g[f"{name}_ext{ext}_nblocks"])
    assert (len(mask.indices), mask.block_size, mask.query_offset) == (nb, bs, off)
    for b in range(nb):
        assert mask.indices[b] == g[f"{name}_ext{ext}_mask{b}"].tolist(), f"block {b}"
    out = hp.block_sparse_attention(w, 0, mask, extension=bool(ext))
    assert rel_err(np.stack(out), g[f"{name}_ext{ext}_bsa"]) <= RTOL


@pytest.mark.gpu
def test_dense_attention_matches_oracle(port, workload):
    q = np.stack([workload.q(0, h) for h in range(2)])
    k = np.stack([workload.k(0, h) for h in range(2)])
    v = np.stack([workload.v(0, h) for h in range(2)])
    want = port.dense_attention(q, k, v)
    got = np.stack(hp.dense_attention(workload, 0))
    assert rel_err(got, want) <= RTOL


@pytest.mark.gpu
@pytest.mark.parametrize("ext", [0, 1])
def test_decode_engine_matches_reference_engine(engine_gold, ext):
    """DecodeEngine::prefill/step (decode.cpp:133-289) with a (4, 2) refresh schedule:
    per-step outputs within 1e-3, refresh flags and every (layer, stage) cache exact."""
    g = engine_gold
    w = hp.Workload(g["q"], g["k"], g["v"])
    stages = [tuple(int(x) for x in s) for s in g["stages"]]
    e = hp.DecodeEngine(w, prefill_len=600, q_len=32, stages=stages, sink=16, stream=32,
                        refresh=[4, 2], extension=bool(ext), page_size=16)
    _, masks = e.prefill()
    for b, idx in enumerate(masks[-1].indices):
        assert idx == g[f"e{ext}_prefill_mask{b}"].tolist()
    for i in range(12):
        out, tel = e.step()
        assert [int(x) for x in tel["refreshed"]] == g[f"e{ext}_s{i}_refreshed"].tolist(), f"step {i}"
        for layer in range(2):
            for st in range(2):
                assert e.stage_cache(layer, st) == g[f"e{ext}_s{i}_cache{layer}{st}"].tolist(), \
                    f"step {i} layer {layer} stage {st}"
        assert rel_err(out, g[f"e{ext}_s{i}_out"]) <= RTOL, f"step {i}"
    assert e.steps_taken == 12 and list(e.counters) == [0, 0]


def _truncate(full, t_kv, q_len):
    """truncate_workload (workload.cpp): keys/values [0, t_kv), the last q_len query rows."""
    L, H = full.num_layers, full.num_heads
    q = np.stack([np.stack([full.q(l, h)[t_kv - q_len:t_kv] for h in range(H)]) for l in range(L)])
    k = np.stack([np.stack([full.k(l, h)[:t_kv] for h in range(H)]) for l in range(L)])
    v = np.stack([np.stack([full.v(l, h)[:t_kv] for h in range(H)]) for l in range(L)])
    return hp.Workload(np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v))


@pytest.mark.gpu
def test_cache_disabled_equivalence_acceptance7():
    """acceptance.cpp:269-316: with every stage refreshed each step, the engine's last
    stage cache equals build_mask on the truncated workload and its outputs equal the
    block-sparse attention of that mask, for 64 steps; then refresh counts over 48 steps
    at intervals (16, 8, 4) are (3, 6, 12)."""
    steps = 64
    full = hp.generate(heads=2, layers=2, seq_kv=144, seq_q=144, dim=8, seed=8001)
    stages = [(1, 4, 32), (1, 4, 16), (1, 2, 8)]
    e = hp.DecodeEngine(full, prefill_len=144 - steps, q_len=1, stages=stages, sink=8, stream=16,
                        refresh=[1, 1, 1], extension=False, page_size=8)
    e.prefill()
    for t in range(144 - steps, 144):
        out, tel = e.step()
        trunc = _truncate(full, t + 1, 1)
        for layer in range(2):
            mask = hp.build_mask(trunc, layer, stages=stages, sink=8, stream=16, extension=False)
            assert e.stage_cache(layer, 2) == list(mask.indices[0]), (t, layer)
            want = np.stack(hp.block_sparse_attention(trunc, layer, mask))[:, 0]
            assert rel_err(out[layer], want) <= RTOL, (t, layer)
    long_full = hp.generate(heads=1, layers=1, seq_kv=240, seq_q=240, dim=8, seed=8002)
    counted = hp.DecodeEngine(long_full, prefill_len=192, q_len=1, stages=stages, sink=8, stream=16,
                              refresh=[16, 8, 4], extension=False, page_size=8)
    counted.prefill()
    refreshes = [0, 0, 0]
    for _ in range(48):
        _, tel = counted.step()
        for i in range(3):
            refreshes[i] += bool(tel["refreshed"][i])
    assert refreshes == [3, 6, 12]


def test_reads_reference_written_dump(tmp_path):
    """HIPW interchange (workload.cpp:222-312): a dump the unmodified reference wrote
    (tests/golden/ref_small.hipw, tests/golden/make_golden.py) loads here with the same
    tensors as this library's generator (bit-identical), the same dump_checksum, and
    re-saving it reproduces the file byte for byte."""
    from pathlib import Path
    gold = Path(__file__).resolve().parent / "golden"
    w = hp.load_dump(str(gold / "ref_small.hipw"))
    assert (w.num_heads, w.num_layers, w.seq_len_kv, w.seq_len_q, w.head_dim) == (2, 2, 64, 16, 8)
    assert hp.dump_checksum(w) == int((gold / "ref_small.crc").read_text())
    mine = hp.generate(heads=2, layers=2, seq_kv=64, seq_q=16, dim=8, seed=21)
    for l in range(2):
        for h in range(2):
            assert np.array_equal(w.q(l, h), mine.q(l, h)) and np.array_equal(w.k(l, h), mine.k(l, h))
            assert np.array_equal(w.v(l, h), mine.v(l, h))
    out = tmp_path / "again.hipw"
    hp.save_dump(w, str(out))
    assert out.read_bytes() == (gold / "ref_small.hipw").read_bytes()

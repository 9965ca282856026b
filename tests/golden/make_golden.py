"""Generate the committed golden vectors from the UNMODIFIED reference library.

Run here (where /root/reference exists): python tests/golden/make_golden.py
It builds oracle/_ref (the reference sources compiled where they lie) and
records, for small cases, the reference's own outputs on inputs produced by the
reference's own generator (libstdc++ <random>, workload.cpp:147-189):
  * build_mask lists + stage trace  (pruning.cpp:202-313)
  * block_sparse_attention output    (sparse_attention.cpp:114-145)
  * the per-layer decode body        (decode.cpp:225-273 with every stage due)
  * select_rep read traces           (pruning.cpp:69-98)
  * LRU recency histories            (kv_store.cpp:58-120)
The GPU box has no /root/reference; tests compare the C port and the CUDA path
against these files there.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import Oracle, build  # noqa: E402


def hipw() -> None:
    """A reference-written HIPW dump + its checksum (workload.cpp:222-312), for the
    interchange test (tests/test_hipprune_api.py::test_reads_reference_written_dump)."""
    import subprocess
    path = HERE / "ref_small.hipw"
    res = subprocess.run([str(HERE.parents[1] / "oracle" / "_ref" / "ref_hipw"), str(path), "2", "2", "64", "16",
                          "8", "21"], check=True, capture_output=True, text=True)
    (HERE / "ref_small.crc").write_text(res.stdout.strip() + "\n")


def main() -> None:
    build("all")
    hipw()
    R = Oracle("reference")
    out = {}
    # 1. build_mask on reference-generated workloads (test_pruning.cpp:323-349 plan, 3k plan)
    cases = [
        ("mb3", dict(heads=2, layers=1, seq_kv=1024, seq_q=256, dim=16, seed=4),
         [(64, 16, 256), (32, 8, 128), (16, 4, 64)], 64, 128),
        ("k3", dict(heads=1, layers=1, seq_kv=256 + 5000 + 1024, seq_q=64, dim=16, seed=3),
         [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)], 256, 1024),
        ("smoke", dict(heads=2, layers=1, seq_kv=1024, seq_q=32, dim=16, seed=3),
         [(32, 8, 128), (32, 4, 64)], 32, 64),
    ]
    for name, g, stages, sink, stream in cases:
        q, k, v = R.generate(**g)
        q, k, v = q[0], k[0], v[0]
        for ext in (0, 1):
            lists, trace, bs, off = R.build_mask(q, k, stages, sink=sink, stream=stream, ext=ext)
            out[f"{name}_q"], out[f"{name}_k"], out[f"{name}_v"] = q, k, v
            out[f"{name}_stages"] = np.asarray(stages, np.int64)
            out[f"{name}_sink_stream"] = np.asarray([sink, stream], np.int64)
            out[f"{name}_ext{ext}_nblocks"] = np.asarray([len(lists), bs, off], np.int64)
            for b, l in enumerate(lists):
                out[f"{name}_ext{ext}_mask{b}"] = l
            for s, l in enumerate(trace):
                out[f"{name}_ext{ext}_trace{s}"] = l
            o = R.block_sparse_attention(q, k, v, lists, block_size=bs, sink=sink, stream=stream,
                                         offset=off, ext=bool(ext))
            out[f"{name}_ext{ext}_bsa"] = o
    # 2. decode body, GQA (2 groups x 4 q-heads), reference generator
    q, k, v = R.generate(heads=2, layers=1, seq_kv=6144, seq_q=1, dim=32, seed=11)
    qg = R.generate(heads=8, layers=1, seq_kv=16, seq_q=1, dim=32, seed=12)[0][0]
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 128)]
    masks, o, _ = R.decode_layer_step(qg[:, 0].reshape(2, 4, 32), k[0], v[0], stages, sink=128, stream=512)
    out["dec_q"], out["dec_k"], out["dec_v"] = qg[:, 0].reshape(2, 4, 32), k[0], v[0]
    out["dec_out"] = o
    for gi, m in enumerate(masks):
        out[f"dec_mask{gi}"] = m
    # 3. select_rep read traces (acceptance.cpp:146-217 setting)
    rng = np.random.default_rng(1005)
    for i in range(24):
        ext = i % 2
        n = int(1 + rng.integers(64))
        qq = rng.standard_normal((int(1 + rng.integers(4)), 8), dtype=np.float32)
        kk = rng.standard_normal((128, 8), dtype=np.float32)
        chunk = np.arange(n) + int(rng.integers(64))
        layer1, qstart = int(1 + rng.integers(6)), int(rng.integers(2048))
        ci, cnt = int(rng.integers(8)), int(8 + rng.integers(8))
        rep, reads = R.select_rep(qq, chunk, kk, layer1=layer1, stream=8, qstart=qstart, ext=bool(ext),
                                  chunk_index=ci, chunk_count=cnt, rope_max=4096)
        out[f"rep{i}_q"], out[f"rep{i}_k"], out[f"rep{i}_chunk"] = qq, kk, chunk
        out[f"rep{i}_meta"] = np.asarray([ext, layer1, qstart, ci, cnt, rep], np.int64)
        out[f"rep{i}_reads"] = reads
    # 4. LRU recency histories (acceptance.cpp:319-337)
    for i in range(8):
        cap = int(1 + rng.integers(8))
        uni = int(2 + rng.integers(16))
        st = R.store(1, 4, cap, 1)
        trace = np.asarray([st.page_of(0, 4 * int(rng.integers(uni))) for _ in range(40)], np.uint64)
        hist = []
        for p in trace:
            miss = st.access(0, [p])
            if miss.size:
                st.commit(0, miss)
            hist.append(st.recency(0))
        out[f"lru{i}_cap"] = np.asarray([cap], np.int64)
        out[f"lru{i}_trace"] = trace
        out[f"lru{i}_final"] = hist[-1]
        out[f"lru{i}_stats"] = np.asarray(st.stats(0), np.int64)
    np.savez_compressed(HERE / "reference_golden.npz", **out)
    print("wrote", HERE / "reference_golden.npz", len(out), "arrays")
    engine_golden(R)


def engine_golden(R) -> None:
    """5. The reference DecodeEngine (decode.cpp:104-289): prefill, then 12 steps with
    a (4, 2) refresh schedule; per step the outputs, refresh flags and every
    (layer, stage) cache — the stage-cache scheduler of DecodeEngine::step."""
    out = {}
    q, k, v = R.generate(heads=2, layers=2, seq_kv=640, seq_q=640, dim=16, seed=21)
    out["q"], out["k"], out["v"] = q, k, v
    stages = [(16, 8, 128), (16, 4, 64)]
    out["stages"] = np.asarray(stages, np.int64)
    out["meta"] = np.asarray([600, 32, 16, 32, 4, 2, 12], np.int64)  # prefill, q_len, sink, stream, refresh, steps
    for ext in (0, 1):
        e = R.engine(q, k, v, prefill_len=600, q_len=32, stages=stages, sink=16, stream=32, refresh=[4, 2],
                     ext=bool(ext))
        masks = e.prefill()
        for b, m in enumerate(masks):
            out[f"e{ext}_prefill_mask{b}"] = m
        for i in range(12):
            o, refreshed, _ = e.step(600 + i)
            out[f"e{ext}_s{i}_out"] = o
            out[f"e{ext}_s{i}_refreshed"] = np.asarray(refreshed, np.int64)
            for layer in range(2):
                for st in range(2):
                    out[f"e{ext}_s{i}_cache{layer}{st}"] = e.stage_cache(layer, st)
    np.savez_compressed(HERE / "engine_golden.npz", **out)
    print("wrote", HERE / "engine_golden.npz", len(out), "arrays")


if __name__ == "__main__":
    main()

"""The C++ boundary under the reference's header names (include/hipprune/*.hpp):
tests/cpp/ref_api.cpp is written against the reference's signatures and must compile
and link against libhipprune_host (CPU); on the GPU its results equal the reference's —
the stage output, the exact number of key reads its instrumented DirectKeySource logs
(acceptance #5's read-trace contract, replayed from the device's branch decisions), the
representative select_rep returns, build_mask through a KvView, and attention_row."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2502_08910_b200" / "_lib"
BIN = LIB / "ref_api_test"


def _build():
    import sysconfig  # noqa: F401
    cuda = Path("/usr/local/cuda")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "ref_api.cpp"),
           "-o", str(BIN), f"-L{LIB}", "-lhipprune_host", "-lhipprune_b200", f"-Wl,-rpath,{LIB}",
           f"-L{cuda / 'lib64'}", "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_reference_header_caller_compiles_and_links():
    if not (LIB / "libhipprune_host.so").exists():
        pytest.skip("host library not built")
    _build()
    assert BIN.exists()


@pytest.mark.gpu
def test_reference_header_caller_matches_reference(port, ref):
    _build()
    got = json.loads(subprocess.run([str(BIN)], check=True, capture_output=True, text=True).stdout)
    q, k, v = ref.generate(heads=2, layers=1, seq_kv=512, seq_q=16, dim=16, seed=11)
    q, k, v = q[0], k[0], v[0]
    idx = np.arange(16, 480)
    want, total, _ = ref.run_pruning_stage((16, 8, 64), idx, q, k, stream=32, qstart=512 - 16, count_reads=True)
    assert got["stage"] == want.tolist()
    assert got["stage_reads"] == total
    chunk = idx[40:48]
    rep, reads = port.select_rep(q[1], chunk, k[1], stream=32, qstart=512 - 16, chunk_index=5, chunk_count=58)
    assert got["rep"] == rep and got["rep_reads"] == len(reads)
    lists, _, bs, off = port.build_mask(q, k, [(16, 8, 64), (8, 4, 32)], sink=16, stream=32)
    assert got["mask_blocks"] == [l.tolist() for l in lists]
    sel = port.selected_indices(lists, bs, 16, 32, off, 15)
    row = port.attention_row(q[0, 15], sel, off + 15, k[0], v[0])
    assert np.abs(np.asarray(got["row"]) - row).max() <= 1e-3 * np.abs(row).max()

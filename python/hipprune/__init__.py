"""Hierarchical context pruning engine on B200: block-sparse attention masks,
stage-cached decoding and a two-tier paged KV cache — the reference ``hipprune``
package (proj/python/hipprune/__init__.py) with the same 14 names, served by
``_hipprune`` (pybind11 over the C++ host layer, include/hipprune/*.hpp, and the
sm_100a kernels of libhipprune_b200.so). Pruning, block-sparse and dense
attention and the decode engine run on the GPU; without a CUDA device they raise
RuntimeError (there is no CPU fallback). ``run_report`` / ``config_hash`` are the
reference's report plumbing over the same operators (``_reports``).

Extra names: ``DecodeEngine``, ``chunk_sparsity_histogram``, ``device_available``,
``ContractViolation``, ``FormatError``.
"""
import os
import sys
from pathlib import Path

try:  # an installed wheel ships _hipprune next to this package
    from . import _hipprune  # noqa: F401
except ImportError:  # in-tree: the module built by paper_2502_08910_b200.build
    _LIB = Path(__file__).resolve().parents[2] / "paper_2502_08910_b200" / "_lib"
    if str(_LIB) not in sys.path:
        sys.path.insert(0, str(_LIB))
    import _hipprune  # noqa: E402

    sys.modules[__name__ + "._hipprune"] = _hipprune

from ._reports import config_hash, run_report  # noqa: E402

_m = sys.modules[__name__ + "._hipprune"]
ContractViolation = _m.ContractViolation
DecodeEngine = _m.DecodeEngine
FormatError = _m.FormatError
SparseBlockMask = _m.SparseBlockMask
Workload = _m.Workload
attention_recall = _m.attention_recall
block_sparse_attention = _m.block_sparse_attention
build_mask = _m.build_mask
chunk_sparsity_histogram = _m.chunk_sparsity_histogram
dense_attention = _m.dense_attention
device_available = _m.device_available
dump_checksum = _m.dump_checksum
exact_topk = _m.exact_topk
generate = _m.generate
load_dump = _m.load_dump
save_dump = _m.save_dump
selected_indices = _m.selected_indices
del _m, os

__all__ = [
    "SparseBlockMask",
    "Workload",
    "attention_recall",
    "block_sparse_attention",
    "build_mask",
    "config_hash",
    "dense_attention",
    "dump_checksum",
    "exact_topk",
    "generate",
    "load_dump",
    "run_report",
    "save_dump",
    "selected_indices",
]

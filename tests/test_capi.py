"""The C-ABI library (include/hipprune_b200.h) — CPU-side checks, no compute calls.

* it loads and exports every function the header declares;
* status codes / messages follow the reference's exception types;
* the host helper hp_build_rope_table is bit-identical to the reference table.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hipprune_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def capi():
    from paper_2502_08910_b200 import _capi
    _capi.lib()
    return _capi


def test_header_symbols_exported(capi):
    decl = declared_functions()
    assert len(decl) >= 15
    lib = capi.lib()
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert set(capi.EXPORTS) == set(decl)


def test_library_is_sm100a():
    """The shipped library carries sm_100a SASS (cross-compiled here)."""
    import shutil
    import subprocess
    from paper_2502_08910_b200._capi import LIB_PATH
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_codes_map_to_reference_exceptions(capi):
    lib = capi.lib()
    # StageConfig::validate (pruning.cpp:102-109): invalid_argument -> HP_INVALID_ARGUMENT
    a = capi.StageArgs(query_block=64, chunk_size=4, keep=10)
    rc = lib.hp_prune_stage(C.byref(a), None)
    assert rc == 2 and b"k must be a positive multiple of l_c" in lib.hp_last_error()
    a = capi.StageArgs(query_block=64, chunk_size=0, keep=8)
    assert lib.hp_prune_stage(C.byref(a), None) == 2
    with pytest.raises(ValueError):
        capi.check(lib.hp_prune_stage(C.byref(a), None))
    # build_rope_table (tensor.cpp:30-44)
    buf = np.zeros(8, np.float32)
    assert lib.hp_build_rope_table(4, 3, 10000.0, buf.ctypes.data, buf.ctypes.data) == 2
    assert lib.hp_build_rope_table(0, 4, 10000.0, buf.ctypes.data, buf.ctypes.data) == 2


def test_rope_table_bit_identical_to_reference(capi, port):
    lib = capi.lib()
    for max_pos, d in ((1, 2), (4, 4), (300, 128), (70, 16)):
        cos = np.empty((max_pos, d // 2), np.float32)
        sin = np.empty((max_pos, d // 2), np.float32)
        assert lib.hp_build_rope_table(max_pos, d, 10000.0, cos.ctypes.data, sin.ctypes.data) == 0
        c2, s2 = port.rope_table(max_pos, d)
        assert np.array_equal(cos, c2) and np.array_equal(sin, s2)


def test_device_probe_reports_no_device_here(capi):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    assert capi.lib().hp_device_available() == 0
    from paper_2502_08910_b200 import device as D
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        D.require_cuda()


def test_product_library_has_no_dev_hooks():
    """The developer hooks (include/hipprune_b200_dev.h) exist only in dev builds."""
    import ctypes
    from paper_2502_08910_b200 import _capi
    if not _capi.LIB_PATH.exists() or "trace" in _capi.LIB_PATH.name or "HP_LIB" in __import__("os").environ:
        pytest.skip("product library not built / a dev build is selected")
    L = ctypes.CDLL(str(_capi.LIB_PATH))
    for name in ("hp_trace_enable", "hp_layer_trace_enable", "hp_debug_cut", "hp_debug_prefill_progress"):
        assert not hasattr(L, name), name

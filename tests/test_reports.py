"""The reference's report plumbing served by the drop-in package (python/hipprune):
config_hash equals the reference's FNV-1a over its canonical config rendering
(config.cpp:197-254), checked against the unmodified reference library (oracle/_ref)."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "python"))

OVERRIDE_SETS = [
    [],
    ["workload.heads=1", "workload.layers=1", "workload.seq_kv=256", "workload.dim=16",
     "plan.stages=16:8:64,8:4:32", "plan.sink=16", "plan.stream=32", "plan.refresh=4,2",
     "store.page_size=8", "store.mask_capacity=16", "store.sa_capacity=16", "run.steps=8"],
    ["plan.preset=5k", "cost.host=40.25", "workload.locality=12.5", "needle.position=77", "needle.strength=100"],
    ["plan.preset=flash", "policy.extension=1", "policy.cutoff=2", "run.capacity_sweep=4,8"],
]


REF_BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ref_config_hash"


def test_config_hash_matches_reference():
    """Against the unmodified reference (oracle/_ref/ref_config_hash, its own process)."""
    import subprocess
    from hipprune import _reports
    if not REF_BIN.exists():
        pytest.skip("oracle/_ref/ref_config_hash not built (needs /root/reference)")
    for ov in OVERRIDE_SETS:
        want = int(subprocess.run([str(REF_BIN), *ov], capture_output=True, text=True, check=True).stdout)
        assert _reports.config_hash(ov) == want, ov


def test_config_errors():
    from hipprune import _reports
    with pytest.raises(_reports.ConfigError):
        _reports.config_hash(["no.such.key=1"])
    with pytest.raises(_reports.ConfigError):
        _reports.config_hash(["workload.heads=x"])
    with pytest.raises(_reports.ConfigError):
        _reports.config_hash(["plan.stages=1:2"])

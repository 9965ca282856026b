"""hipprune_b200: B200-native InfiniteHiP attention hot path.

Hierarchical context pruning -> paged block-sparse attention -> GPU block cache,
as hand-written sm_100a CUDA behind a C ABI (include/hipprune_b200.h), mirroring
the reference hipprune operator API. See DESIGN.md.
"""
from . import _capi  # noqa: F401

__version__ = "0.1.0"

"""Synthetic inputs shaped like the reference generator (workload.cpp:147-189):
q, v ~ N(0,1); k = N(0,1) box-smoothed over +-locality rows, renormalised to
||k|| = sqrt(d). Values differ from libstdc++'s stream (a different RNG) but
the statistics — and therefore the pruning behaviour — are the same."""
from __future__ import annotations

import numpy as np


def smooth_keys(noise: np.ndarray, locality: int = 64) -> np.ndarray:
    t, d = noise.shape
    half = min(int(locality), t)
    pre = np.zeros((t + 1, d), np.float64)
    np.cumsum(noise, axis=0, dtype=np.float64, out=pre[1:])
    r = np.arange(t)
    lo = np.maximum(r - half, 0)
    hi = np.minimum(r + half, t - 1)
    out = ((pre[hi + 1] - pre[lo]) / (hi - lo + 1)[:, None]).astype(np.float32)
    norm = np.sqrt((out.astype(np.float64) ** 2).sum(1))
    scale = np.where(norm > 0, np.sqrt(d) / np.where(norm > 0, norm, 1), 1.0).astype(np.float32)
    return out * scale[:, None]


def workload(seed: int, h_q: int, h_kv: int, t_q: int, t_kv: int, d: int, locality: int = 64,
             bf16: bool = False):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((h_q, t_q, d), dtype=np.float32)
    k = np.stack([smooth_keys(rng.standard_normal((t_kv, d), dtype=np.float32), locality)
                  for _ in range(h_kv)])
    v = rng.standard_normal((h_kv, t_kv, d), dtype=np.float32)
    if bf16:
        q, k, v = (round_bf16(x) for x in (q, k, v))
    return q, k, v


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as fp32 (the values both sides see)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)

"""Synthetic Q/K/V generated on the device with the reference generator's recipe
(workload.cpp:147-189): Q, V ~ N(0,1); K = N(0,1) noise box-smoothed over
+-locality rows (prefix sums in double), rows renormalised to ||k|| = sqrt(d).
Used by bench.py (no datasets or checkpoints are reachable); the RNG stream is
torch's, not libstdc++'s, so values differ from the reference generator while
the statistics — and hence the pruning workload — match.
"""
from __future__ import annotations

import torch


def smooth_keys(noise: torch.Tensor, locality: int = 64) -> torch.Tensor:
    """noise [T, d] fp32 -> smoothed, renormalised keys [T, d] fp32 (same device)."""
    t, d = noise.shape
    half = min(int(locality), t)
    pre = torch.zeros((t + 1, d), dtype=torch.float64, device=noise.device)
    torch.cumsum(noise.double(), dim=0, out=pre[1:])
    r = torch.arange(t, device=noise.device)
    lo = (r - half).clamp_min(0)
    hi = (r + half).clamp_max(t - 1)
    out = ((pre[hi + 1] - pre[lo]) / (hi - lo + 1).unsqueeze(1).double()).float()
    norm = out.double().pow(2).sum(1).sqrt()
    scale = torch.where(norm > 0, (d ** 0.5) / norm.clamp_min(1e-300), torch.ones_like(norm)).float()
    return out * scale.unsqueeze(1)


@torch.no_grad()
def generate(h_q: int, h_kv: int, t_kv: int, d: int, *, t_q: int = 1, seed: int = 1,
             locality: int = 64, dtype=torch.bfloat16, device="cuda"):
    """Returns q fp32 [h_q, t_q, d] (bf16-rounded when dtype is bf16) and k, v
    [h_kv, t_kv, d] in `dtype`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = torch.randn((h_q, t_q, d), generator=g, device=device, dtype=torch.float32)
    k = torch.empty((h_kv, t_kv, d), dtype=dtype, device=device)
    for h in range(h_kv):
        noise = torch.randn((t_kv, d), generator=g, device=device, dtype=torch.float32)
        k[h] = smooth_keys(noise, locality).to(dtype)
        del noise
    v = torch.randn((h_kv, t_kv, d), generator=g, device=device, dtype=torch.float32).to(dtype)
    if dtype == torch.bfloat16:
        q = q.to(torch.bfloat16).float()
    return q, k, v

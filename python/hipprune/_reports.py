"""The reference's report plumbing over this package's device operators:
``run_report`` (decode-sim, sparsity-report) and ``config_hash``.

Follows /root/reference/proj/src/config.cpp (defaults, presets, ``key=value``
overrides, the canonical rendering hashed with FNV-1a) and commands.cpp
(run_decode_sim: one scenario per number of frozen leading stages — "none",
"s1", "s12", ..., "all" — each a DecodeEngine run with per-step JSONL telemetry;
run_sparsity_report: exact top-k mass per chunk size). The engine runs on the
device; its page accounting (Mask / SA banks, CostModel latency) equals the
reference engine's step by step (tests/test_gpu_decode_sim.py).
"""
from __future__ import annotations

import copy
import json
import zlib

import numpy as np

_U64 = (1 << 64) - 1


class ConfigError(RuntimeError):
    """hipprune::ConfigError (config.hpp)."""


def _preset(name: str) -> dict:
    if name in ("3k", "fast", "flash"):
        stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    elif name == "5k":
        stages = [(64, 64, 32768), (64, 32, 16384), (64, 16, 4096)]
    else:
        raise ConfigError(f"unknown preset '{name}' (expected 3k, 5k, fast, flash)")
    refresh = {"fast": [32, 16, 8], "flash": [96, 24, 8]}.get(name, [16, 8, 4])
    return {"stages": stages, "sink": 256, "stream": 1024, "refresh": refresh}


def default_config() -> dict:
    c = {"workload": {"heads": 2, "layers": 2, "seq_kv": 8192, "seq_q": 64, "dim": 64, "locality": 64.0,
                      "seed": 1, "dump": ""},
         "needles": [],
         "store": {"page_size": 64, "mask_capacity": 128, "sa_capacity": 64},
         "cost": {"device": 1.0, "host": 31.5},
         "run": {"steps": 48, "seeds": 20, "threads": 1, "sparsity_topk": 2048, "capacity_sweep": [8, 16, 32, 64, 128]}}
    _apply_preset(c, "3k")
    return c


def _apply_preset(c: dict, name: str) -> None:
    c["plan"] = _preset(name)
    c["policy"] = {"extension": False, "cutoff": 3}
    c["preset"] = name


def _u64(key, v):
    try:
        x = int(v.strip(), 10)
        if x < 0:
            raise ValueError
        return x
    except ValueError:
        raise ConfigError(f"config key '{key}': not an unsigned integer: '{v}'") from None


def _f64(key, v):
    try:
        return float(v)
    except ValueError:
        raise ConfigError(f"config key '{key}': not a number: '{v}'") from None


def apply_override(c: dict, key: str, value: str) -> None:
    """config.cpp apply_override: one ``key=value``."""
    w, p, s, r = c["workload"], c["plan"], c["store"], c["run"]
    simple = {"workload.heads": (w, "heads", _u64), "workload.layers": (w, "layers", _u64),
              "workload.seq_kv": (w, "seq_kv", _u64), "workload.seq_q": (w, "seq_q", _u64),
              "workload.dim": (w, "dim", _u64), "workload.locality": (w, "locality", _f64),
              "workload.seed": (w, "seed", _u64), "plan.sink": (p, "sink", _u64),
              "plan.stream": (p, "stream", _u64), "policy.cutoff": (c["policy"], "cutoff", _u64),
              "store.page_size": (s, "page_size", _u64), "store.mask_capacity": (s, "mask_capacity", _u64),
              "store.sa_capacity": (s, "sa_capacity", _u64), "cost.device": (c["cost"], "device", _f64),
              "cost.host": (c["cost"], "host", _f64), "run.steps": (r, "steps", _u64),
              "run.seeds": (r, "seeds", _u64), "run.threads": (r, "threads", _u64),
              "run.sparsity_topk": (r, "sparsity_topk", _u64)}
    if key in simple:
        d, k, f = simple[key]
        d[k] = f(key, value)
    elif key == "workload.dump":
        w["dump"] = value
    elif key in ("needle.position", "needle.strength"):
        if not c["needles"]:
            c["needles"].append([0, 0.0])
        if key == "needle.position":
            c["needles"][0][0] = _u64(key, value)
        else:
            c["needles"][0][1] = float(np.float32(_f64(key, value)))
    elif key == "plan.preset":
        _apply_preset(c, value)
    elif key == "plan.stages":
        stages = []
        for part in [x.strip() for x in value.split(",")]:
            f = [x.strip() for x in part.split(":")]
            if len(f) != 3:
                raise ConfigError(f"plan.stages: expected bq:lc:k, got '{part}'")
            stages.append(tuple(_u64(key, x) for x in f))
        p["stages"] = stages
    elif key == "plan.refresh":
        p["refresh"] = [_u64(key, x.strip()) for x in value.split(",")]
    elif key == "policy.extension":
        c["policy"]["extension"] = _u64(key, value) != 0
    elif key == "run.capacity_sweep":
        r["capacity_sweep"] = [_u64(key, x.strip()) for x in value.split(",")]
    else:
        raise ConfigError(f"unknown config key '{key}'")


def config_from_overrides(overrides) -> dict:
    c = default_config()
    for kv in overrides:
        if "=" not in kv:
            raise ConfigError(f"override must be key=value: '{kv}'")
        k, v = kv.split("=", 1)
        apply_override(c, k, v)
    return c


def _g(x) -> str:
    """std::ostream << double (default precision 6, %g)."""
    return format(x, "g")


def canonical_config(c: dict) -> str:
    """config.cpp canonical_config: the flat rendering the hash covers."""
    w, p, s, r = c["workload"], c["plan"], c["store"], c["run"]
    lines = [f"cost.device={_g(c['cost']['device'])}", f"cost.host={_g(c['cost']['host'])}"]
    lines += [f"needle.{i}={pos}:{_g(st)}" for i, (pos, st) in enumerate(c["needles"])]
    lines += [f"plan.preset={c['preset']}", "plan.refresh=" + ",".join(str(x) for x in p["refresh"]),
              f"plan.sink={p['sink']}", "plan.stages=" + ",".join(f"{a}:{b}:{k}" for a, b, k in p["stages"]),
              f"plan.stream={p['stream']}", f"policy.cutoff={c['policy']['cutoff']}",
              f"policy.extension={1 if c['policy']['extension'] else 0}",
              "run.capacity_sweep=" + ",".join(str(x) for x in r["capacity_sweep"]), f"run.seeds={r['seeds']}",
              f"run.sparsity_topk={r['sparsity_topk']}", f"run.steps={r['steps']}", f"run.threads={r['threads']}",
              f"store.mask_capacity={s['mask_capacity']}", f"store.page_size={s['page_size']}",
              f"store.sa_capacity={s['sa_capacity']}", f"workload.dim={w['dim']}", f"workload.dump={w['dump']}",
              f"workload.heads={w['heads']}", f"workload.layers={w['layers']}",
              f"workload.locality={_g(w['locality'])}", f"workload.seed={w['seed']}", f"workload.seq_kv={w['seq_kv']}",
              f"workload.seq_q={w['seq_q']}"]
    return "\n".join(lines) + "\n"


def _fnv1a(text: str) -> int:
    h = 0xCBF29CE484222325
    for ch in text.encode():
        h ^= ch
        h = (h * 0x100000001B3) & _U64
    return h


def config_hash(overrides=()) -> int:
    return _fnv1a(canonical_config(config_from_overrides(list(overrides))))


def _workload(c: dict, decode: bool):
    from . import _hipprune as H
    w = c["workload"]
    if w["dump"]:
        return H.load_dump(w["dump"])
    seq_q = w["seq_kv"] if decode else w["seq_q"]
    return H.generate(heads=w["heads"], layers=w["layers"], seq_kv=w["seq_kv"], seq_q=seq_q, dim=w["dim"],
                      locality=w["locality"], seed=w["seed"], needles=[tuple(n) for n in c["needles"]])


def _header(c: dict, command: str) -> dict:
    return {"command": command, "config_hash": hex(_fnv1a(canonical_config(c))), "seed": c["workload"]["seed"]}


def _decode_sim(c: dict) -> dict:
    from . import _hipprune as H
    full = _workload(c, decode=True)
    steps = c["run"]["steps"]
    if steps == 0 or steps >= full.seq_len_kv:
        raise ConfigError("decode simulation: run.steps must be in (0, seq_kv)")
    prefill_len = full.seq_len_kv - steps
    p = c["plan"]
    q_len = min(p["stages"][0][0], prefill_len)
    n = len(p["stages"])
    scenarios = []
    for cached in range(n + 1):
        name = "none" if cached == 0 else "all" if cached == n else "s1" + "".join(str(i + 1) for i in range(1, cached))
        scenarios.append((name, [i < cached for i in range(n)]))
    summary = _header(c, "decode-sim")
    summary["steps"] = steps
    rows, extras = [], {}
    csv = "scenario,mean_step_latency,mask_hit_ratio,sa_hit_ratio,bsa_latency" + "".join(
        f",stage{i + 1}_latency" for i in range(n)) + "\n"
    for name, frozen in scenarios:
        eng = H.DecodeEngine(full, prefill_len, q_len=q_len, stages=[tuple(s) for s in p["stages"]], sink=p["sink"],
                             stream=p["stream"], refresh=list(p["refresh"]), extension=c["policy"]["extension"],
                             page_size=c["store"]["page_size"], mask_capacity=c["store"]["mask_capacity"],
                             sa_capacity=c["store"]["sa_capacity"], device_cost=c["cost"]["device"],
                             host_cost=c["cost"]["host"], cutoff=c["policy"]["cutoff"])
        eng.set_frozen_stages(frozen)
        eng.prefill()
        eng.reset_store_stats()
        stage_lat = [0.0] * n
        bsa = total = 0.0
        mh = ma = sh = sa = 0
        crc = 0
        msum = 0.0
        lines = []
        for _ in range(steps):
            out, tel = eng.step()
            for i, x in enumerate(tel["stage_latency"]):
                stage_lat[i] += x
            bsa += tel["bsa_latency"]
            total += tel["bsa_latency"] + sum(tel["stage_latency"])
            mh += tel["mask_hits"]; ma += tel["mask_accesses"]; sh += tel["sa_hits"]; sa += tel["sa_accesses"]
            msum += tel["mask_sizes"][-1]
            crc = zlib.crc32(np.ascontiguousarray(out, np.float32).tobytes(), crc)
            lines.append(json.dumps({k: tel[k] for k in ("step", "refreshed", "stage_latency", "bsa_latency",
                                                         "mask_hits", "mask_accesses", "sa_hits", "sa_accesses",
                                                         "mask_sizes")}))
        rows.append({"name": name, "frozen_stages": frozen, "mean_step_latency": total / steps,
                     "stage_latency": stage_lat, "bsa_latency": bsa, "mask_hits": mh, "mask_accesses": ma,
                     "mask_hit_ratio": mh / ma if ma else None, "sa_hits": sh, "sa_accesses": sa,
                     "sa_hit_ratio": sh / sa if sa else None, "mean_final_mask_size": msum / steps,
                     "output_crc": crc})
        csv += f"{name},{total / steps},{mh / ma if ma else ''},{sh / sa if sa else ''},{bsa}" + "".join(
            f",{x}" for x in stage_lat) + "\n"
        extras[name + ".jsonl"] = "\n".join(lines) + "\n"
    summary["scenarios"] = rows
    return {"json": json.dumps(summary, indent=2) + "\n", "csv": csv, "extras": extras}


def _sparsity_report(c: dict) -> dict:
    from . import _hipprune as H
    wl = _workload(c, decode=False)
    k = min(c["run"]["sparsity_topk"], wl.seq_len_kv)
    edges = (0.125, 0.25, 0.5, 1.0)
    rows = []
    csv = "chunk_size,empty_fraction,share_le_0.125,share_le_0.25,share_le_0.5,share_le_1\n"
    for cs in (8, 16, 32, 64, 128, 256):
        if cs > wl.seq_len_kv:
            continue
        empties, bins, nonempty = [], [0.0] * 4, 0
        for layer in range(wl.num_layers):
            for h in range(wl.num_heads):
                q = wl.q(layer, h)[wl.seq_len_q - 1]
                counts, empty = H.chunk_sparsity_histogram(q, wl.k(layer, h), k, cs)
                empties.append(empty)
                for cnt in counts:
                    if cnt == 0:
                        continue
                    share = cnt / k
                    b = next((i for i, e in enumerate(edges) if share <= e), 3)
                    bins[b] += 1
                    nonempty += 1
        shares = [b / nonempty if nonempty else 0.0 for b in bins]
        rows.append({"chunk_size": cs, "top_k": k, "empty_fraction": float(np.mean(empties)) if empties else 0.0,
                     "nonempty_share_bins": shares})
        csv += f"{cs},{rows[-1]['empty_fraction']}" + "".join(f",{x}" for x in shares) + "\n"
    out = _header(c, "sparsity-report")
    out["rows"] = rows
    return {"json": json.dumps(out, indent=2) + "\n", "csv": csv, "extras": {}}


def run_report(command: str, overrides=()) -> dict:
    """bindings.cpp run_report: {"json", "csv", "extras"} of one report command."""
    c = config_from_overrides(list(overrides))
    if command == "decode-sim":
        return _decode_sim(c)
    if command == "sparsity-report":
        return _sparsity_report(c)
    if command in ("recall-report", "offload-report"):
        raise NotImplementedError(f"run_report('{command}'): not served by the B200 package (decode-sim and "
                                  "sparsity-report are; the recall quality checks are tests/test_gpu_quality.py)")
    raise ValueError(f"unknown report command '{command}'")

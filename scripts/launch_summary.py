"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): this repo's kernels,
launches, total and mean time, share of the total. Dev tool:
python scripts/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/..._summary.txt"""
import collections
import csv
import re
import sys

OURS = r"(decode_|materialize_kernel|prune_|bsa_|select|selected_kernel|commit_|remap_kernel|lse_|append|cache_)"

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hd = rows[h]
ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
agg, missing = collections.OrderedDict(), collections.Counter()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].replace("<unnamed>::", "").split("(")[0].replace("void ", "")
    if not re.match(OURS, name):
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        v = float("nan")
    if v != v:  # no value (e.g. a launch that failed under the profiler)
        missing[name] += 1
        continue
    v = {"ns": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(r[ui], v / 1e3)
    agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
print(f"# ncu launch list of `{sys.argv[2] if len(sys.argv) > 2 else '?'}`")
print("# (--metrics gpu__time_duration.sum --clock-control none): this repo's kernels. ncu serialises launches")
print("# (no PDL overlap, cold caches), so per-launch times exceed the in-graph ones; the SHARE is what counts.")
print(f"{'kernel':52s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:52]:52s} {len(v):8d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:5.1f}%")
if missing:
    print("# launches ncu reported no value for: " + ", ".join(f"{k} x{n}" for k, n in missing.items()))

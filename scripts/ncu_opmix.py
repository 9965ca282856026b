"""Executed-instruction mix (by opcode) of the N-th kernel in an ncu report (source page). Dev tool."""
import csv, io, subprocess, sys, collections
rep, nth = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
s = starts[nth]; e = starts[nth + 1] if nth + 1 < len(starts) else len(rows)
block = rows[s:e]
print(block[0][1][:100])
h = block[1]; data = [r for r in block[2:] if len(r) == len(h)]
src = h.index("Source"); ie = h.index("Instructions Executed")
mix = collections.Counter()
for r in data:
    op = r[src].split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    mix[o.split(".")[0]] += int(float(r[ie] or 0))
tot = sum(mix.values())
print("total", tot)
for o, c in mix.most_common(25):
    print(f"{o:12s} {c:10d} {100*c/tot:5.1f}%")

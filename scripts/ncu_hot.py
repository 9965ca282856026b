"""Top SASS hot spots (stall samples) of the N-th profiled kernel in an ncu report."""
import csv, io, subprocess, sys
rep, nth = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
s = starts[nth]; e = starts[nth + 1] if nth + 1 < len(starts) else len(rows)
block = rows[s:e]
print(block[0][1][:100])
h = block[1]; data = [r for r in block[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data) or 1
print("samples", tot, "instructions", len(data))
for k, r in sorted(enumerate(data), key=lambda kr: -float(kr[1][si] or 0))[:top]:
    rs = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:2]
    print(f"{k:5d} {float(r[si] or 0):6.0f} {100*float(r[si] or 0)/tot:5.1f}% {r[ie]:>9s} {r[src][:58]:58s} {rs}")

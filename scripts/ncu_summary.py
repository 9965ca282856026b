"""Summarise an ncu report: per-kernel duration, DRAM bytes, key utilisation, top stalls."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__waves_per_multiprocessor", "sm__cycles_elapsed.avg.per_second"]
idx = [h.index(w) for w in want if w in h]
for r in rows[2:]:
    print("----")
    for i in idx:
        print(f"  {h[i]:55s} {r[i][:70]} {rows[1][i]}")
    st = [(float(r[i]), h[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in range(len(h))
          if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued") and r[i]]
    tot = sum(x for x, _ in st) or 1
    st.sort(reverse=True)
    print("  stalls:", ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in st[:6]))

#!/usr/bin/env python
"""Per-source-line table of one kernel in an ncu report: samples, warp instructions,
avg threads, long-scoreboard stalls.
    python scripts/src_cols.py <report.ncu-rep> <kernel-regex> [n] [sort-column]
"""
import csv, io, os, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
col = {k: i for i, k in enumerate(h)}
data = []
fname = "?"
for r in rows:
    if r and r[0] in ("File Path", "File Name") and len(r) > 1:
        fname = os.path.basename(r[1])
        continue
    if len(r) != len(h) or r[0] == "Line No" or r[2] != "-" or r[0] in ("", "-"):
        continue
    def f(k):
        try:
            return float(r[col[k]])
        except (ValueError, KeyError):
            return 0.0
    data.append((f(key), fname[:10] + ":" + r[0], r[1][:80], f("# Samples"), f("Instructions Executed"),
                 f("Avg. Threads Executed"), f("stall_long_sb"), f("stall_wait")))
tot_i = sum(d[4] for d in data)
tot_s = sum(d[3] for d in data)
print(f"total warp inst {tot_i:.3e}  samples {tot_s:.0f}")
print(f"{'line':>16} {'inst%':>6} {'samp%':>6} {'thr':>5} {'lsb':>6} {'wait':>6}  source")
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[1]:>16} {100*d[4]/tot_i:6.2f} {100*d[3]/max(tot_s,1):6.2f} {d[5]:5.1f} {d[6]:6.0f} {d[7]:6.0f}  {d[2]}")

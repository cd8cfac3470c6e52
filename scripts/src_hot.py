#!/usr/bin/env python
"""Rank source lines / SASS of one kernel in an ncu report by stall samples.
    python scripts/src_hot.py <report.ncu-rep> <kernel-regex> [n]
"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cuda, sass = [], []
for r in rows[3:]:
    if len(r) < 5:
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    if r[0] not in ("-", ""):
        cuda.append((s, r[0], r[1][:100]))
    if r[2] != "-":
        sass.append((s, r[2][-5:], r[3][:90]))
print("total samples", sum(s for s, _, _ in cuda))
for s, l, t in sorted(cuda, reverse=True)[:n]:
    print(f"{s:6d} {l:>5} {t}")
print()
for s, a, t in sorted(sass, reverse=True)[:n]:
    print(f"{s:6d} {a} {t}")

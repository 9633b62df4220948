#!/usr/bin/env python3
"""Hottest SASS lines of an ncu report (warp-stall samples): ncu_hot.py REP [N]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
k = h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[1:] if len(r) > k and r[k].isdigit()]
tot = sum(int(r[k]) for r in body) or 1
for i, r in sorted(enumerate(body), key=lambda t: -int(t[1][k]))[:n]:
    print(f"{int(r[k]):6d} {100 * int(r[k]) / tot:5.1f}%  #{i:4d} {r[1].strip()[:100]}")

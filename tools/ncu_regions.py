#!/usr/bin/env python3
"""Stall reasons summed over SASS line ranges containing given mnemonics:
ncu_regions.py REP  -> per-mnemonic-group totals of each stall reason."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in stalls}
ie = h.index("Instructions Executed")
tot = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(float)
for r in rows[1:]:
    if len(r) <= ie:
        continue
    op = r[1].strip().split()
    if not op:
        continue
    m = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else op[0])
    m = m.split(".")[0]
    try:
        cnt[m] += float(r[ie] or 0)
    except ValueError:
        pass
    for c in stalls:
        try:
            tot[m][c] += float(r[idx[c]] or 0)
        except ValueError:
            pass
grand = sum(sum(v.values()) for v in tot.values()) or 1
for m, v in sorted(tot.items(), key=lambda t: -sum(t[1].values()))[:14]:
    s = sum(v.values())
    top = ", ".join(f"{k[6:]} {100 * x / grand:.1f}" for k, x in sorted(v.items(), key=lambda t: -t[1])[:4] if x)
    print(f"{m:10s} {100 * s / grand:5.1f}%  inst {cnt[m]:.3g}  [{top}]")

#!/usr/bin/env python3
"""Summarise an ncu report (key roofline metrics per captured launch) and a
launch list CSV (per-kernel share of device time) into markdown.

usage: ncu_summary.py --rep X.ncu-rep [--launches launches.csv] [--flops F ...]
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("l1tex__m_l1tex2xbar_write_bytes.sum", "SM->L2 write bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block", "smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us (serialised) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"### `{d.get('Kernel Name', '?')[:90]}` grid {d.get('Grid Size')} block {d.get('Block Size')}")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, label in KEYS:
            if k in d:
                out.append(f"| {label} (`{k}`) | {d[k]} {units[hdr.index(k)]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
        print()
    if a.rep:
        print(report(a.rep))

#!/usr/bin/env python3
"""Print selected raw metrics of every kernel in an .ncu-rep (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum"]
STALLS = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    for row in r[2:]:
        print("-----", row[h.index("Kernel Name")][:60])
        for k, un, v in zip(h, u, row):
            if k in KEYS or k in extra or (k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")
                                           and v not in ("0", "") and float(v.replace(",", "")) > 0.05):
                print(f"  {k} {un} {v}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""One-screen summary of a bench.py JSON line: bench_brief.py FILE."""
import json
import sys

try:
    b = json.load(open(sys.argv[1]))
except Exception as e:  # noqa: BLE001
    print("bench parse failed", e)
    sys.exit(0)
print("TTFT", b.get("ttft_p50_ms"), "e2e", b.get("e2e", {}).get("ttft_p50_ms"), "r_c", b["config"].get("r_c"))
print("restore", b.get("restore"))
h = b.get("roofline", {})
print("roofline", h.get("class"), h.get("frac"), h.get("avg_launch_us"), "ser", h.get("achieved_serialised"))
for k, v in b.get("rooflines", {}).items():
    print("  ", k, v.get("frac"), v.get("avg_launch_us"), v.get("ms_per_step"), v.get("achieved_serialised"))
print("policies", {k: v["ttft_ms"] for k, v in b.get("policies", {}).items()})
print("calib", b.get("calibration", {}).get("calibration_ttft_ms"))
tl = b.get("timeline_ms")
if tl:
    print("load_done", tl.get("load_done"))
    print("new_done ", tl.get("new_prefill_done"))

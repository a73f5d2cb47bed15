"""Prints tools/pair_profile.py output as a per-phase table (all pairs vs the slowest pair)."""
import json
import sys

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pair_profile.json"))
print("kernel_ms", round(d["kernel_ms"], 1), "slowest pair", d.get("slowest_pair"),
      [(t["pair"], t["events"], t["plan"]) for t in d["top"][:3]])
for k, v in d["phases"].items():
    w = d.get("slowest_phases", {}).get(k, {"count": 0, "cycles_per": 0, "cycles": 0})
    print(f"{k:20s} all: n={v['count']:10d} c/n={round(v['cycles_per']):6d} | slowest: n={w['count']:8d} "
          f"c/n={round(w['cycles_per']):6d} tot={w['cycles'] / 1e6:8.1f}M")

#!/usr/bin/env python
"""Print the per-kernel-class table of a bench JSON line (file with the line last)."""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(line)
print("ms/step", round(d["ms_per_step"], 2), "K", d["config"].get("schwarz_iters_per_step"),
      "frac8", round(d["config"]["step_roofline"]["frac_of_8TBs"], 4))
for k, v in sorted((d.get("kernel_classes") or {}).items(), key=lambda x: -x[1]["ms"]):
    print(f"{k:18s} {v['launches']:5d} {v['ms']:8.2f} {v['GBps'] or 0:8.0f}")

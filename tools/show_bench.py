#!/usr/bin/env python
"""Print the key numbers of a bench.py JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value %.4g %s  ms/step %.2f  K %s" % (d["value"], d["unit"], d["ms_per_step"], d["config"].get("schwarz_iters_per_step")))
print("step roofline", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d["config"]["step_roofline"].items()})
print("dominant", d["roofline"]["kernel"], "%.0f GB/s frac %.3f share %.3f" % (d["roofline"]["achieved"] or 0, d["roofline"]["frac"] or 0, d["roofline"]["share_of_step"]))
tot = sum(v["ms"] for v in d["kernel_classes"].values())
for k, v in list(d["kernel_classes"].items())[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print("  %-18s %5d launches %8.1f ms %5.1f%%  %s GB/s" % (k, v["launches"], v["ms"], 100 * v["ms"] / tot,
                                                            "%.0f" % v["GBps"] if v["GBps"] else "-"))
print("e2e", d.get("e2e"), "\ncpu", d.get("cpu_baseline"), "\nclocks", d.get("clocks"), "launches", d.get("gpu_launches"))

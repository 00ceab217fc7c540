#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel template instance: launches, total/avg device time, share."""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, top=40):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0, ""])
    for d in data:
        name = d["Kernel Name"].replace("void ", "")
        key = re.sub(r"\(.*\)$", "", name)
        us = float(d["Metric Value"]) * UNIT[d["Metric Unit"]]
        a = agg[key]
        a[0] += 1
        a[1] += us
        a[2] = d["Grid Size"] + " x " + d["Block Size"]
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e3:.2f} ms total (cold-cache, serialised)\n")
    print("| kernel | launches | total ms | share | avg us | grid x block |")
    print("|---|---:|---:|---:|---:|---|")
    for k, (n, us, gb) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| `{k}` | {n} | {us / 1e3:.2f} | {100 * us / tot:.1f}% | {us / n:.1f} | {gb} |")


if __name__ == "__main__":
    main(sys.argv[1])

#!/usr/bin/env python
"""Summarise an `ncu --set full` report: per launch the device time, DRAM bytes
(read + write = the bench line's `traffic`), achieved DRAM GB/s, issue rate,
occupancy and executed instructions.  Usage: ncu_full_summary.py prof.ncu-rep"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print("| kernel | grid | " + " | ".join(c[1] for c in COLS) + " | DRAM GB/s |")
    print("|---|---|" + "---:|" * (len(COLS) + 1))
    for r in rows[2:]:
        vals = []
        t_us = mb = None
        for name, _ in COLS:
            if name not in h:
                vals.append("-")
                continue
            i = h.index(name)
            v = r[i].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[i], 1.0)
            except ValueError:
                vals.append(v)
                continue
            if name == "gpu__time_duration.sum":
                t_us = x
            if name.startswith("dram__bytes"):
                mb = (mb or 0.0) + x
            vals.append(f"{x:.1f}" if abs(x) < 1e6 else f"{x:.3g}")
        gbs = f"{mb * 1e6 / (t_us * 1e-6) / 1e9:.0f}" if (t_us and mb) else "-"
        name = r[h.index("Kernel Name")].replace("void ", "").split("(")[0]
        print(f"| `{name}` | {r[h.index('Grid Size')]} | " + " | ".join(vals) + f" | {gbs} |")
    # warp-state breakdown: cycles a warp spends per issued instruction, by reason
    st = [i for i, x in enumerate(h) if x.startswith("smsp__average_warps_issue_stalled_")
          and x.endswith("_per_issue_active.ratio")]
    if st:
        print()
        print("Warp stall reasons (cycles per issued instruction, top 5 per launch):")
        print()
        print("| kernel | top stall reasons |")
        print("|---|---|")
        for r in rows[2:]:
            vals = []
            for i in st:
                try:
                    vals.append((float(r[i].replace(",", "")), h[i][34:-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
            vals.sort(reverse=True)
            name = r[h.index("Kernel Name")].replace("void ", "").split("(")[0]
            print(f"| `{name}` | " + ", ".join(f"{b} {a:.2f}" for a, b in vals[:5]) + " |")


if __name__ == "__main__":
    main(sys.argv[1])

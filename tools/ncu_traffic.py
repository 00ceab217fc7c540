#!/usr/bin/env python
"""Per kernel class (bench.py / yy_api.cu ProfScope names) the mean DRAM bytes per
launch (dram__bytes_read.sum + dram__bytes_write.sum) of an `ncu --set full`
report -> the JSON profiles/traffic.json that bench.py's roofline `traffic` reads.
Usage: ncu_traffic.py prof.ncu-rep [build-label] > traffic.json"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

Q = ["T", "ur", "ut", "up"]
AX = ["r", "th", "ph"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def klass(name):
    m = re.search(r"k_(line_tma|line_th|line|resid|pres)<([^>]*)>", name)
    if not m:
        return None
    a = [int(re.sub(r"\(int\)|\(bool\)", "", x).strip().replace("true", "1").replace("false", "0"))
         for x in m.group(2).split(",")]
    if m.group(1) in ("line_tma", "line_th"):   # k_line_tma<Q, AX, MODE, P, M>, k_line_th<Q, AX, MODE>
        return f"sweep_{Q[a[0]]}_{AX[a[1]]}" + ("_fin" if a[2] == 2 else "")
    if m.group(1) == "resid":          # k_resid<Q, S, IB>
        return "resid_" + Q[a[0]] + ("" if a[0] == 0 else str(a[1]))
    if m.group(1) == "pres":           # k_pres<S>
        return f"pres_{a[0]}"
    q, ax, mode = a[0], a[1], a[2]     # k_line<Q, AX, MODE, S, P, M>
    if mode == 3:
        return None                    # radial-slab sweeps (multi-GPU layout)
    return f"sweep_{Q[q]}_{AX[ax]}" + ("_fin" if mode == 2 else "")


def main(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    acc = collections.defaultdict(list)
    for r in rows[2:]:
        c = klass(r[h.index("Kernel Name")])
        if c:
            b = float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]]
            acc[c].append(b)
    print(json.dumps({"build": label,
                      "source": "ncu --set full --clock-control none, dram__bytes_read.sum + dram__bytes_write.sum "
                                "per launch (mean over the captured launches of the class), C3",
                      "bytes_per_launch": {k: round(sum(v) / len(v)) for k, v in sorted(acc.items())}}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")

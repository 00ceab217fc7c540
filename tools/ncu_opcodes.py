#!/usr/bin/env python
"""Dynamic SASS opcode histogram of one launch of an `ncu --set full
--import-source on` report (the source page's executed instructions per SASS
line), per thread-element if the element count is given.
    python tools/ncu_opcodes.py report.ncu-rep LAUNCH_INDEX [elements]"""
import csv
import io
import subprocess
import sys


def main(path, idx, elems=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1]
    h = rows[1]
    ie, isrc = h.index("Instructions Executed"), h.index("Source")
    hist = {}
    for r in rows[2:]:
        if len(r) <= max(ie, isrc):
            continue
        src = r[isrc].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        op = op.split(".")[0]
        if not (r[ie] or "0").isdigit():     # a second source section repeats the SASS: stop
            break
        hist[op] = hist.get(op, 0) + int(r[ie] or 0)
    tot = sum(hist.values())
    name = name.replace("(int)", "").replace("void ", "").split("(")[0]
    print(f"`{name}`: {tot:.3g} warp instructions" +
          (f", {32 * tot / elems:.1f} thread instructions per element" if elems else ""))
    print()
    print("| opcode | warp inst | share |" + (" per element |" if elems else ""))
    print("|---|---:|---:|" + ("---:|" if elems else ""))
    for op, n in sorted(hist.items(), key=lambda kv: -kv[1])[:18]:
        print(f"| {op} | {n:.3g} | {100 * n / tot:.1f} % |" + (f" {32 * n / elems:.1f} |" if elems else ""))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), float(sys.argv[3]) if len(sys.argv) > 3 else None)

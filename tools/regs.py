#!/usr/bin/env python
"""Registers / spills per kernel from the ptxas log of csrc/build.sh."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1905_02300_b200/.ptxas.log").read()
pat = (r"Compiling entry function '(\S+)' for 'sm_100a'\nptxas info\s+: Function properties for \S+\n"
       r"\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers")
for m in re.finditer(pat, log):
    t = re.search(r"(k_\w+?)I(.*)EE?v", m.group(1))
    name = (t.group(1) + "<" + t.group(2) + ">") if t else m.group(1)
    print(f"{name:60s} regs {m.group(5):>4s} spill {m.group(3)}")

#!/usr/bin/env python
"""Copy one evidence run (tools/gpu_round2_final.sh / gpu_round2b.sh outputs under
gpurun_out/ or a directory given as argv[1]) into profiles/r02_* and regenerate
BASELINE.md §5:  bench logs -> the JSON line, logs as they are."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
BENCH = {"bench_c1": "r02_bench_c1", "bench_c2": "r02_bench_c2", "bench_c2_200": "r02_bench_c2_200",
         "bench_c3": "r02_bench_c3", "bench_c3_100": "r02_bench_c3_100", "bench_c3_imex": "r02_bench_c3_imex",
         "bench_c5": "r02_bench_c5", "bench_c5_50": "r02_bench_c5_50", "bench_c5_k10": "r02_bench_c5_k10",
         "bench_ref_c3": "r02_bench_ref_c3", "c4": "r02_c4_kernels"}
PLAIN = {"pytest_gpu.log": "r02_pytest_gpu.log", "smoke.log": "r02_smoke.log",
         "fullsize_parity.json": "r02_fullsize_parity.json", "parity_per_field.json": "r02_parity_per_field.json",
         "launches.md": "r02_launches.md", "ncu_full.md": "r02_ncu_full.md", "ncu_opcodes.txt": "r02_ncu_opcodes.txt"}
for src, dst in BENCH.items():
    path = os.path.join(SRC, src + ".log")
    if not os.path.exists(path):
        continue
    lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
    if not lines:
        print("no JSON line in", path)
        continue
    json.loads(lines[-1])
    with open(os.path.join(P, dst + ".json"), "w") as f:
        f.write(lines[-1] + "\n")
    print(dst)
for src, dst in PLAIN.items():
    path = os.path.join(SRC, src)
    if os.path.exists(path) and os.path.getsize(path) > 0:
        shutil.copy(path, os.path.join(P, dst))
        print(dst)
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "results_table.py")], check=False)

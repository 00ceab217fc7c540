#!/usr/bin/env python
"""Fill BASELINE.md §5 ("Measured results") from the committed evidence under
profiles/: the bench lines (profiles/r02_bench_<cfg>.json), the ncu DRAM
traffic of the dominant kernel (profiles/traffic.json, C3), the full-size
golden parity results (profiles/r02_fullsize_parity.json) and the per-field
parity metric of the reduced-size tests (profiles/r02_parity_per_field.json).

    python tools/results_table.py            # rewrites the table in BASELINE.md
"""
import json
import os
import re
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def load(name):
    try:
        with open(os.path.join(P, name)) as f:
            txt = f.read().strip()
        return json.loads(txt.splitlines()[-1]) if txt.startswith("{") and "\n{" in txt else json.loads(txt)
    except (OSError, ValueError):
        return None


def row(cfg, label, bench, parity, traffic):
    if not bench:
        return f"| {label} | 1 | — | — | — | — | — | — | — |"
    Ks = bench["config"].get("schwarz_iters_per_step", [])
    sr = bench["config"].get("step_roofline", {})
    cpu = bench.get("cpu_baseline") or {}
    rf = bench.get("roofline") or {}
    tr = "—"
    if traffic and rf.get("bytes_per_launch") and cfg == "C3":     # the ncu capture is of C3
        t = traffic.get("bytes_per_launch", {}).get(rf.get("kernel"))
        if t:
            tr = f"{t / rf['bytes_per_launch']:.2f} ({rf['kernel']})"
    par = "—"
    if parity:
        cases = {k: v for k, v in parity.items() if k.startswith(cfg + "_chi16")}
        if cases:
            first = [v for k, v in cases.items() if k.endswith("_step1")]
            last_k = max(cases, key=lambda k: int(k.rsplit("step", 1)[1]))
            par = (f"{max(v['worst_rel_err'] for v in first):.1e} / {cases[last_k]['worst_rel_err']:.1e} "
                   f"({last_k.rsplit('_', 1)[1]})") if first else "—"
    keq = ("yes (every golden step)" if parity and any(k.startswith(cfg + "_chi16") for k in parity)
           else "yes (reduced sizes)")
    return (f"| {label} | {bench['n_gpus']} | {statistics.mean(Ks):.1f} | {bench['value']:.3g} | "
            f"{100 * sr.get('frac_of_8TBs', 0):.1f} % ({100 * sr.get('frac_of_measured_hbm', 0):.1f} % of the measured {(bench.get('roofline') or {}).get('peak', 0):.0f} GB/s) | "
            f"{tr} | {('%.3g (%s)' % (cpu['value'], cpu['cores'])) if cpu else '—'} | {par} | {keq} |")


def main():
    traffic = load("traffic.json")
    parity = load("r02_fullsize_parity.json")
    lines = ["| Config | GPUs | K per step (mean) | cell-updates/s | % of M1 roofline @ 8 TB/s | ncu DRAM bytes / M1 "
             "(dominant kernel) | Oracle cell-updates/s (cores) | Parity max rel err (step 1 / last golden step) | "
             "Iteration counts equal? |",
             "|---|---|---|---|---|---|---|---|---|"]
    for cfg, tag, label in (("C1", "c1", "C1 16×16×48"), ("C2", "c2", "C2 48×64×192"),
                            ("C2", "c2_200", "C2, all 200 BASELINE steps"),
                            ("C3", "c3", "C3 96×128×384"), ("C3", "c3_100", "C3, all 100 BASELINE steps"),
                            ("C5", "c5", "C5 (N = 1: 2 × 64×192×576)"), ("C5", "c5_50", "C5, all 50 BASELINE steps"),
                            ("C5", "c5_k10", "C5, fixed K = 10 (P:L634)")):
        lines.append(row(cfg, label, load(f"r02_bench_{tag}.json"), parity, traffic))
    c4 = load("r02_c4_kernels.json")
    if c4:
        ax = c4["axes"]
        lines.append("| C4 256×384×1152 (kernel only, one sweep per axis) | 1 | n/a | r / θ / φ: "
                     + " / ".join(f"{ax[a]['ms']:.2f} ms ({ax[a]['GBps'] / 1e3:.2f} TB/s)" for a in ("r", "theta", "phi"))
                     + " | " + " / ".join(f"{100 * ax[a]['GBps'] / 8000:.0f} %" for a in ("r", "theta", "phi"))
                     + " of 24 B/elem | — | — | every line of every axis (`test_c4_line_solves_full_size`) | n/a |")
    table = "\n".join(lines)
    path = os.path.join(ROOT, "BASELINE.md")
    s = open(path).read()
    head = s[:s.index("## 5. Measured results")]
    body = ("## 5. Measured results\n\nWritten by `tools/results_table.py` from `profiles/` (round 2; χ = 16, "
            "DESIGN.md RD-E4).  Parity: the CUDA path against the oracle's full-size goldens (512 sampled nodes "
            "per field, RD-E3 metric); reduced sizes compare every element (`tests/test_gpu_parity.py`).  The "
            "oracle rate is the full-grid oracle's static part + one Schwarz iteration, extrapolated to the GPU "
            "steps' K (bench.py `cpu_baseline`).\n\n" + table + "\n")
    open(path, "w").write(head + body)
    print(table)


if __name__ == "__main__":
    main()

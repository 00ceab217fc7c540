#!/usr/bin/env python
"""Additive (RD26) vs multiplicative (Algorithm 1 as printed)
Schwarz, and the mass-flux correction on/off,
Schwarz on C3 with one patch per context (yy_create_pair on one GPU): device
time per step and Schwarz iterations per step."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402
from tools.slab_overhead import time_step  # noqa: E402


def main():
    cfg = W.config(sys.argv[1] if len(sys.argv) > 1 else "C3")
    wl = W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    out = {}
    for mode in ("additive", "multiplicative"):
        g = Shell.pair(*args, schwarz=mode)
        for sh in g:
            sh.load_workload(wl)
        ms, ks = time_step(g, cfg, steps=3)
        out[mode] = {"ms_per_step": ms, "schwarz_iters": ks, "cell_updates_per_s": 2 * cfg.cells / (ms / 1e3)}
        for sh in g:
            sh.close()
    # Algorithm 1 step 4 on the single context
    for eps in (None, 1e-6):
        sh = Shell(*args, flux_fix_eps=eps)
        sh.load_workload(wl)
        ms, ks = time_step([sh], cfg, steps=3)
        out["single" + ("+flux_fix" if eps else "")] = {"ms_per_step": ms, "schwarz_iters": ks,
                                                       "cell_updates_per_s": 2 * cfg.cells / (ms / 1e3)}
        sh.close()
    print(json.dumps({"workload": "C3", "layout": "yy_create_pair (one patch per context, one GPU)", "modes": out}))


if __name__ == "__main__":
    main()

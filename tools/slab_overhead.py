#!/usr/bin/env python
"""Device time of one C3 step on ONE GPU: the single context vs the radial-slab
layout of 2*nslab ranks emulated in one process (yy_create_slabs: every rank's
kernels run back to back on the one device, transfers are device copies).  The
ratio is the extra work of the distributed layout (halo rows, partitioned
r-solve, packed fringe), not a scaling measurement."""
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402


def time_step(shells, cfg, steps=2):
    st = torch.cuda.Stream()
    for sh in shells:
        sh.set_stream(st.cuda_stream)
    shells[0].step(1, cfg.tol)              # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    shells[0].step(steps, cfg.tol)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps, [k for k, _ in shells[0].stats()[-steps:]]


def main():
    cfg = W.config(sys.argv[1] if len(sys.argv) > 1 else "C3")
    wl = W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    out = {}
    one = Shell(*args)
    one.load_workload(wl)
    out["single"] = time_step([one], cfg)
    one.close()
    for S in (1, 2, 4):
        g = Shell.slabs(*args, nslab=S)
        for sh in g:
            sh.load_workload(wl)
        out[f"ranks{2 * S}"] = time_step(g, cfg)
        for sh in g:
            sh.close()
    print(json.dumps({"workload": cfg.name if hasattr(cfg, "name") else "C3", "ms_per_step_and_K": out}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Heat-only Douglas scheme (YY_HEAT_ONLY) on the C3 grid and
temperature data (u = 0): device time per step, Schwarz iterations, and the
fraction of the 8 TB/s roofline of its M1 bytes (T path: static 6 values per
step, residual + three sweeps 17 values per iteration)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402


def main(steps=3):
    cfg = W.config("C3")
    wl = W.make_workload(cfg)
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, 0.0, cfg.dt, heat_only=True)
    for p, pd in enumerate(wl["patches"]):
        sh.set_fields(p, 0, 0, T=pd["n"]["T"])
        sh.set_fields(p, 1, 0, T=pd["nm1"]["T"])
        sh.set_wall(p, [(t, {"T": d["T"]}) for t, d in pd["walls"] if "T" in d])
    st = torch.cuda.Stream()
    sh.set_stream(st.cuda_stream)
    sh.step(1, cfg.tol)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sh.step(steps, cfg.tol)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    Ks = [k for k, _ in sh.stats()[-steps:]]
    cells = 2 * cfg.cells
    model = sum(cells * 8 * (6 + 17 * k) for k in Ks) / steps
    print(json.dumps({"workload": "C3 grid, heat only (u = 0, Ra = 0), tol 1e-10", "ms_per_step": ms,
                      "schwarz_iters": Ks, "cell_updates_per_s": cells / (ms / 1e3),
                      "M1_bytes_per_step": model, "frac_of_8TBs": model / 8e12 / (ms / 1e3)}))


if __name__ == "__main__":
    main()

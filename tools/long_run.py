#!/usr/bin/env python
"""Run a BASELINE workload for its configured number of steps on the GPU and
print per-step Schwarz counts and max |u|, |p|, |T| (stability check).
    python tools/long_run.py C3 [steps] [chi]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402

name = sys.argv[1]
cfg = W.config(name)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.steps
chi = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi)
sh.load_workload(W.make_workload(cfg))
for s in range(steps):
    sh.step(1, cfg.tol)
    if s % 10 == 9 or s == steps - 1:
        f = sh.get_fields(0, 0, 2)
        print("step %4d t=%.5f K=%3d  max|u_r|=%.3e max|u_th|=%.3e max|p|=%.4e max|T|=%.4f"
              % (s + 1, sh.time(), sh.stats()[-1][0], np.abs(f["ur"]).max(), np.abs(f["ut"]).max(),
                 np.abs(f["p"]).max(), np.abs(f["T"]).max()), flush=True)

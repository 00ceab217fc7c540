#!/usr/bin/env python
"""Schwarz counts and ms/step of a BASELINE workload on the GPU at several chi
(DESIGN.md RD-E4).   python tools/chi_k.py C3 5 1,10,16"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402

name, steps = sys.argv[1], int(sys.argv[2])
for chi in (float(x) for x in sys.argv[3].split(",")):
    cfg = W.config(name)
    st = torch.cuda.Stream()
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi, stream=st.cuda_stream)
    sh.load_workload(W.make_workload(cfg))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh.step(steps, cfg.tol)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    print(json.dumps({"workload": name, "chi": chi, "K": [k for k, _ in sh.stats()], "ms_per_step": ms}), flush=True)
    sh.close()

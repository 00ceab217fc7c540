#!/usr/bin/env python
"""BASELINE C5 weak-scaling layout at G GPUs, checked at FULL size on ONE GPU:
the 2*nslab radial-slab contexts of the G-rank layout (yy_create_slabs: the
yy_create_dist data path with device copies instead of NCCL) against a single
two-patch context on the same grid (patch Nr = 64 G).  The slab r-solve changes
only the rounding order, so: equal Schwarz counts every step and fields equal to
rounding.  Also times one step of each (the emulation runs every rank's kernels
back to back on the one GPU — a correctness check, not a scaling number).

    python tools/c5_layout_check.py [G=8] [steps=2]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402


def main(G=8, steps=2):
    cfg = W.config("C5", G=G)
    wl = W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    out = {"config": "C5", "G": G, "grid_per_patch": [cfg.nr, cfg.nth, cfg.nph], "steps": steps}
    res = {}
    for layout in ("single", "slabs"):
        st = torch.cuda.Stream()
        grp = [Shell(*args, stream=st.cuda_stream)] if layout == "single" else \
            Shell.slabs(*args, nslab=G // 2, stream=st.cuda_stream)
        for sh in grp:
            sh.load_workload(wl)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        grp[0].step(steps, cfg.tol)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        ks = [k for k, _ in grp[0].stats()[-steps:]]
        fields = []
        for p in range(2):
            for s in (1, 2):
                f = {n: np.zeros(grp[0].shape(n)) for n in ("ur", "ut", "up", "p", "T")}
                for sh in grp:
                    if p in sh.patches:
                        sh.get_fields(p, 0, s, out=f)
                fields.append(f)
        res[layout] = (ks, fields)
        out[layout] = {"schwarz_iters": ks, "s_per_step": dt}
        for sh in grp:
            sh.close()
        del grp
        torch.cuda.synchronize()
    worst = 0.0
    for fa, fb in zip(res["single"][1], res["slabs"][1]):
        vmax = max(np.max(np.abs(fa[q])) for q in ("ur", "ut", "up"))
        for k in fa:
            den = vmax if k in ("ur", "ut", "up") else max(np.max(np.abs(fa[k])), 1e-300)
            worst = max(worst, float(np.max(np.abs(fa[k] - fb[k])) / den))
    out["max_rel_diff"] = worst
    out["equal_iteration_counts"] = res["single"][0] == res["slabs"][0]
    print(json.dumps(out))
    return 0 if out["equal_iteration_counts"] and worst <= 1e-11 else 1


if __name__ == "__main__":
    sys.exit(main(*(int(x) for x in sys.argv[1:])))

#!/usr/bin/env python
"""C2 (Landau jet) for its BASELINE length on the GPU: per step the
Schwarz count K and the distance of the solution from the exact steady jet
(the initial field), max-norm and omega-weighted l2 over solved nodes of both
patches, for u (system 2 = the answer) and for p modulo its mean.

    python tools/c2_drift.py [steps=200] [chi=1] [every=5] [out.json]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402


def weights(cfg, kind):
    r, th, _ = W.node_axes(cfg, kind)
    dr = (cfg.R2 - cfg.R1) / cfg.nr
    (_, dth, _), (_, dph, _) = W.axes(cfg)[1:]
    return (r[:, None, None] ** 2 * np.sin(th)[None, :, None] * dr * dth * dph)


def solved(a, kind):
    i0, i1 = (1, a.shape[0] - 1) if kind == "R" else (0, a.shape[0])
    return a[i0:i1, 1:-1, 1:-1]


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    chi = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    every = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    out = sys.argv[4] if len(sys.argv) > 4 else None
    cfg = W.config("C2")
    wl = W.make_workload(cfg)
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi)
    sh.load_workload(wl)
    ex = [wl["patches"][p]["n"] for p in range(2)]
    kinds = {"ur": "R", "ut": "TH", "up": "PH", "p": "C"}
    wts = {k: weights(cfg, kd) for k, kd in kinds.items()}
    umax = max(np.abs(solved(ex[p][q], kinds[q])).max() for p in range(2) for q in ("ur", "ut", "up"))
    rows = []
    for s in range(1, steps + 1):
        sh.step(1, cfg.tol)
        if s % every and s != steps:
            continue
        f = [sh.get_fields(p, 0, 2) for p in range(2)]
        eu_max, eu2, ep_max, ep2 = 0.0, 0.0, 0.0, 0.0
        for p in range(2):
            for q in ("ur", "ut", "up"):
                d = solved(f[p][q] - ex[p][q], kinds[q])
                eu_max = max(eu_max, float(np.abs(d).max()))
                eu2 += float(np.sum(solved(np.broadcast_to(wts[q], f[p][q].shape), kinds[q]) * d * d))
        pw = solved(np.broadcast_to(wts["p"], f[0]["p"].shape), "C")
        dp = [solved(f[p]["p"] - ex[p]["p2"], "C") for p in range(2)]
        mean = sum(float(np.sum(pw * d)) for d in dp) / (2 * float(np.sum(pw)))
        for d in dp:
            ep_max = max(ep_max, float(np.abs(d - mean).max()))
            ep2 += float(np.sum(pw * (d - mean) ** 2))
        K = sh.stats()[-1][0]
        row = {"step": s, "t": sh.time(), "K": K, "K_window": [k for k, _ in sh.stats()[-every:]],
               "u_err_max_rel": eu_max / umax, "u_err_l2": eu2 ** 0.5, "p_err_max": ep_max, "p_err_l2": ep2 ** 0.5,
               "p_mean_drift": mean}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump({"config": "C2 48x64x192 per patch, Landau jet, dt 5e-4, tol 1e-10", "chi": chi,
                       "steps": steps, "all_K": [k for k, _ in sh.stats()], "rows": rows}, fh, indent=1)
    sh.close()


if __name__ == "__main__":
    main()

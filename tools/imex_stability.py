#!/usr/bin/env python
"""Stability of the two places of the linearised advection: inside
the direction-wise factors (the paper's scheme, YY_ADVECTION = 0) versus IMEX
(explicit transport terms, YY_ADVECTION = 1).  The paper: "our
numerical experience demonstrated that the second approach [advection in the
split operator] yields an algorithm that has better stability performance".

On the GPU: eq:Exact scaled by amp (advection ~ amp), 16 x 32 x 96 per
patch, Pr = 1, Ra = 1, chi = 16, for a ladder of time steps, up to t = 1 (at
most 400 steps).  A run is stable when it finishes with finite fields, the
Schwarz iteration converges every step (K < K_max = 200) and the error against
the exact solution stays below the solution's own size.

    python tools/imex_stability.py [out.json]
"""
import json
import math
import os
import sys

import numpy as np

KMAX = 200

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402
from paper_1905_02300_b200.yy import YYError  # noqa: E402


def run(amp, dt, advection, grid=(16, 32, 96), tend=1.0, maxsteps=400):
    cfg = W.small("C1", *grid, Ra=1.0, dt=dt, extra={"amp": amp})
    wl = W.make_workload(cfg)
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=16.0, max_iters=KMAX,
               advection=advection)
    sh.load_workload(wl)
    ex0 = [wl["patches"][p]["n"] for p in range(2)]
    umax = max(np.abs(ex0[p][q]).max() for p in range(2) for q in ("ur", "ut", "up"))
    nsteps = min(maxsteps, int(round(tend / dt)))
    status, worst, Ks = "stable", 0.0, []
    try:
        for s in range(1, nsteps + 1):
            st = sh.step(1, cfg.tol)
            Ks.append(sh.stats()[-1][0])
            if st == 4:
                status = "no Schwarz convergence"
                break
            if s % 10 == 0 or s == nsteps:
                c = math.cos(sh.time())
                err = 0.0
                for p in range(2):
                    f = sh.get_fields(p, 0, 2)
                    for q in ("ur", "ut", "up"):
                        d = f[q][1:-1, 1:-1, 1:-1] - c * ex0[p][q][1:-1, 1:-1, 1:-1]
                        err = max(err, float(np.abs(d).max()))
                worst = max(worst, err / umax)
                if not np.isfinite(err) or err > umax:
                    status = "blow-up"
                    break
    except YYError as e:
        status = f"error: {e}"
    sh.close()
    return {"amp": amp, "dt": dt, "advection": advection, "steps": len(Ks), "status": status,
            "max_err_rel": worst, "K_max": max(Ks) if Ks else None, "K_last": Ks[-1] if Ks else None}


AMPS = (1.0, 8.0, 16.0, 32.0)
DTS = (5e-4, 1e-3, 1.5e-3, 2e-3, 3e-3, 4e-3, 6e-3)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    rows = []
    for amp in AMPS:
        for adv in ("split", "imex"):
            for dt in DTS:
                r = run(amp, dt, adv)
                rows.append(r)
                print(json.dumps(r), flush=True)
    summary = {}
    for amp in AMPS:
        for adv in ("split", "imex"):
            ok = [r["dt"] for r in rows if r["amp"] == amp and r["advection"] == adv and r["status"] == "stable"]
            summary[f"amp={amp:g} {adv}"] = max(ok) if ok else None
    print(json.dumps({"largest_stable_dt": summary}), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump({"what": __doc__.splitlines()[0], "rows": rows, "largest_stable_dt": summary}, fh, indent=1)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Write tests/golden/<cfg>_step1.json: the CPU oracle's first full time step
of a BASELINE.json workload at FULL size — Schwarz iteration count, final rho,
and the values of every field (both patches, both systems, level n after the
step) at seeded sample nodes.  Calls only oracle/ and workloads/ (the stored
values never come from the CUDA path).

    python tools/make_golden.py C3 [C2 C5 ...]          first step -> <cfg>_step1.json
    python tools/make_golden.py --steps 3 C3           three steps -> <cfg>_step3.json
"""
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle.scheme import Oracle  # noqa: E402

NSAMPLE = 512


def sample_index(shape, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return [tuple(int(rng.integers(0, s)) for s in shape) for _ in range(NSAMPLE)]


def main(name, steps=1):
    cfg = W.config(name)
    t0 = time.time()
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    o.load_workload(W.make_workload(cfg))
    o.step(steps, cfg.tol)
    k, rho = o.stats[-1]
    out = {"config": name, "grid": [cfg.nr, cfg.nth, cfg.nph], "dt": cfg.dt, "tol": cfg.tol, "steps": steps,
           "schwarz_iters": int(k), "schwarz_iters_per_step": [int(x[0]) for x in o.stats],
           "rho": float(rho), "seconds": time.time() - t0,
           "oracle_commit": subprocess.run(["git", "rev-parse", "HEAD"], cwd=ROOT, capture_output=True,
                                           text=True).stdout.strip(),
           "samples": {}}
    for p in range(2):
        for s in (1, 2):
            f = o.get_fields(p, 0, s)
            for q, arr in f.items():
                idx = sample_index(arr.shape, 1000 * p + 100 * s + "ur ut up p T".split().index(q))
                out["samples"][f"{p}/{s}/{q}"] = {"index": idx, "value": [float(arr[i]) for i in idx],
                                                  "absmax": float(np.max(np.abs(arr)))}
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_step{steps}.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print(name, "K", k, "rho", rho, "%.0f s" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    nsteps = 1
    if args[:1] == ["--steps"]:
        nsteps, args = int(args[1]), args[2:]
    for n in args:
        main(n, nsteps)

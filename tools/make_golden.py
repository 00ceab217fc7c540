#!/usr/bin/env python
"""Write tests/golden/<cfg>_step1.json: the CPU oracle's first full time step
of a BASELINE.json workload at FULL size — Schwarz iteration count, final rho,
and the values of every field (both patches, both systems, level n after the
step) at seeded sample nodes.  Calls only oracle/ and workloads/ (the stored
values never come from the CUDA path).

    python tools/make_golden.py C3 [C2 C5 ...]
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


def main(name):
    cfg = W.config(name)
    t0 = time.time()
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    o.load_workload(W.make_workload(cfg))
    o.step(1, cfg.tol)
    k, rho = o.stats[-1]
    out = {"config": name, "grid": [cfg.nr, cfg.nth, cfg.nph], "dt": cfg.dt, "tol": cfg.tol,
           "schwarz_iters": int(k), "rho": float(rho), "seconds": time.time() - t0,
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
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_step1.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print(name, "K", k, "rho", rho, "%.0f s" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        main(n)

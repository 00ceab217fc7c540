#!/usr/bin/env python
"""Write tests/golden/<cfg>_step1.json: the CPU oracle's first full time step
of a BASELINE.json workload at FULL size — Schwarz iteration count, final rho,
and the values of every field (both patches, both systems, level n after the
step) at seeded sample nodes.  Calls only oracle/ and workloads/ (the stored
values never come from the CUDA path).

    python tools/make_golden.py C3 [C2 C5 ...]            first step -> <cfg>_chi16_step1.json
    python tools/make_golden.py --steps 1,3,10 C3        a golden after steps 1, 3 and 10
    python tools/make_golden.py --chi 1 --steps 3 C3     round-1 chi = 1 files <cfg>_step3.json
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


def write(o, name, cfg, chi, t0, tag):
    k, rho = o.stats[-1]
    steps = len(o.stats)
    out = {"config": name, "grid": [cfg.nr, cfg.nth, cfg.nph], "dt": cfg.dt, "tol": cfg.tol, "steps": steps,
           "chi": chi, "schwarz_iters": int(k), "schwarz_iters_per_step": [int(x[0]) for x in o.stats],
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
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}{tag}_step{steps}.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print(name, "chi", chi, "steps", steps, "K", [int(x[0]) for x in o.stats][-5:], "rho", rho,
          "%.0f s" % (time.time() - t0), "->", os.path.basename(path), flush=True)


def main(name, checkpoints, chi=None):
    """Run the workload to the last checkpoint, writing a golden at each one.
    chi None: the workload's own chi (cfg.chi, file <cfg>_chi<chi>_step<k>.json);
    chi 1: the round-1 files <cfg>_step<k>.json."""
    cfg = W.config(name)
    chi = cfg.chi if chi is None else chi
    tag = "" if chi == 1.0 else f"_chi{chi:g}"
    t0 = time.time()
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi)
    o.load_workload(W.make_workload(cfg))
    done = 0
    for c in sorted(checkpoints):
        o.step(c - done, cfg.tol)
        done = c
        write(o, name, cfg, chi, t0, tag)


if __name__ == "__main__":
    args = sys.argv[1:]
    cps, chi = [1], None
    while args and args[0].startswith("--"):
        if args[0] == "--steps":
            cps, args = [int(x) for x in args[1].split(",")], args[2:]
        elif args[0] == "--chi":
            chi, args = float(args[1]), args[2:]
        else:
            raise SystemExit(f"unknown option {args[0]}")
    for n in args:
        main(n, cps, chi)

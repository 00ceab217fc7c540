#!/usr/bin/env python
"""Richardson self-convergence in time of the oracle step on eq:Exact
(P:L548-564), one process per time step size.

    python tools/time_order_study.py --tf 0.5 --dts 0.02,0.01,0.005,0.0025 \
        --grid 4,12,28 --chi 10 [--amp 1] [--R1 1 --R2 2] [--tol 1e-10]

Prints, per system and field, the omega-weighted l2 norm of the difference of
consecutive dt levels at T_f and the observed orders log2(e_i / e_{i+1}).
Run from the repo root (it puts the root on sys.path itself)."""
from __future__ import annotations

import argparse
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

KIND = {"ur": "R", "ut": "TH", "up": "PH", "T": "C", "p": "C", "p~": "C"}


def run_level(args):
    dt, tf, grid, amp, chi, R1, R2, tol, variant, flux = args
    import workloads as W
    from oracle.scheme import Oracle
    cfg = W.small("C1", *grid, Ra=1.0, dt=dt, extra={"amp": amp}, R1=R1, R2=R2)
    kw = {}
    if variant:
        kw["advection"] = variant          # "split" (the paper's scheme) or "imex"
    if flux:
        kw["flux_fix_eps"] = flux
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi, **kw)
    o.load_workload(W.make_workload(cfg))
    t0 = time.time()
    o.step(int(round(tf / dt)), tol * amp)
    fields = {s: [o.get_fields(p, 0, s) for p in range(2)] for s in (1, 2)}
    return dt, time.time() - t0, [st[0] for st in o.stats], fields


def orders(levels, grid, R1, R2):
    """errs[sys][field] = list of ||f(dt_i) - f(dt_{i+1})||_omega."""
    import workloads as W
    from oracle.grid import Grid
    g = Grid(*grid, R1, R2)
    out = {}
    for s in (1, 2):
        for f, kind in KIND.items():
            nr, nt, npp = g.shape(kind)
            i0, i1 = (1, nr - 1) if kind == "R" else (0, nr)
            blk = (slice(i0, i1), slice(1, nt - 1), slice(1, npp - 1))
            w = g.weights_omega(kind)[blk]
            errs = []
            def val(lev, p):
                if f != "p~":
                    return lev[3][s][p][f][blk]
                # pressure modulo its omega-weighted mean over both patches (the
                # AC pressure is defined up to a constant)
                m = sum(float(np.sum(w * lev[3][s][q]["p"][blk])) for q in range(2)) / (2 * float(np.sum(w)))
                return lev[3][s][p]["p"][blk] - m
            for a in range(len(levels) - 1):
                e2 = 0.0
                for p in range(2):
                    d = val(levels[a], p) - val(levels[a + 1], p)
                    e2 += float(np.sum(w * d * d))
                errs.append(math.sqrt(e2))
            out[(s, f)] = errs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tf", type=float, default=0.5)
    ap.add_argument("--dts", default="0.02,0.01,0.005,0.0025")
    ap.add_argument("--grid", default="4,12,28")
    ap.add_argument("--amp", type=float, default=1.0)
    ap.add_argument("--chi", type=float, default=10.0)
    ap.add_argument("--R1", type=float, default=1.0)
    ap.add_argument("--R2", type=float, default=2.0)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--variant", default="", help="advection: split (default) | imex")
    ap.add_argument("--flux", type=float, default=0.0, help="mass-flux correction eps (Alg. 1 step 4); 0 = off")
    a = ap.parse_args()
    dts = [float(x) for x in a.dts.split(",")]
    grid = tuple(int(x) for x in a.grid.split(","))
    jobs = [(dt, a.tf, grid, a.amp, a.chi, a.R1, a.R2, a.tol, a.variant, a.flux) for dt in dts]
    with ProcessPoolExecutor(max_workers=len(jobs)) as ex:
        levels = list(ex.map(run_level, jobs))
    for dt, sec, its, _ in levels:
        print(f"dt {dt:g}: {sec:.1f} s, iterations {its[:4]} ... {its[-2:]}", flush=True)
    errs = orders(levels, grid, a.R1, a.R2)
    print(f"chi {a.chi} tf {a.tf} grid {grid} R {a.R1},{a.R2} amp {a.amp} flux {a.flux} variant {a.variant!r}")
    for (s, f), e in errs.items():
        sl = [round(math.log2(e[i] / e[i + 1]), 2) for i in range(len(e) - 1)]
        print(f"system {s} {f:2s} diffs {['%.2e' % x for x in e]} orders {sl}", flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — full Yin-Yang AC direction-splitting time steps on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl yy|reference] [--workload C3]

One "step" = one full time step of the paper's method (SURVEY.md §8(a) rows
a1-a9: static RHS, additive Schwarz iterated to tol with splitting-error
reduction, pressure updates) on both Yin-Yang patches of the workload.
Prints ONE JSON line (rank 0).  Metric: cell-updates/s = 2 patches x cells
per patch x steps / device time (BASELINE.json metric); inputs larger than L2
(the C3 working set is ~2.8 GB), so no flush is needed between steps.

--impl reference runs the CPU oracle (oracle/, plain numpy fp64) on the same
workload at full size, bounded: the static part of one step and a few Schwarz
iterations, each timed, extrapolated to the oracle's own Schwarz count.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full time steps: cell-updates/s and % of HBM roofline at 1/2/4/8 B200"
UNIT = "cell-updates/s"
HBM_NOMINAL_GBS = 8000.0          # BASELINE.json roofline denominator (8 TB/s)


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------------
# algorithmic bytes (SURVEY.md §8(d) model M1: each pass reads each input array
# once and writes each output once, 8 B per value; halos and 1-D tables free)
# ---------------------------------------------------------------------------------
def kind_nodes(cfg, kind):
    nr, nt, npp = cfg.nr, cfg.nth, cfg.nph
    return {"C": nr * nt * npp, "R": (nr + 1) * nt * npp, "TH": nr * (nt + 1) * npp,
            "PH": nr * nt * (npp + 1)}[kind]


QK = {"T": "C", "ur": "R", "ut": "TH", "up": "PH"}


def m1_bytes(name, cfg, nsrc):
    """Algorithmic bytes of ONE launch of kernel class `name` (both patches)."""
    P = 2
    if "+resid_" in name:
        # fused first sweep: the residual's reads + the sweep's own a* reads + one
        # write (the R round trip of the unfused pair is not moved)
        sw, rs = name.split("+")
        return m1_bytes(rs, cfg, nsrc) + m1_bytes(sw, cfg, nsrc) - 8 * P * kind_nodes(cfg, QK[sw.split("_")[1]]) * 2
    if name.startswith("sweep_"):
        _, q, ax = name.split("_")[:3]
        fin = name.endswith("_fin")
        extra = 0
        if q == "ut" and ax == "th":
            extra = 1          # reaction -(a_r/r) u reads a*_r
        if q == "up" and ax == "ph":
            extra = 2          # reaction reads a*_r, a*_th
        arrays = 1 + 1 + extra + 1 + (1 if fin else 0)   # rhs, a*_ax, extras, write, (+psi read)
        return 8 * P * kind_nodes(cfg, QK[q]) * arrays
    if name.startswith("resid_"):
        q = name[6:8] if name[6:8] in ("ur", "ut", "up") else "T"
        s = name[-1]
        ins = {"T": 0, "ur": 2, "ut": 2, "up": 4}[q] + (2 if (q != "T" and s == "2") else 0)
        return 8 * P * kind_nodes(cfg, QK[q]) * (6 + ins + 1)
    if name.startswith("static_"):
        q = name[7:]
        reads = {"T": 5, "ur": 17, "ut": 13, "up": 9}[q] + nsrc
        writes = 1 if q == "T" else 2
        return 8 * P * kind_nodes(cfg, QK[q]) * (reads + writes)
    if name.startswith("pres_"):
        return 8 * P * kind_nodes(cfg, "C") * (8 + (2 if name.endswith("2") else 0) + 1)
    if name == "astar":      # one launch: the three components of a* = 1.5 u2^n - 0.5 u2^{n-1}
        return 8 * P * 3 * sum(kind_nodes(cfg, k) for k in ("R", "TH", "PH"))
    return 0


def traffic_of(name, workload):
    """DRAM bytes per launch of a kernel class from the committed ncu capture
    (profiles/traffic.json), or None."""
    if workload != "C3":
        return None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f)["bytes_per_launch"].get(name)
    except (OSError, ValueError, KeyError):
        return None


def step_model_bytes(cfg, K, forced):
    """M1 bytes of one full step with K Schwarz iterations."""
    per_cell = (352 if forced else 256) + 1320 * K
    return 2 * cfg.cells * per_cell


# ---------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------
def oracle_full_grid(cfg_name, n_iters):
    """The plain numpy oracle on the workload's FULL grid: the static part of one
    time step (a*, G) and its first n_iters Schwarz iterations, each timed (the
    oracle's own timing hooks).  A full step costs t_static + K t_iter, so the
    rate at any Schwarz count K follows without running all K iterations.
    Returns (cells, t_static, [t_iter ...])."""
    import workloads as W
    from oracle.scheme import Oracle
    c = W.config(cfg_name)
    o = Oracle(c.nr, c.nth, c.nph, c.R1, c.R2, c.Pr, c.Ra, c.dt, chi=c.chi, fixed_iters=n_iters)
    o.load_workload(W.make_workload(c))
    o.step(1, c.tol)
    return 2 * c.cells, o.timing["static"], list(o.timing["iters"])


def oracle_reference_K(cfg_name):
    """The oracle's own Schwarz count for the first step of the workload at full
    size, from the committed golden (tools/make_golden.py, oracle only), or None."""
    import workloads as W
    chi = W.config(cfg_name).chi
    tag = "" if chi == 1.0 else f"_chi{chi:g}"
    try:
        with open(os.path.join(ROOT, "tests", "golden", f"{cfg_name.lower()}{tag}_step1.json")) as f:
            return int(json.load(f)["schwarz_iters"])
    except (OSError, ValueError, KeyError):
        return None


def cpu_cores_used():
    return 1   # numpy elementwise kernels run single-threaded (no BLAS in the oracle step)


# ---------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: launch the N ranks ourselves, exactly
    as the driver's `python -m torch.distributed.run --nnodes=1 --nproc-per-node N
    --master-addr 127.0.0.1` would, after checking that N devices exist (fails
    loudly otherwise: a silent one-GPU run would mislabel the result)."""
    if not args.launch_check:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_launch_check(args):
    """Rank plumbing only (no GPU): every rank joins a gloo group, the ranks agree
    on the world size and the max-over-ranks reduction the timed path uses."""
    import torch
    import torch.distributed as td
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    td.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    td.all_reduce(t, op=td.ReduceOp.MAX)
    ranks = [None] * world
    td.all_gather_object(ranks, rank)
    if rank == 0:
        emit({"launch_check": True, "world": world, "n_gpus": args.gpus, "ranks": ranks, "max_over_ranks": float(t)})
    td.destroy_process_group()
    return 0


def emit(obj):
    print(json.dumps(obj), flush=True)


def run_reference(args):
    """The reference arm: the CPU oracle as it stands on the workload's full grid.
    One bench step = one Schwarz iteration of the full-grid step (the static part
    is timed once before); the line's value is the full-step rate at the oracle's
    own Schwarz count K (golden of the first step), cells / (t_static + K t_iter)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cells, t_static, iters = oracle_full_grid(args.workload, args.warmup + args.steps)
    timed = iters[args.warmup:]
    t_iter = sum(timed) / len(timed)
    K = oracle_reference_K(args.workload) or len(iters)
    t_step = t_static + K * t_iter
    v = cells / t_step
    sample = (f"{args.workload} at full size (2 x {cells // 2} cells): the static part of the first time step "
              f"({t_static:.1f} s) and {args.warmup} untimed + {args.steps} timed Schwarz iterations "
              f"({t_iter:.1f} s each), extrapolated to the oracle's own K = {K} of that step")
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": max(world, args.gpus),
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_step,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic", "config": {"workload": args.workload, "sample": sample, "schwarz_iters": K},
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle", "sample": sample},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    return 0


def run_yy(args):
    import numpy as np
    import torch

    import workloads as W
    from paper_1905_02300_b200 import Shell

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus} (launch with torchrun, or "
                         "without WORLD_SIZE to let bench.py start the ranks)")
    if world > 1:
        return run_yy_dist(args, rank, world, local)
    torch.cuda.set_device(local)
    cfg = W.config(args.workload)
    wl = W.make_workload(cfg)
    nsrc = len(wl["patches"][0]["sources"])
    forced = nsrc > 0
    stream = torch.cuda.Stream()
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, stream=stream.cuda_stream,
               chi=cfg.chi, advection=args.advection, **({"fixed_iters": args.fixed_iters} if args.fixed_iters else {}))
    sh.load_workload(wl)
    W_ = max(3, args.warmup)
    for _ in range(W_):
        sh.step(1, cfg.tol)
    torch.cuda.synchronize()
    l0 = sh.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    ev0.record(stream)
    sh.step(args.steps, cfg.tol)                   # the timed region: no per-kernel events in it
    ev1.record(stream)
    ev1.synchronize()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    launches = sh.launch_count() - l0
    stats = sh.stats()[-args.steps:]
    Ks = [k for k, _ in stats]
    # per-kernel-class pass: the next K steps with CUDA events around every kernel
    # class on the launch stream (kept out of the timed region, which they perturb)
    sh.profile(True)
    sh.step(args.steps, cfg.tol)
    torch.cuda.synchronize()
    prof = sh.profile_report()
    sh.profile(False)
    Ks_prof = [k for k, _ in sh.stats()[-args.steps:]]
    cells = 2 * cfg.cells
    value = cells * args.steps / (ms / 1e3)
    peak, peak_kind = measured_peak()
    # dominant kernel class
    dom = max(prof.items(), key=lambda kv: kv[1][1])
    dname, (dcount, dms) = dom
    dbytes = m1_bytes(dname, cfg, nsrc)
    davg_s = dms / dcount / 1e3
    achieved = dbytes / davg_s / 1e9 if dbytes else None
    share = dms / sum(t for _, t in prof.values())
    # whole-step model roofline
    model_bytes = sum(step_model_bytes(cfg, k, forced) for k in Ks)
    t_roof_8 = model_bytes / (HBM_NOMINAL_GBS * 1e9)
    t_roof_m = model_bytes / (peak * 1e9)

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = a
            return t.numpy()
        host = []
        h2d = 0
        for pd in wl["patches"]:
            n, m = pd["n"], pd["nm1"]
            d = {"n1": {k: pinned(n[k]) for k in ("ur", "ut", "up", "T")},
                 "p1": pinned(n["p1"]), "p2": pinned(n["p2"]),
                 "m": {k: pinned(m[k]) for k in ("ur", "ut", "up", "T")}}
            u_b = sum(d["n1"][k].nbytes for k in ("ur", "ut", "up"))
            # host -> device bytes of the yy_set_fields calls: level 0 system 0 (u, T, p1
            # once; system 2's copies are device-to-device), level 0 system 2 (p2),
            # level 1 system 0 (u, T once)
            h2d += u_b + d["n1"]["T"].nbytes + d["p1"].nbytes
            h2d += d["p2"].nbytes
            h2d += u_b + d["m"]["T"].nbytes
            host.append(d)
        outs = [{k: pinned(np.zeros(sh.shape(k))) for k in ("ur", "ut", "up", "p", "T")} for _ in range(2)]
        d2h = sum(v.nbytes for o in outs for v in o.values())
        from paper_1905_02300_b200.yy import _ptr, yy_fields
        import ctypes

        def upload_step_download():
            for p, d in enumerate(host):
                sh.set_fields(p, 0, 0, ur=d["n1"]["ur"], ut=d["n1"]["ut"], up=d["n1"]["up"], T=d["n1"]["T"], p=d["p1"])
                sh.set_fields(p, 0, 2, p=d["p2"])
                sh.set_fields(p, 1, 0, **d["m"])
            sh.step(1, cfg.tol)
            for p in range(2):
                f = yy_fields()
                for k, a in outs[p].items():
                    setattr(f, k, _ptr(a))
                sh._check(sh.L.yy_get_fields(sh.h, p, 0, 2, ctypes.byref(f)), "yy_get_fields")
        upload_step_download()          # warm
        ne = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ne):
            upload_step_download()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / ne
        e2e = {"value": cells / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s,
               "schwarz_iters": sh.stats()[-1][0], "timing": "host perf_counter, device synchronised"}

    cpu = None
    if not args.no_cpu_baseline:
        c_cells, t_static, t_iters = oracle_full_grid(args.workload, 1)
        K_mean = sum(Ks) / len(Ks)
        c_sec = t_static + K_mean * t_iters[0]
        cpu = {"value": c_cells / c_sec, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
               "sample": f"{args.workload} at full size: the static part ({t_static:.1f} s) and the first "
                         f"Schwarz iteration ({t_iters[0]:.1f} s) of one full-grid time step by the plain numpy "
                         f"oracle, extrapolated to the GPU steps' mean K = {K_mean:.1f}",
               "per_schwarz_iteration": {"value": c_cells / t_iters[0], "unit": "cell-iterations/s"}}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": W_,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "grid_per_patch": [cfg.nr, cfg.nth, cfg.nph], "patches": 2,
                   "dt": cfg.dt, "Pr": cfg.Pr, "Ra": cfg.Ra, "chi": cfg.chi, "advection": args.advection,
                   "schwarz_tol": cfg.tol if not args.fixed_iters else f"fixed K = {args.fixed_iters}",
                   "schwarz_iters_per_step": Ks, "l2_flush": "inputs larger than L2 (working set ~37 fp64 fields)",
                   "step_roofline": {"model": "SURVEY M1 bytes/cell = %d + 1320 K" % (352 if forced else 256),
                                     "model_bytes": model_bytes,
                                     "frac_of_8TBs": t_roof_8 / (ms / 1e3),
                                     "frac_of_measured_hbm": t_roof_m / (ms / 1e3)}},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic_of(dname, args.workload),
                     "traffic_source": "profiles/traffic.json (ncu --set full capture of this kernel class, C3)",
                     "peak_source": peak_kind, "bytes_per_launch": dbytes, "avg_launch_ms": davg_s * 1e3,
                     "launches": dcount, "share_of_step": share},
        "kernel_timing": {"how": "separate pass of the next %d steps (Schwarz K %s) with CUDA events around "
                                 "every kernel class on the launch stream" % (args.steps, Ks_prof)},
        "kernel_classes": {k: {"launches": n, "ms": t, "GBps": (m1_bytes(k, cfg, nsrc) * n / (t / 1e3) / 1e9)
                               if t > 0 and m1_bytes(k, cfg, nsrc) else None}
                           for k, (n, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    emit(out)
    sh.close()
    return 0


def run_yy_dist(args, rank, world, local):
    """N = 2 nslab GPUs (yy_create_dist over NCCL): rank = patch * nslab + slab,
    radial slabs of nr / nslab rows.  C1-C3: the workload is the N = 1 one, so the
    total work is fixed ("scaling": "strong"); C5 (BASELINE's weak-scaling config):
    patch Nr = 64 N, a fixed 128x192x576 shard per GPU ("scaling": "weak")."""
    import torch
    import torch.distributed as td

    import workloads as W
    from paper_1905_02300_b200 import Shell, dist

    torch.cuda.set_device(local)
    td.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = dist.share_unique_id(rank, device=torch.device("cuda", local))
    weak = args.workload == "C5"
    cfg = W.config(args.workload, G=world) if weak else W.config(args.workload)
    wl = W.make_workload(cfg)
    stream = torch.cuda.Stream()
    dist.plan(world, rank, cfg.nr)                 # validates the slab split
    sh = Shell.dist(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, world, rank, uid, local,
                    stream=stream.cuda_stream, chi=cfg.chi,
                    **({"fixed_iters": args.fixed_iters} if args.fixed_iters else {}))
    sh.load_workload(wl)
    W_ = max(3, args.warmup)
    for _ in range(W_):
        sh.step(1, cfg.tol)
    torch.cuda.synchronize()
    td.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    td.barrier()
    l0 = sh.launch_count()
    ev0.record(stream)
    sh.step(args.steps, cfg.tol)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    td.barrier()
    clocks = clk.stop()
    ms = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    td.all_reduce(ms, op=td.ReduceOp.MAX)
    ms = float(ms.item())
    nl = torch.tensor([sh.launch_count() - l0], device="cuda", dtype=torch.int64)
    td.all_reduce(nl, op=td.ReduceOp.SUM)
    launches = int(nl.item())
    Ks = [k for k, _ in sh.stats()[-args.steps:]]
    forced = len(wl["patches"][0]["sources"]) > 0
    model_bytes = sum(step_model_bytes(cfg, k, forced) for k in Ks)
    if rank == 0:
        emit({"metric": METRIC, "value": 2 * cfg.cells * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
              "steps": args.steps, "warmup": W_, "ms_per_step": ms / args.steps, "higher_is_better": True,
              "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
              "config": {"workload": args.workload, "grid_per_patch": [cfg.nr, cfg.nth, cfg.nph], "patches": 2,
                         "parallelism": f"Yin on ranks 0..{world // 2 - 1}, Yang on the others, "
                                        f"{world // 2} radial slab(s) per patch; NCCL p2p fringe, halos, "
                                        "slab r-solve interfaces, norms",
                         "schwarz_iters_per_step": Ks,
                         "step_roofline": {"model": "SURVEY M1 bytes/cell = %d + 1320 K" % (352 if forced else 256),
                                           "frac_of_8TBs_per_gpu": model_bytes / (world * HBM_NOMINAL_GBS * 1e9)
                                           / (ms / 1e3)}},
              # the step as a whole against the HBM peak of all ranks (the per-class
              # roofline of the dominant kernel is the N = 1 line's)
              "roofline": {"bound": "hbm", "kernel": "whole step (all ranks)",
                           "achieved": model_bytes / (ms / 1e3) / 1e9, "peak": world * measured_peak()[0],
                           "unit": "GB/s", "frac": model_bytes / (ms / 1e3) / 1e9 / (world * measured_peak()[0]),
                           "traffic": None},
              "gpu_launches": launches,
              "e2e": None, "cpu_baseline": None,   # measured at N = 1 only (host-buffer round trip, oracle)
              "clocks": clocks, "timing": "CUDA events on each rank's stream, max over ranks"})
    sh.close()
    td.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="yy", choices=("yy", "reference"))
    ap.add_argument("--workload", default="C3", choices=("C1", "C2", "C3", "C5"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fixed-iters", type=int, default=0,
                    help="Schwarz iterations per step fixed (the paper's scaling protocol, C5: 10); 0 = to tolerance")
    ap.add_argument("--advection", default="split", choices=("split", "imex"),
                    help="transport terms in the split factors (the paper's scheme) or IMEX (SURVEY NEXT-3)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)   # CPU test of the rank launch
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.launch_check:
        return run_launch_check(args)
    return run_yy(args)


if __name__ == "__main__":
    sys.exit(main())

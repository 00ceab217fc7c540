import sys, os
sys.path.insert(0, '.')
print('start', flush=True)
import workloads as W
from paper_1905_02300_b200 import Shell
cfg = W.small("C1", 6, 12, 30, dt=1e-3)
wl = W.make_workload(cfg)
print('creating', flush=True)
sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
print('created', flush=True)
sh.load_workload(wl)
print('loaded', flush=True)
try:
    sh.step(1, cfg.tol)
    print('stepped', sh.stats(), flush=True)
except Exception as e:
    print('EXC', e, flush=True)

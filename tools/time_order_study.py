#!/usr/bin/env python
"""Richardson self-convergence in time of the oracle step (manufactured eq:Exact,
scaled by amp): python tools/time_order_study.py Tf dt1,dt2,... nr,nth,nph amp chi R1 R2"""
import time, numpy as np, workloads as W, math, sys
from oracle.scheme import Oracle
Tf=float(sys.argv[1]); dts=[float(x) for x in sys.argv[2].split(',')]; grid=tuple(int(x) for x in sys.argv[3].split(','))
amp=float(sys.argv[4]); chi=float(sys.argv[5]); R1=float(sys.argv[6]); R2=float(sys.argv[7])
sols=[]
for dt in dts:
    cfg = W.small('C1', *grid, Ra=1.0, dt=dt, extra={'amp': amp}, R1=R1, R2=R2)
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=chi)
    o.load_workload(W.make_workload(cfg))
    t0=time.time(); o.step(int(round(Tf/dt)), 1e-11*amp)
    print(dt, 'time %.1f'%(time.time()-t0), 'iters', [s[0] for s in o.stats][:6], flush=True)
    sols.append((o, [o.get_fields(p,0,1) for p in range(2)], [o.get_fields(p,0,2) for p in range(2)]))
for sysn in (1,2):
  for k in ('ur','ut','up','T','p'):
    errs=[]
    for a in range(len(dts)-1):
        o=sols[a][0]
        kind={'ur':'R','ut':'TH','up':'PH','T':'C','p':'C'}[k]
        blk=o.solved(kind); w=o.g.weights_omega(kind)[blk]
        e2=0
        for p in range(2):
            d=sols[a][sysn][p][k][blk]-sols[a+1][sysn][p][k][blk]
            e2+=np.sum(w*d*d)
        errs.append(math.sqrt(e2))
    print(sysn,k,['%.2e'%e for e in errs],[round(math.log2(errs[i]/errs[i+1]),2) for i in range(len(errs)-1)], flush=True)

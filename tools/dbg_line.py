import sys
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
from paper_1905_02300_b200 import Shell
print('start', flush=True)
nr, nt, npp = 9, 21, 67
a, rhs = W.c4_inputs(nr, nt, npp)
sh = Shell(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, 1e-4)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
for axis in range(3):
    x = dev(rhs)
    print('axis', axis, flush=True)
    sh.line_solve(axis, dev(a["ur"]), dev(a["ut"]), dev(a["up"]), x)
    torch.cuda.synchronize()
    print('ok', axis, float(x.abs().max()), flush=True)

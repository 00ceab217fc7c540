#!/usr/bin/env python
"""C4 kernel-only workload: one 256x384x1152 patch, the T-factor
rows (I - tau/2 A_d) with hats, a* ~ U[-1,1), rhs ~ U[-1,1), one sweep per axis
through yy_line_solve (the same k_line kernels the step uses).  Algorithmic
bytes per element: read rhs, read a*_d, write x = 24 B.  Prints one
JSON line: per axis the CUDA-event time per sweep, the achieved GB/s and the
fraction of the measured HBM copy peak."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1905_02300_b200 import Shell  # noqa: E402


def main(reps=10):
    nr, nt, npp = 256, 384, 1152
    a, rhs = W.c4_inputs(nr, nt, npp)
    sh = Shell(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, 1e-4)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dar, dat, dap = dev(a["ur"]), dev(a["ut"]), dev(a["up"])
    x0 = dev(rhs)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    st = torch.cuda.current_stream()
    sh.set_stream(st.cuda_stream)
    out = {}
    for axis, name in enumerate(("r", "theta", "phi")):
        n = (nr, nt - 2, npp - 2)[axis]
        elems = (nt - 2) * (npp - 2) * nr if axis == 0 else (nr * (npp - 2) * (nt - 2) if axis == 1 else nr * (nt - 2) * (npp - 2))
        bytes_ = 24 * elems
        x = x0.clone()
        sh.line_prepare(dar, dat, dap)             # row weights of a* (the per-step precompute)
        sh.line_solve(axis, None, None, None, x)   # warm-up
        ts = []
        for _ in range(reps):
            x.copy_(x0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            sh.line_solve(axis, None, None, None, x)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        gbs = bytes_ / (ms / 1e3) / 1e9
        out[name] = {"line_len": n, "elements": elems, "ms": ms, "GBps": gbs, "frac_measured_peak": gbs / peak}
    print(json.dumps({"workload": "C4 kernel-only", "grid": [nr, nt, npp], "bytes_per_elem": 24,
                      "peak_GBps": peak, "axes": out, "timing": "CUDA events, median of %d, rhs re-copied "
                      "between launches (inputs 2.7 GB >> L2)" % reps}))


if __name__ == "__main__":
    main()

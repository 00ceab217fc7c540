"""The converged Schwarz iteration against a dense unsplit solve (P:L538-545:
"the iteration becomes a block-preconditioned overlapping domain decomposition
iteration, the preconditioner being the factorized operator"): with the
splitting-error reduction eq:er iterated to tolerance, the temperature of one
step is the solution of the coupled linear system

    (I - tau/2 L^_T)(T_p - T_p^n) = G_T,p   on the solved nodes of each patch p,
    fringe of T_p = Lagrange interpolation of T_{3-p},

which this test assembles column by column and solves densely (numpy LAPACK),
on a 6 x 12 x 28 grid, for both places of the linearised advection:
inside the split factors (the paper's scheme) and IMEX (explicit, SURVEY
NEXT-3).  The two fixed points differ, each equals its own dense solve.  The factorised sweeps, the increment form and the Schwarz loop are
what is pinned; the operator rows are pinned in test_oracle_ops.py."""
import numpy as np
import pytest

import workloads as W
from oracle.scheme import Oracle


def _oracle(adv, tol):
    cfg = W.small("C1", 6, 12, 28, dt=2e-2, Ra=1.0)
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, chi=16.0, advection=adv,
               max_iters=400)
    o.load_workload(W.make_workload(cfg))
    return o, cfg


def _dense_T(o):
    """Assemble and solve the coupled fixed-point system of T for the next step."""
    tau, t = o.prm.dt, o.t
    o._cc = {}
    stat = [o.static(p, t) for p in range(2)]
    blk = o.solved("C")
    shp = o.g.shape("C")
    nsol = int(np.prod([s.stop - s.start for s in blk]))
    wnew = [o.wall(p, "T", t + tau) for p in range(2)]
    wdiff = [wnew[p] - o.wall(p, "T", t) for p in range(2)]
    Tn = [o.state[p]["n"]["T"] for p in range(2)]

    def F(x):
        T = []
        for p in range(2):
            a = Tn[p].copy()
            a[blk] = x[p * nsol:(p + 1) * nsol].reshape(a[blk].shape)
            T.append(a)
        out = []
        for p in range(2):
            a = T[p].copy()
            o.ex.fill_scalar("C", a, T[1 - p])          # fringe from the other patch
            X = a - Tn[p]
            astar, G = stat[p]
            r = X - 0.5 * tau * o.L("T", X, wdiff[p], True, astar) - G["T"]
            out.append(r[blk].ravel())
        return np.concatenate(out)

    x0 = np.concatenate([Tn[p][blk].ravel() for p in range(2)])
    f0 = F(x0)
    A = np.empty((2 * nsol, 2 * nsol))
    for i in range(2 * nsol):
        e = x0.copy()
        e[i] += 1.0
        A[:, i] = F(e) - f0
    x = x0 + np.linalg.solve(A, -f0)
    out = []
    for p in range(2):
        a = np.zeros(shp)
        a[blk] = x[p * nsol:(p + 1) * nsol].reshape(a[blk].shape)
        out.append(a)
    return out


@pytest.mark.parametrize("adv", ["split", "imex"])
def test_converged_iteration_equals_dense_solve(adv):
    o, cfg = _oracle(adv, 1e-14)
    o.step(2, 1e-13)                    # leave the start-up step; a* from two levels
    ref = _dense_T(o)
    o.step(1, 1e-13)
    blk = o.solved("C")
    for p in range(2):
        got = o.state[p]["n"]["T"][blk]
        assert np.max(np.abs(got - ref[p][blk])) <= 1e-10 * np.max(np.abs(ref[p][blk])), (adv, p)


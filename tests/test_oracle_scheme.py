"""Pins of the whole oracle step (oracle/scheme.py) against the mathematics:

* second-order spatial convergence to the manufactured solution eq:Exact
  ('second order accuracy of the scheme in space'),
* second-order temporal convergence of the Douglas/eq:er temperature path on a
  heat-only manufactured case (eq:HeatDouglas),
* recovery of the steady Landau jet with errors falling ~h^2,
* exact invariants: zero stays zero; with the splitting-error reduction
  iterated to tolerance the step does not depend on the factor order
  (SPEC S:L489); the pressure update identity.
These use only closed forms (workloads/) as references.
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import ops
from oracle.scheme import Oracle

KIND = {"ur": "R", "ut": "TH", "up": "PH", "T": "C", "p": "C"}


def _run(cfg, steps, tol=1e-10, **kw):
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, **kw)
    wl = W.make_workload(cfg)
    o.load_workload(wl)
    o.step(steps, tol)
    return o, wl


def _l2(o, a, b, k, demean=False):
    blk = o.solved(KIND[k])
    w = o.g.weights_omega(KIND[k])[blk]
    e2 = 0.0
    for p in range(2):
        d = a[p][k][blk] - b[p][k][blk]
        if demean:
            d = d - np.sum(w * d) / np.sum(w)
        e2 += np.sum(w * d * d)
    return math.sqrt(e2)


def _exact_at(wl, t, A=1.0):
    c = math.cos(t)
    out = []
    for pd in wl["patches"]:
        d = {k: pd["n"][k] * c for k in ("ur", "ut", "up", "T")}
        d["p"] = pd["n"]["p2"] * c
        out.append(d)
    return out


def test_zero_state_stays_zero():
    cfg = W.small("C1", 4, 12, 28, problem="zero")
    o, _ = _run(cfg, 2)
    for p in range(2):
        for s in (1, 2):
            for k, v in o.get_fields(p, 0, s).items():
                assert np.all(v == 0.0), k


@pytest.mark.slow
def test_space_second_order_manufactured():
    errs = []
    for n in ((8, 20, 52), (16, 36, 100)):
        cfg = W.small("C1", *n, Ra=1.0, dt=1e-3)
        o, wl = _run(cfg, 10)
        ex = _exact_at(wl, o.t)
        got = [o.get_fields(p, 0, 2) for p in range(2)]
        errs.append({k: _l2(o, got, ex, k, demean=(k == "p")) for k in KIND})
    for k in KIND:
        order = math.log2(errs[0][k] / errs[1][k])
        assert order > 1.7, (k, errs)


@pytest.mark.slow
def test_time_second_order_heat():
    sols = []
    for dt in (0.02, 0.01, 0.005):
        cfg = W.small("C1", 4, 12, 28, Ra=0.0, dt=dt, problem="heat")
        o, _ = _run(cfg, int(round(0.2 / dt)), tol=1e-11)
        sols.append([o.get_fields(p, 0, 2) for p in range(2)])
    e1 = _l2(o, sols[0], sols[1], "T")
    e2 = _l2(o, sols[1], sols[2], "T")
    assert math.log2(e1 / e2) > 1.8, (e1, e2)


@pytest.mark.slow
def test_landau_recovery():
    errs = []
    for n in ((8, 20, 52), (16, 36, 100)):
        cfg = W.small("C2", *n, dt=5e-4)
        o, wl = _run(cfg, 8)
        ex = [{k: pd["n"]["p2" if k == "p" else k] for k in ("ur", "ut", "up", "p")} for pd in wl["patches"]]
        got = [o.get_fields(p, 0, 2) for p in range(2)]
        errs.append({k: _l2(o, got, ex, k, demean=(k == "p")) for k in ("ur", "ut", "up", "p")})
    # after 8 steps the velocity error is still in its initial transient
    # (ratio ~2.2 at 8 steps, ~3.4 at 20 steps); the pressure is at O(h^2)
    for k in ("ur", "ut", "up"):
        assert errs[1][k] < errs[0][k] / 2.0, (k, errs)
    assert errs[1]["p"] < errs[0]["p"] / 3.5, errs
    assert errs[1]["ur"] < 1e-3 * 0.08          # |u| ~ 4 nu/(a-1) = 0.08 at r = 1


def test_converged_step_independent_of_factor_order():
    cfg = W.small("C1", 4, 12, 28, Ra=1.0, dt=2e-3)
    o1, _ = _run(cfg, 2, tol=1e-13, max_iters=400)
    o2, _ = _run(cfg, 2, tol=1e-13, max_iters=400,
                 factor_order={"T": (2, 1, 0), "ur": (0, 1, 2), "ut": (1, 0, 2), "up": (2, 0, 1)})
    assert o1.stats[-1][1] < 1e-13 and o2.stats[-1][1] < 1e-13
    for p in range(2):
        a, b = o1.get_fields(p, 0, 2), o2.get_fields(p, 0, 2)
        for k in a:
            assert np.max(np.abs(a[k] - b[k])) <= 1e-9 * np.max(np.abs(a[k])), k


def test_pressure_update_identity():
    cfg = W.small("C1", 4, 12, 28, Ra=1.0, dt=1e-3)
    o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    o.load_workload(W.make_workload(cfg))
    before = [o.get_fields(p, 0, 1) for p in range(2)]
    o.step(1, 1e-10)
    after = [o.get_fields(p, 0, 1) for p in range(2)]
    blk = o.solved("C")
    for p in range(2):
        ub = [0.5 * (after[p][q] + before[p][q]) for q in ("ur", "ut", "up")]
        d = ops.div(o.g, *ub)
        lhs = after[p]["p"] - before[p]["p"] + d / o.prm.chi
        assert np.max(np.abs(lhs[blk])) < 1e-12 * np.max(np.abs(after[p]["p"]))


def test_schwarz_iteration_converges_and_counts_recorded():
    cfg = W.small("C1", 4, 12, 28, Ra=1.0, dt=1e-3)
    o, _ = _run(cfg, 2)
    assert all(1 < k < 30 and r < 1e-10 for k, r in o.stats)


def test_multiplicative_and_additive_fixed_points_agree():
    """SURVEY NEXT-1 / S:L482: the multiplicative Schwarz of Algorithm 1 as printed
    (Yin with Yang's k-1, then Yang with Yin's fresh k) and the
    additive variant (RD26) iterate to the same per-step fixed point, within
    10 tol, from the same inputs; with one iteration per step they differ (the
    multiplicative Yang sweep sees the new Yin fringe)."""
    import workloads as W
    cfg = W.small("C1", 6, 12, 30, dt=1e-3)
    wl = W.make_workload(cfg)
    tol = 1e-10
    out = {}
    for mode in ("additive", "multiplicative"):
        o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, schwarz=mode)
        o.load_workload(wl)
        o.step(2, tol)
        assert all(r < tol for _, r in o.stats)
        out[mode] = [o.get_fields(p, 0, s) for p in range(2) for s in (1, 2)]
    for a, b in zip(out["additive"], out["multiplicative"]):
        for k in a:
            assert np.max(np.abs(a[k] - b[k])) <= 10 * tol, k
    one = {}
    for mode in ("additive", "multiplicative"):
        o = Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, schwarz=mode, fixed_iters=1)
        o.load_workload(wl)
        o.step(1, tol)
        one[mode] = o.get_fields(1, 0, 2)      # Yang
    assert max(np.max(np.abs(one["additive"][k] - one["multiplicative"][k])) for k in one["additive"]) > 1e-12

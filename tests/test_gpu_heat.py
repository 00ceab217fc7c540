"""the heat Douglas scheme alone (eq:HeatDouglas), the
T path of the step with u = 0 (YY_HEAT_ONLY skips the momentum and pressure
kernels).  Parity against the oracle's full step with u = 0 (where the momentum
and pressure increments vanish identically), and the unconditional stability of
Theorem 1 in the form of SPEC criterion 4: homogeneous
problem, random initial data, 8x24x48 per patch, 200 steps for tau up to 100, one
split step per time step: finite and max-norm bounded by 10x the initial one."""
import numpy as np
import pytest

import workloads as W
from oracle.scheme import Oracle

pytestmark = pytest.mark.gpu


def _random_heat(nr, nt, npp, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, (nr, nt, npp)) for _ in range(2)]


@pytest.mark.parametrize("tau,fixed", [(1e-3, 0), (1.0, 0), (10.0, 1)])
def test_heat_only_matches_oracle(tau, fixed):
    from paper_1905_02300_b200 import Shell
    nr, nt, npp = 8, 24, 48
    Ts = _random_heat(nr, nt, npp, 3)
    sh = Shell(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, tau, heat_only=True, fixed_iters=fixed or None, max_iters=40)
    o = Oracle(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, tau, fixed_iters=fixed, max_iters=40)
    for p in range(2):
        sh.set_fields(p, 0, 0, T=Ts[p])
        sh.set_fields(p, 1, 0, T=Ts[p])
        o.set_fields(p, 0, 0, {"T": Ts[p]})
        o.set_fields(p, 1, 0, {"T": Ts[p]})
    for _ in range(3):
        sh.step(1, 1e-10)
        o.step(1, 1e-10)
        assert sh.stats()[-1][0] == o.stats[-1][0]
        for p in range(2):
            a = sh.get_fields(p, 0, 1, names=("T",))["T"]
            b = o.get_fields(p, 0, 1)["T"]
            assert np.max(np.abs(a - b)) <= 1e-11 * np.max(np.abs(b))


@pytest.mark.parametrize("tau", [0.1, 1.0, 10.0, 100.0])
def test_heat_douglas_unconditionally_stable(tau):
    from paper_1905_02300_b200 import Shell
    nr, nt, npp = 8, 24, 48
    Ts = _random_heat(nr, nt, npp, 7)
    sh = Shell(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, tau, heat_only=True, fixed_iters=1)
    for p in range(2):
        sh.set_fields(p, 0, 0, T=Ts[p])
        sh.set_fields(p, 1, 0, T=Ts[p])
    m0 = max(np.max(np.abs(t)) for t in Ts)
    worst = 0.0
    for _ in range(20):
        sh.step(10, 1e-10)
        m = max(np.max(np.abs(sh.get_fields(p, 0, 1, names=("T",))["T"])) for p in range(2))
        assert np.isfinite(m)
        worst = max(worst, m)
    assert worst <= 10 * m0, (tau, worst / m0)


@pytest.mark.parametrize("tau", [0.1, 1.0, 10.0, 100.0])
def test_theorem1_energy_parity_and_monotone(tau):
    """Theorem 1 proper (eq:Stability): single domains (YY_SCHWARZ = 2, no
    exchange), homogeneous Dirichlet data on every side (zero fringe and walls),
    one factored solve per step (eq:HeatDouglas).  The left side of eq:Stability
    from yy_energy is non-increasing step by step, and equals the oracle's
    (oracle/energy.py) step by step within 1e-11 relative (SPEC criterion 4 grid
    and tau values)."""
    from oracle.energy import stability_terms
    from paper_1905_02300_b200 import Shell
    nr, nt, npp = 8, 24, 48
    rng = np.random.default_rng(4)
    sh = Shell(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, tau, heat_only=True, fixed_iters=1, schwarz="none")
    o = Oracle(nr, nt, npp, 1.0, 2.0, 1.0, 0.0, tau, fixed_iters=1, schwarz="none")
    for p in range(2):
        T = np.zeros((nr, nt, npp))
        T[:, 1:-1, 1:-1] = rng.standard_normal((nr, nt - 2, npp - 2))
        sh.set_fields(p, 0, 0, T=T)
        sh.set_fields(p, 1, 0, T=T)
        o.set_fields(p, 0, 0, {"T": T})
        o.set_fields(p, 1, 0, {"T": T})
    Sg, So, acc_g, acc_o = [], [], 0.0, 0.0
    for n in range(13):
        if n:
            sh.step(1, 1e-10)
            o.step(1, 1e-10)
        eg = sh.energy()
        eo = [sum(x) for x in zip(*(stability_terms(o, p) for p in range(2)))]
        for a, b in zip(eg, eo):
            assert abs(a - b) <= 1e-11 * max(abs(eo[0]), 1e-300), (n, eg, eo)
        acc_g += eg[2] / tau if n else 0.0
        acc_o += eo[2] / tau if n else 0.0
        Sg.append(acc_g + eg[0] + eg[1])
        So.append(acc_o + eo[0] + eo[1])
    dS = np.diff(Sg)
    assert np.all(dS < 0) and np.all(dS <= 1e-12 * Sg[0]), dS / Sg[0]
    assert np.max(np.abs(np.array(Sg) - np.array(So))) <= 1e-11 * So[0]

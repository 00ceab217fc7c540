"""Theorem 1 (eq:Stability) as a pin of the oracle's heat
path: the Douglas scheme eq:HeatDouglas (one factored solve per step = the
first Schwarz iteration, RD25) on single patches (no exchange) with homogeneous
Dirichlet data is unconditionally stable, the left side of eq:Stability
(oracle/energy.py) non-increasing step by step at any tau (SPEC criterion 4:
8x24x48, tau in {0.1, 1, 10, 100})."""
import numpy as np
import pytest

from oracle.energy import stability_terms
from oracle.scheme import Oracle


def run_energy(tau, steps, grid=(8, 24, 48), seed=4):
    o = Oracle(*grid, 1.0, 2.0, 1.0, 0.0, tau, fixed_iters=1, schwarz="none")
    rng = np.random.default_rng(seed)
    for p in range(2):
        T = np.zeros(o.g.shape("C"))
        T[o.solved("C")] = rng.standard_normal(T[o.solved("C")].shape)
        o.set_fields(p, 0, 1, {"T": T})
        o.set_fields(p, 1, 1, {"T": T})
    seq, acc = [], 0.0
    e = [stability_terms(o, p) for p in range(2)]
    seq.append(sum(x[0] + x[1] for x in e))
    for _ in range(steps):
        o.step(1)
        e = [stability_terms(o, p) for p in range(2)]
        acc += sum(x[2] for x in e) / tau
        seq.append(acc + sum(x[0] + x[1] for x in e))
    return np.array(seq), o


@pytest.mark.parametrize("tau", [0.1, 1.0, 10.0, 100.0])
def test_theorem1_energy_non_increasing(tau):
    S, o = run_energy(tau, 12)
    assert np.all(np.isfinite(S)) and S[0] > 0
    dS = np.diff(S)
    assert np.all(dS <= 1e-12 * S[0]), (tau, dS / S[0])
    # the estimate is not vacuous: every step strictly drains it
    assert np.all(dS < 0) and S[-1] < S[0] * (1 - 1e-7)
    # momentum and pressure stay exactly zero (u = 0, Ra = 0, no data)
    f = o.get_fields(0, 0, 2)
    assert max(np.abs(f[k]).max() for k in ("ur", "ut", "up", "p")) == 0.0


def _mode(g, r, th, ph):
    """sin(pi (r-R1)/(R2-R1)) sin(pi (th-a)/L_th) sin(pi (ph-b)/L_ph): zero on the
    walls and on the fringe node centres of kind C (the homogeneous Dirichlet
    data of the theorem)."""
    a, b = g.x0[1] + 0.5 * g.dth, g.x0[2] + 0.5 * g.dph
    Lt, Lp = (g.nth - 1) * g.dth, (g.nph - 1) * g.dph
    return (np.sin(np.pi * (r - g.R1) / (g.R2 - g.R1)) * np.sin(np.pi * (th - a) / Lt)
            * np.sin(np.pi * (ph - b) / Lp)), (a, Lt, b, Lp)


def _continuous_terms(g, ngl=48):
    """1/2 int |grad T|^2 and 1/4 int [(r^2/R1^2 - 1) sin(th) T_th^2 +
    (r^2 sin(th)/(R1^2 sin^2 th_1) - 1/sin(th)) T_ph^2] dr dth dph over the box
    between the fringe centres (Gauss-Legendre, closed-form derivatives)."""
    _, (a, Lt, b, Lp) = _mode(g, np.zeros(1), np.zeros(1), np.zeros(1))
    x, w = np.polynomial.legendre.leggauss(ngl)
    def nodes(lo, hi):
        return 0.5 * (hi - lo) * x + 0.5 * (hi + lo), 0.5 * (hi - lo) * w
    r, wr = nodes(g.R1, g.R2)
    th, wt = nodes(a, a + Lt)
    ph, wp = nodes(b, b + Lp)
    R, TH, PH = np.meshgrid(r, th, ph, indexing="ij")
    W = wr[:, None, None] * wt[None, :, None] * wp[None, None, :]
    kr, kt, kp = np.pi / (g.R2 - g.R1), np.pi / Lt, np.pi / Lp
    sr, st, sp = np.sin(kr * (R - g.R1)), np.sin(kt * (TH - a)), np.sin(kp * (PH - b))
    Tr = kr * np.cos(kr * (R - g.R1)) * st * sp
    Tt = kt * sr * np.cos(kt * (TH - a)) * sp
    Tp = kp * sr * st * np.cos(kp * (PH - b))
    grad2 = Tr ** 2 + Tt ** 2 / R ** 2 + Tp ** 2 / (R ** 2 * np.sin(TH) ** 2)
    e_grad = 0.5 * np.sum(W * grad2 * R ** 2 * np.sin(TH))
    s1 = np.sin(g.theta1) ** 2
    e_hat = 0.25 * np.sum(W * ((R ** 2 / g.R1 ** 2 - 1) * np.sin(TH) * Tt ** 2
                               + (R ** 2 * np.sin(TH) / (g.R1 ** 2 * s1) - 1 / np.sin(TH)) * Tp ** 2))
    return e_grad, e_hat


def test_energy_terms_converge_to_the_continuous_functional():
    # the discrete terms of eq:Stability (full and hat operators, omega weights)
    # against their continuous integrals (integration by parts of P:L243-249 and
    # eq:StabProof3-4 with the positive weights of RD34), evaluated by Gauss
    # quadrature: second-order convergence.  A wrong hat constant, a dropped
    # metric factor or a sign error changes the limit.
    rel = []
    for n in (1, 2, 4):
        o = Oracle(4 * n, 12 * n, 28 * n, 1.0, 2.0, 1.0, 0.0, 1.0, fixed_iters=1, schwarz="none")
        g = o.g
        T, _ = _mode(g, g.bcast("C", 0), g.bcast("C", 1), g.bcast("C", 2))
        T = np.broadcast_to(T, g.shape("C")).copy()
        o.set_fields(0, 0, 1, {"T": T})
        o.set_fields(0, 1, 1, {"T": np.zeros_like(T)})     # dT^n = T
        eg, eh, ed = stability_terms(o, 0)
        cg, ch = _continuous_terms(g)
        rel.append((abs(eg - cg) / cg, abs(eh - ch) / ch))
    assert rel[-1][0] < 5e-3 and rel[-1][1] < 5e-3, rel
    for (a0, _), (a1, _) in zip(rel, rel[1:]):
        assert a0 / a1 > 3.0, rel                  # second order (gradient part)
    # the hat part starts small (error cancellation) but still converges
    assert all(b < 2e-3 for _, b in rel) and rel[-1][1] < rel[0][1] / 3, rel

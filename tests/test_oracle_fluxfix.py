"""Pins of the mass-flux correction (Algorithm 1 step 4; oracle/fluxfix.py)."""
import numpy as np

from oracle import fluxfix, ops
from oracle.grid import Grid


def _rand_u(g, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(g.shape("R")), rng.standard_normal(g.shape("TH")),
            rng.standard_normal(g.shape("PH")))


def test_net_flux_is_the_divergence_theorem():
    """oint u.n over the cell-box surface = sum over every cell of div(u) * volume,
    with div the MAC divergence of ops: exact for any u."""
    g = Grid(6, 14, 40)
    ur, ut, up = _rand_u(g, 1)
    dv = ops.div(g, ur, ut, up)
    vol = g.bcast("C", 0) ** 2 * np.sin(g.bcast("C", 1)) * g.dr * g.dth * g.dph
    lhs = fluxfix.net_flux(g, ur, ut, up)
    rhs = float((dv * vol).sum())
    assert abs(lhs - rhs) <= 1e-12 * (abs(rhs) + np.abs(dv * vol).sum())


def test_zero_flux_and_no_penalty_leave_the_data_unchanged():
    g = Grid(6, 14, 40)
    z = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    assert not fluxfix.flux_fix(g, *z, tol=1e-12)
    ur, ut, up = _rand_u(g, 2)
    ut0, up0 = ut.copy(), up.copy()
    fluxfix.flux_fix(g, ur, ut, up, tol=0.0, eps=1e30)      # eps -> infinity: penalty off
    assert np.max(np.abs(ut - ut0)) < 1e-20 and np.max(np.abs(up - up0)) < 1e-20


def test_uniform_normal_velocity_is_corrected_by_the_area_weights():
    """uniform outward normal velocity c on the theta/phi sides, no wall flux:
    the correction is -mu a (area weighted) and the remaining flux is the penalty
    share eps A^2 / (eps A^2 + |a|^2) of the initial one."""
    g = Grid(6, 14, 40)
    ur = np.zeros(g.shape("R"))
    ut = np.zeros(g.shape("TH"))
    up = np.zeros(g.shape("PH"))
    c = 0.3
    ut[:, 0, :], ut[:, -1, :] = -c, c
    up[:, :, 0], up[:, :, -1] = -c, c
    F0 = fluxfix.net_flux(g, ur, ut, up)
    at, ap = fluxfix.side_areas(g)
    assert abs(F0 - c * (np.abs(at).sum() + np.abs(ap).sum())) < 1e-12 * F0
    eps = 1e-6
    assert fluxfix.flux_fix(g, ur, ut, up, tol=1e-12, eps=eps)
    a2 = (at ** 2).sum() + (ap ** 2).sum()
    A = fluxfix.total_area(g)
    share = eps * A * A / (eps * A * A + a2)
    assert abs(fluxfix.net_flux(g, ur, ut, up) - share * F0) <= 1e-12 * F0
    d = ut[:, 0, :] + c                           # the change at the theta_min side
    assert np.allclose(d / at[0], d.flat[0] / at[0].flat[0])


def test_closed_form_minimises_J():
    """The rank-one closed form is the minimiser of J as printed:
    J at the returned v is below J at random perturbations of it."""
    g = Grid(5, 12, 32)
    ur, ut, up = _rand_u(g, 3)
    eps = 1e-3
    at, ap = fluxfix.side_areas(g)
    aw = fluxfix.wall_areas(g)
    A = fluxfix.total_area(g)
    b = (aw[0][:, None] * ur[0]).sum() + (aw[1][:, None] * ur[-1]).sum()
    u0 = np.concatenate([ut[:, 0, :].ravel(), ut[:, -1, :].ravel(), up[:, :, 0].ravel(), up[:, :, -1].ravel()])
    avec = np.concatenate([at[0].ravel(), at[1].ravel(), ap[0].ravel(), ap[1].ravel()])

    def J(v):
        return 0.5 * ((v - u0) ** 2).sum() + 0.5 / (eps * A * A) * (avec @ v + b) ** 2

    fluxfix.flux_fix(g, ur, ut, up, tol=0.0, eps=eps)
    v = np.concatenate([ut[:, 0, :].ravel(), ut[:, -1, :].ravel(), up[:, :, 0].ravel(), up[:, :, -1].ravel()])
    rng = np.random.default_rng(4)
    for _ in range(20):
        assert J(v) <= J(v + 1e-4 * rng.standard_normal(v.size))
    # stationarity: grad J = (v - u0) + (a.v + b)/(eps A^2) a = 0
    grad = (v - u0) + (avec @ v + b) / (eps * A * A) * avec
    assert np.max(np.abs(grad)) <= 1e-10 * np.max(np.abs(u0))

"""Algorithm 1 step 4: mass-flux correction of the
interpolated boundary velocity of one patch.  TEST INFRASTRUCTURE (oracle):
only tests/, __graft_entry__.smoke() and bench.py's CPU legs use it.

If |oint_{dOmega_i} u_bd . n| >= tol, replace the interpolated normal velocities v
on the theta/phi sides of the patch by the minimiser of

    J(v) = 1/2 |v - u_bd|^2_{l2}
         + 1/(2 eps |dOmega_i|^2) | oint_{theta,phi sides} v . n + oint_{r walls} u_bd . n |^2

(P:L500-503).  J is quadratic with a rank-one penalty, so the minimiser the paper
reaches by conjugate gradients is written out:

    v = u - mu a,   mu = (a . u + b) / (eps |dOmega|^2 + |a|^2),

a = the signed face areas of the side faces, b = the wall flux.

Reading RD-E5: the closed surface is the boundary of the patch's
whole cell box (fringe cells included) — the theta-faces j = 0, nth of u_theta and
the phi-faces k = 0, nph of u_phi (the fringe normal velocities, RD3) and the two
walls (u_r at i = 0, nr); face areas r sin(theta) dr dphi (theta-faces),
r dr dtheta (phi-faces), r^2 sin(theta) dtheta dphi (walls) at the face centres;
|dOmega| = the sum of all of them; the l2 norm is the plain sum over the side
values; eps defaults to 1e-6."""
from __future__ import annotations

import numpy as np

from .grid import Grid


def side_areas(g: Grid):
    """Signed areas (outward normal) of the theta-faces j = 0, nth (shape (2, nr, nph))
    and of the phi-faces k = 0, nph (shape (2, nr, nth))."""
    rc = g.centres(0)
    tf = g.faces(1)
    at = np.empty((2, g.nr, g.nph))
    at[0] = -(rc * np.sin(tf[0]))[:, None] * g.dr * g.dph
    at[1] = +(rc * np.sin(tf[-1]))[:, None] * g.dr * g.dph
    ap = np.empty((2, g.nr, g.nth))
    ap[0] = -(rc[:, None] * g.dr * g.dth) * np.ones((1, g.nth))
    ap[1] = +(rc[:, None] * g.dr * g.dth) * np.ones((1, g.nth))
    return at, ap


def wall_areas(g: Grid):
    """Outward wall areas r^2 sin(theta_c) dtheta dphi at r = R1 (negative) and R2, shape (2, nth)."""
    tc = g.centres(1)
    return np.stack([-g.R1 ** 2 * np.sin(tc) * g.dth * g.dph, g.R2 ** 2 * np.sin(tc) * g.dth * g.dph])


def total_area(g: Grid) -> float:
    at, ap = side_areas(g)
    aw = wall_areas(g)
    return float(np.abs(at).sum() + np.abs(ap).sum() + np.abs(aw).sum() * g.nph)


def net_flux(g: Grid, ur, ut, up) -> float:
    """oint u . n over the patch's cell-box surface (side normals + walls)."""
    at, ap = side_areas(g)
    aw = wall_areas(g)
    f = (at[0] * ut[:, 0, :]).sum() + (at[1] * ut[:, -1, :]).sum()
    f += (ap[0] * up[:, :, 0]).sum() + (ap[1] * up[:, :, -1]).sum()
    f += (aw[0][:, None] * ur[0]).sum() + (aw[1][:, None] * ur[-1]).sum()
    return float(f)


def flux_fix(g: Grid, ur, ut, up, tol: float, eps: float = 1e-6) -> bool:
    """Apply Algorithm 1 step 4 in place to the side normal velocities of ut, up.
    Returns whether the correction was applied (|net flux| >= tol)."""
    F = net_flux(g, ur, ut, up)
    if not abs(F) >= tol:
        return False
    at, ap = side_areas(g)
    a2 = float((at ** 2).sum() + (ap ** 2).sum())
    A = total_area(g)
    mu = F / (eps * A * A + a2)
    ut[:, 0, :] -= mu * at[0]
    ut[:, -1, :] -= mu * at[1]
    up[:, :, 0] -= mu * ap[0]
    up[:, :, -1] -= mu * ap[1]
    return True

"""MAC finite-difference operators on one chart (plain numpy, fp64).

PAPER.md §3.2 (L185-226) defines the split Laplacian and the hat operators;
§3.3 (L364-454) the grad-div split D_ij and the three component operators
L_{q,d}; §4 (L473-475) second-order centred FD on a MAC grid.  The discrete
forms are SURVEY.md Appendix A (reading RD30): flux forms for Delta_rr,
Delta_thth and div; centred first differences; arithmetic averages for
staggered transfers (2-point per differing axis).

Conventions: every array has its kind's full shape; entries an operator
cannot define (a missing neighbour) are NaN, so a NaN reaching a solved node
fails loudly.  Quantities: q in {"T", "ur", "ut", "up"}; kinds C, R, TH, PH.
"""
from __future__ import annotations

import numpy as np

from .grid import KINDS, Grid

QKIND = {"T": "C", "p": "C", "ur": "R", "ut": "TH", "up": "PH"}
CENTRED_R = ("C", "TH", "PH")      # kinds whose r-nodes are cell centres (wall ghost RD22)


# ---- elementary index shifts ----------------------------------------------------
def shift(X: np.ndarray, axis: int, s: int) -> np.ndarray:
    """Y[.., i, ..] = X[.., i+s, ..] along axis; NaN where i+s is out of range."""
    Y = np.full(X.shape, np.nan)
    n = X.shape[axis]
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if s > 0:
        src[axis] = slice(s, n)
        dst[axis] = slice(0, n - s)
    else:
        src[axis] = slice(0, n + s)
        dst[axis] = slice(-s, n)
    Y[tuple(dst)] = X[tuple(src)]
    return Y


def shift_r_ghost(X: np.ndarray, s: int, wall) -> np.ndarray:
    """r-shift of an r-centred field with the wall ghost psi_{-1} = 2 w_lo - psi_0,
    psi_{Nr} = 2 w_hi - psi_{Nr-1} (reading RD22)."""
    Y = shift(X, 0, s)
    if s == -1:
        Y[0] = 2.0 * wall[0] - X[0]
    else:
        Y[-1] = 2.0 * wall[1] - X[-1]
    return Y


def to_kind(X: np.ndarray, src: str, dst: str) -> np.ndarray:
    """Arithmetic average of X (kind src) to the nodes of kind dst: along every
    axis where the staggerings differ, face->centre = mean of the two bounding
    faces; centre->face = mean of the two adjacent centres (NaN on boundary
    faces).  SURVEY.md Appendix A 'Advection' (2-point or 4-point averages)."""
    Y = X
    for a in range(3):
        fs, fd = KINDS[src][a], KINDS[dst][a]
        if fs == fd:
            continue
        if fs == "f":   # faces n+1 -> centres n
            Y = 0.5 * (np.take(Y, range(0, Y.shape[a] - 1), axis=a) + np.take(Y, range(1, Y.shape[a]), axis=a))
        else:           # centres n -> faces n+1, interior faces only
            inner = 0.5 * (np.take(Y, range(0, Y.shape[a] - 1), axis=a) + np.take(Y, range(1, Y.shape[a]), axis=a))
            shp = list(Y.shape)
            shp[a] = Y.shape[a] + 1
            Z = np.full(shp, np.nan)
            idx = [slice(None)] * 3
            idx[a] = slice(1, Y.shape[a])
            Z[tuple(idx)] = inner
            Y = Z
    return Y


# ---- divergence contributions and gradients (Appendix A) ----------
def div1(g: Grid, ur):
    """(1/r^2) d_r(r^2 u_r) at cell centres, flux form."""
    rf = g.faces(0)[:, None, None]
    rc = g.centres(0)[:, None, None]
    return (rf[1:] ** 2 * ur[1:] - rf[:-1] ** 2 * ur[:-1]) / (rc ** 2 * g.dr)


def div2(g: Grid, ut):
    """(1/(r sin th)) d_th(sin th u_th) at cell centres."""
    rc = g.centres(0)[:, None, None]
    sf = np.sin(g.faces(1))[None, :, None]
    sc = np.sin(g.centres(1))[None, :, None]
    return (sf[:, 1:] * ut[:, 1:] - sf[:, :-1] * ut[:, :-1]) / (rc * sc * g.dth)


def div3(g: Grid, up):
    """(1/(r sin th)) d_ph u_ph at cell centres."""
    rc = g.centres(0)[:, None, None]
    sc = np.sin(g.centres(1))[None, :, None]
    return (up[:, :, 1:] - up[:, :, :-1]) / (rc * sc * g.dph)


def div(g: Grid, ur, ut, up):
    """MAC divergence (used by the pressure update eq:nst_Mass1)."""
    return div1(g, ur) + div2(g, ut) + div3(g, up)


def grad1(g: Grid, c):
    """d_r c at r-faces (interior faces; NaN on the walls)."""
    out = np.full(g.shape("R"), np.nan)
    out[1:-1] = (c[1:] - c[:-1]) / g.dr
    return out


def grad2(g: Grid, c):
    """(1/r) d_th c at theta-faces."""
    out = np.full(g.shape("TH"), np.nan)
    rc = g.centres(0)[:, None, None]
    out[:, 1:-1] = (c[:, 1:] - c[:, :-1]) / (rc * g.dth)
    return out


def grad3(g: Grid, c):
    """(1/(r sin th)) d_ph c at phi-faces."""
    out = np.full(g.shape("PH"), np.nan)
    rc = g.centres(0)[:, None, None]
    sc = np.sin(g.centres(1))[None, :, None]
    out[:, :, 1:-1] = (c[:, :, 1:] - c[:, :, :-1]) / (rc * sc * g.dph)
    return out


# ---- three-point directional operators -------------------------------------------
class Params:
    """Physical / scheme parameters: nu = Pr (RD33), kappa = 1, c_chi = 1/(2 chi) (RD11)."""

    def __init__(self, Pr: float, Ra: float, dt: float, chi: float = 1.0):
        self.Pr, self.Ra, self.dt, self.chi = Pr, Ra, dt, chi
        self.nu = Pr
        self.kappa = 1.0
        self.cchi = 1.0 / (2.0 * chi)


def _zeros3(g, kind):
    return [np.zeros(g.shape(kind)) for _ in range(3)]


def _lap_r(g: Grid, kind: str, coef: float):
    """Delta_rr = (1/r^2) d_r(r^2 d_r) in flux form at the kind's r-nodes."""
    am, a0, ap = _zeros3(g, kind)
    rn = g.bcast(kind, 0)
    if KINDS[kind][0] == "c":
        rf = g.faces(0)
        rm = rf[:-1].reshape(-1, 1, 1)
        rp = rf[1:].reshape(-1, 1, 1)
    else:
        rc = g.centres(0)
        rm = np.concatenate([[np.nan], rc]).reshape(-1, 1, 1)
        rp = np.concatenate([rc, [np.nan]]).reshape(-1, 1, 1)
    am = am + coef * rm ** 2 / (rn ** 2 * g.dr ** 2)
    ap = ap + coef * rp ** 2 / (rn ** 2 * g.dr ** 2)
    a0 = a0 - am - ap
    return am, a0, ap


def _lap_th(g: Grid, kind: str, coef: float, hat: bool):
    """Delta_thth = (1/(rho^2 sin th)) d_th(sin th d_th); rho = R1 for the hat
    operator, rho = r for the full one."""
    rn = g.bcast(kind, 0)
    rho2 = g.R1 ** 2 if hat else rn ** 2
    th = g.bcast(kind, 1)
    if KINDS[kind][1] == "c":
        tf = g.faces(1)
        tm = tf[:-1].reshape(1, -1, 1)
        tp = tf[1:].reshape(1, -1, 1)
    else:
        tc = g.centres(1)
        tm = np.concatenate([[np.nan], tc]).reshape(1, -1, 1)
        tp = np.concatenate([tc, [np.nan]]).reshape(1, -1, 1)
    shp = g.shape(kind)
    am = np.broadcast_to(coef * np.sin(tm) / (rho2 * np.sin(th) * g.dth ** 2), shp).copy()
    ap = np.broadcast_to(coef * np.sin(tp) / (rho2 * np.sin(th) * g.dth ** 2), shp).copy()
    a0 = -am - ap
    return am, a0, ap


def _lap_ph(g: Grid, kind: str, coef: float, hat: bool):
    """Delta_phph = d_phph/(r^2 sin^2 th); hat: 1/(R1^2 sin^2 th_1), th_1 = pi/4 - delta (RD31)."""
    shp = g.shape(kind)
    if hat:
        c = coef / (g.R1 ** 2 * np.sin(g.theta1) ** 2 * g.dph ** 2)
        am = np.full(shp, c)
    else:
        rn = g.bcast(kind, 0)
        th = g.bcast(kind, 1)
        am = np.broadcast_to(coef / (rn ** 2 * np.sin(th) ** 2 * g.dph ** 2), shp).copy()
    ap = am.copy()
    a0 = -2.0 * am
    return am, a0, ap


def _adv(g: Grid, kind: str, axis: int, abar):
    """-abar_d * (centred first derivative along d with its metric factor):
    r: d_r; theta: d_th / r; phi: d_ph / (r sin th)  (RD15/RD16)."""
    rn = g.bcast(kind, 0)
    th = g.bcast(kind, 1)
    if axis == 0:
        m = 1.0 / (2 * g.dr)
    elif axis == 1:
        m = 1.0 / (2 * rn * g.dth)
    else:
        m = 1.0 / (2 * rn * np.sin(th) * g.dph)
    c = np.broadcast_to(abar * m, g.shape(kind))
    return c.copy(), np.zeros(g.shape(kind)), -c


def _add(*ops):
    am = sum(o[0] for o in ops)
    a0 = sum(o[1] for o in ops)
    ap = sum(o[2] for o in ops)
    return am, a0, ap


def abar(g: Grid, astar, kind: str, axis: int):
    """Component `axis` of the transport velocity a* = u2^{*,n+1/2} averaged to
    the nodes of `kind` (RD8, Appendix A)."""
    src = ("R", "TH", "PH")[axis]
    return to_kind(astar[axis], src, kind)


def coeffs(g: Grid, prm: Params, q: str, axis: int, hat: bool, astar):
    """Three-point weights (am, a0, ap) of the directional operator L_{q,axis}:
    (L X)[n] = am X[n - e_axis] + a0 X[n] + ap X[n + e_axis].

    T   (eq:Convect_Douglas; RD6-RD8):
        L_r = Drr - a_r d_r,  L_th = D^thth - a_th d_th/r,  L_ph = D^phph - a_ph d_ph/(r sin th)
    u_r (eq:r_comp; RD11):
        L_rr = nu(Drr u - 2u/r^2 + (2/r^3) d_r(r^2 u)) + c_chi D11 u - a_r d_r u
        L_rth = nu D^thth - a_th d_th/r,  L_rph = nu D^phph - a_ph d_ph/(r sin th)
    u_th (eq:theta_comp; RD13-RD15):
        L_thr = nu Drr - a_r d_r,  L_thph = nu D^phph - a_ph d_ph/(r sin th)
        L_thth = nu(D^thth u - u/(r^2 sin^2 th) + (2 cos th/(r^2 sin^2 th)) d_th(u sin th))
                 + c_chi D22 u - (a_th/r) d_th u - (a_r/r) u
    u_ph (eq:phi_comp; RD12, RD16):
        L_phr = nu Drr - a_r d_r,  L_phth = nu D^thth - a_th d_th/r
        L_phph = nu(D^phph u - u/(r^2 sin^2 th)) + c_chi D33 u - (a_ph/(r sin th)) d_ph u
                 - ((a_r + a_th cot th)/r) u
    `hat` selects D^ (split/implicit operators) vs the full Delta_thth /
    Delta_phph (the explicit L u^* on the right-hand side, RD10)."""
    kind = QKIND[q]
    coef = prm.kappa if q == "T" else prm.nu
    ab = abar(g, astar, kind, axis)
    if axis == 0:
        base = _add(_lap_r(g, kind, coef), _adv(g, kind, 0, ab))
    elif axis == 1:
        base = _add(_lap_th(g, kind, coef, hat), _adv(g, kind, 1, ab))
    else:
        base = _add(_lap_ph(g, kind, coef, hat), _adv(g, kind, 2, ab))
    am, a0, ap = (x.copy() for x in base)
    rn = g.bcast(kind, 0)
    th = g.bcast(kind, 1)
    shp = g.shape(kind)
    if q == "ur" and axis == 0:
        # metric: nu(-2u/r^2 + (2/r^3) d_r(r^2 u)), centred d_r on r-faces
        rf = g.faces(0)
        rfm = np.concatenate([[np.nan], rf[:-1]]).reshape(-1, 1, 1)
        rfp = np.concatenate([rf[1:], [np.nan]]).reshape(-1, 1, 1)
        a0 = a0 - prm.nu * 2.0 / rn ** 2
        ap = ap + prm.nu * 2.0 * rfp ** 2 / (rn ** 3 * 2 * g.dr)
        am = am - prm.nu * 2.0 * rfm ** 2 / (rn ** 3 * 2 * g.dr)
        # c_chi D11 = c_chi grad1(div1(.)), tridiagonal in r
        rc = g.centres(0)
        rcm = np.concatenate([[np.nan], rc]).reshape(-1, 1, 1)     # r_c(i-1)
        rcp = np.concatenate([rc, [np.nan]]).reshape(-1, 1, 1)     # r_c(i)
        ap = ap + prm.cchi * rfp ** 2 / (rcp ** 2 * g.dr ** 2)
        am = am + prm.cchi * rfm ** 2 / (rcm ** 2 * g.dr ** 2)
        a0 = a0 - prm.cchi * rn ** 2 * (1.0 / rcp ** 2 + 1.0 / rcm ** 2) / g.dr ** 2
    elif q == "ut" and axis == 1:
        st = np.sin(th)
        ct = np.cos(th)
        tc = g.centres(1)
        tcm = np.concatenate([[np.nan], tc]).reshape(1, -1, 1)   # th_c(j-1)
        tcp = np.concatenate([tc, [np.nan]]).reshape(1, -1, 1)   # th_c(j)
        tf = g.faces(1)
        tfm = np.concatenate([[np.nan], tf[:-1]]).reshape(1, -1, 1)
        tfp = np.concatenate([tf[1:], [np.nan]]).reshape(1, -1, 1)
        a0 = a0 - prm.nu / (rn ** 2 * st ** 2)
        k = prm.nu * 2.0 * ct / (rn ** 2 * st ** 2 * 2 * g.dth)
        ap = ap + k * np.sin(tfp)
        am = am - k * np.sin(tfm)
        # c_chi D22 = c_chi grad2(div2(.))
        ap = ap + prm.cchi * np.sin(tfp) / (rn ** 2 * np.sin(tcp) * g.dth ** 2)
        am = am + prm.cchi * np.sin(tfm) / (rn ** 2 * np.sin(tcm) * g.dth ** 2)
        a0 = a0 - prm.cchi * st * (1.0 / np.sin(tcp) + 1.0 / np.sin(tcm)) / (rn ** 2 * g.dth ** 2)
        a0 = a0 - abar(g, astar, "TH", 0) / rn
    elif q == "up" and axis == 2:
        st = np.sin(th)
        ct = np.cos(th)
        a0 = a0 - prm.nu / (rn ** 2 * st ** 2)
        c = prm.cchi / (rn ** 2 * st ** 2 * g.dph ** 2)
        ap = ap + c
        am = am + c
        a0 = a0 - 2 * c
        a0 = a0 - (abar(g, astar, "PH", 0) + abar(g, astar, "PH", 1) * ct / st) / rn
    return (np.broadcast_to(am, shp).copy(), np.broadcast_to(a0, shp).copy(),
            np.broadcast_to(ap, shp).copy())


def apply_dir(g: Grid, q: str, X: np.ndarray, axis: int, w, wall=None) -> np.ndarray:
    """(L_{q,axis} X) with weights w = (am, a0, ap).  Missing neighbours are NaN,
    except the r-neighbours of an r-centred field, which use the wall ghost of
    `wall` = (w_lo, w_hi) (RD22)."""
    kind = QKIND[q]
    if axis == 0 and kind in CENTRED_R:
        Xm = shift_r_ghost(X, -1, wall)
        Xp = shift_r_ghost(X, +1, wall)
    else:
        Xm = shift(X, axis, -1)
        Xp = shift(X, axis, +1)
    am, a0, ap = w
    # 0 * NaN would poison nodes whose weight is exactly zero; only the
    # neighbours a row really uses are read.
    return am * Xm + a0 * X + ap * Xp


FACTOR_ORDER = {"T": (0, 1, 2), "ur": (1, 2, 0), "ut": (2, 0, 1), "up": (0, 1, 2)}
"""Printed factor orders (RD28): T r,th,ph (eq:Convect_Douglas); u_r th,ph,r
(eq:r_comp P:L399-401); u_th ph,r,th (eq:theta_comp P:L423-425); u_ph r,th,ph
(eq:phi_comp P:L447-449).  The first factor is solved first (P:L461-472)."""

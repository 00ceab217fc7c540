"""Chart geometry, MAC node placement and Yin<->Yang interpolation stencils.

PAPER.md §2 (L118-146): Yin chart x = r sin(th) cos(ph), y = r sin(th) sin(ph),
z = r cos(th); Yang chart x = -r sin(th) cos(ph), y = r cos(th),
z = r sin(th) sin(ph); both cover the same coordinate box.  The printed box is
garbled (RD1); we take th in [pi/4 - d, 3pi/4 + d], ph in [-3pi/4 - d, 3pi/4 + d]
with the overlap d = 2 theta-cells and cell counts covering the extended patch
(RD2).  MAC staggering: scalars at cell centres, velocity
components on their own faces.

Fringe (RD3): the outermost theta/phi node layer of every staggered array holds
Dirichlet data interpolated from the other patch with 4x4 Lagrange in the
donor's own (theta, phi) lattice at the same r index (RD4), vectors rotated by
M_ab = e_a . e~_b (RD5).
"""
from __future__ import annotations

import math

import numpy as np

# staggering per axis (r, theta, phi): c = cell centre, f = face
KINDS = {"C": "ccc", "R": "fcc", "TH": "cfc", "PH": "ccf"}


class Grid:
    """One patch's MAC grid (both patches use identical arrays)."""

    def __init__(self, nr: int, nth: int, nph: int, R1: float = 1.0, R2: float = 2.0):
        if nr < 2 or nth < 8 or nph < 8 or not (0 < R1 < R2):
            raise ValueError("grid too small or bad radii")
        self.nr, self.nth, self.nph, self.R1, self.R2 = nr, nth, nph, R1, R2
        self.dr = (R2 - R1) / nr
        self.dth = math.pi / (2 * (nth - 4))          # RD2
        self.delta = 2 * self.dth                       # overlap, 2 cells
        self.dph = (1.5 * math.pi + 2 * self.delta) / nph
        self.x0 = (R1, math.pi / 4 - self.delta, -0.75 * math.pi - self.delta)
        self.h = (self.dr, self.dth, self.dph)
        self.n = (nr, nth, nph)
        self.theta1 = math.pi / 4 - self.delta          # RD31: theta_1 of the hat phi-operator

    # ---- 1-D node coordinates --------------------------------------------------
    def centres(self, axis: int) -> np.ndarray:
        return self.x0[axis] + self.h[axis] * (np.arange(self.n[axis]) + 0.5)

    def faces(self, axis: int) -> np.ndarray:
        return self.x0[axis] + self.h[axis] * np.arange(self.n[axis] + 1)

    def coord(self, kind: str, axis: int) -> np.ndarray:
        return self.faces(axis) if KINDS[kind][axis] == "f" else self.centres(axis)

    def shape(self, kind: str):
        return tuple(self.n[a] + (1 if KINDS[kind][a] == "f" else 0) for a in range(3))

    def bcast(self, kind: str, axis: int) -> np.ndarray:
        """coordinate of `axis` broadcastable over the kind's 3-D shape."""
        c = self.coord(kind, axis)
        sh = [1, 1, 1]
        sh[axis] = len(c)
        return c.reshape(sh)

    # ---- node classes (RD3) ------------------------------------------------------
    def solved_mask(self, kind: str) -> np.ndarray:
        """Unknowns of the implicit solves: not fringe, and not a u_r wall face."""
        m = np.zeros(self.shape(kind), dtype=bool)
        nr, nt, npp = self.shape(kind)
        i0, i1 = (1, nr - 1) if kind == "R" else (0, nr)
        m[i0:i1, 1:nt - 1, 1:npp - 1] = True
        return m

    def fringe_nodes(self, kind: str):
        """(j, k) of the outermost theta/phi layer of a kind's array (RD3)."""
        _, nt, npp = self.shape(kind)
        out = []
        for j in range(nt):
            for k in range(npp):
                if j == 0 or j == nt - 1 or k == 0 or k == npp - 1:
                    out.append((j, k))
        return out

    def weights_omega(self, kind: str) -> np.ndarray:
        """w = r^2 sin(th) dr dth dph at each node's own (r, th) (A8, RD24)."""
        r = self.bcast(kind, 0)
        th = self.bcast(kind, 1)
        return np.broadcast_to(r * r * np.sin(th) * self.dr * self.dth * self.dph, self.shape(kind))


# ---- chart maps ---------------------------------------------
def yin_to_cart(r, th, ph):
    return r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph), r * np.cos(th)


def yang_to_cart(r, th, ph):
    return -r * np.sin(th) * np.cos(ph), r * np.cos(th), r * np.sin(th) * np.sin(ph)


def cart_to_yin(x, y, z):
    r = np.sqrt(x * x + y * y + z * z)
    return r, np.arccos(np.clip(z / r, -1, 1)), np.arctan2(y, x)


def cart_to_yang(x, y, z):
    r = np.sqrt(x * x + y * y + z * z)
    return r, np.arccos(np.clip(y / r, -1, 1)), np.arctan2(z, -x)


def other_chart(th, ph):
    """(th, ph) of one chart -> coordinates of the same point in the other chart.

    Yin -> Yang: push through Cartesian and invert the Yang map.  The map is an
    involution ('the coordinate transformations ... and its
    inverse ... are identical'), so the same function serves Yang -> Yin."""
    x, y, z = yin_to_cart(1.0, th, ph)
    _, tt, pp = cart_to_yang(x, y, z)
    return tt, pp


def yin_basis(th, ph):
    """Cartesian (e_theta, e_phi) of the Yin chart."""
    return ((np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), -np.sin(th)),
            (-np.sin(ph), np.cos(ph), 0.0 * ph))


def yang_basis(th, ph):
    """Cartesian (e_theta, e_phi) of the Yang chart (derivatives of yang_to_cart)."""
    return ((-np.cos(th) * np.cos(ph), -np.sin(th), np.cos(th) * np.sin(ph)),
            (np.sin(ph), 0.0 * ph, np.cos(ph)))


def rotation(th, ph):
    """M_ab = e_a(target, Yin chart at (th,ph)) . e~_b(donor, Yang chart at the
    mapped point) for a, b in (theta, phi) (RD5).  By the symmetry of the two
    charts the same matrix serves Yang targets with Yin donors."""
    tt, pp = other_chart(th, ph)
    et, ep = yin_basis(th, ph)
    ett, etp = yang_basis(tt, pp)
    dot = lambda a, b: a[0] * b[0] + a[1] * b[1] + a[2] * b[2]
    return np.array([[dot(et, ett), dot(et, etp)], [dot(ep, ett), dot(ep, etp)]])


# ---- Lagrange stencils (RD4, RD42) ---------------------------------------------
def lagrange4(s: float):
    """4-point Lagrange weights at fractional lattice index s.

    Stencil base = ceil(s) - 2 (RD42): nodes base..base+3, two on each side."""
    base = math.ceil(s) - 2
    xs = [base + a for a in range(4)]
    w = []
    for a in range(4):
        v = 1.0
        for b in range(4):
            if b != a:
                v *= (s - xs[b]) / (xs[a] - xs[b])
        w.append(v)
    return base, w


class Stencil:
    """Donor stencil of one fringe node from one donor lattice."""
    __slots__ = ("jb", "kb", "wt", "wp")

    def __init__(self, jb, kb, wt, wp):
        self.jb, self.kb, self.wt, self.wp = jb, kb, wt, wp


def build_stencil(grid: Grid, th_t: float, ph_t: float, donor_kind: str) -> Stencil:
    """Map target (th_t, ph_t) to the other chart and build the 4x4 stencil on
    the donor kind's (theta, phi) lattice.  Checks the stencil stays on donor
    solved nodes (never reads the donor's own fringe)."""
    tt, pp = other_chart(th_t, ph_t)
    st = (tt - grid.coord(donor_kind, 1)[0]) / grid.dth
    sp = (pp - grid.coord(donor_kind, 2)[0]) / grid.dph
    jb, wt = lagrange4(st)
    kb, wp = lagrange4(sp)
    _, nt, npp = grid.shape(donor_kind)
    if jb < 1 or jb + 3 > nt - 2 or kb < 1 or kb + 3 > npp - 2:
        raise ValueError(f"overlap too small: donor stencil ({jb},{kb}) touches the donor fringe")
    return Stencil(jb, kb, wt, wp)


class Exchange:
    """All fringe stencils of one grid (identical for both patch directions).

    Stencils are stored as arrays over the fringe entries so one interpolation
    is a plain gather: value[i, e] = sum_ab wt[e,a] wp[e,b] X[i, jb[e]+a, kb[e]+b]."""

    def __init__(self, grid: Grid):
        self.grid = grid
        self.scalar = {}          # kind C / R: (j, k, jb, kb, wt, wp) arrays
        for kind in ("C", "R"):
            th = grid.coord(kind, 1)
            ph = grid.coord(kind, 2)
            nodes = grid.fringe_nodes(kind)
            sts = [build_stencil(grid, th[j], ph[k], kind) for (j, k) in nodes]
            self.scalar[kind] = self._pack(nodes, sts)
        self.vector = {}          # kind TH / PH: (j, k, stencil_TH, stencil_PH, M row)
        for kind, row in (("TH", 0), ("PH", 1)):
            th = grid.coord(kind, 1)
            ph = grid.coord(kind, 2)
            nodes = grid.fringe_nodes(kind)
            s_t = [build_stencil(grid, th[j], ph[k], "TH") for (j, k) in nodes]
            s_p = [build_stencil(grid, th[j], ph[k], "PH") for (j, k) in nodes]
            M = np.array([rotation(th[j], ph[k])[row] for (j, k) in nodes])
            self.vector[kind] = (self._pack(nodes, s_t), self._pack(nodes, s_p), M)

    @staticmethod
    def _pack(nodes, sts):
        j = np.array([n[0] for n in nodes])
        k = np.array([n[1] for n in nodes])
        jb = np.array([s.jb for s in sts])
        kb = np.array([s.kb for s in sts])
        wt = np.array([s.wt for s in sts])
        wp = np.array([s.wp for s in sts])
        return j, k, jb, kb, wt, wp

    @staticmethod
    def apply(pk, X: np.ndarray) -> np.ndarray:
        """Lagrange interpolation of X at every fringe entry, every r index: (nr, ne)."""
        _, _, jb, kb, wt, wp = pk
        out = np.zeros((X.shape[0], len(jb)))
        for a in range(4):
            for b in range(4):
                out = out + (wt[:, a] * wp[:, b])[None, :] * X[:, jb + a, kb + b]
        return out

    def fill_scalar(self, kind: str, target: np.ndarray, donor: np.ndarray):
        """Alg. 1 steps 1/7: fringe of a scalar-like field."""
        pk = self.scalar[kind]
        target[:, pk[0], pk[1]] = self.apply(pk, donor)

    def fill_vector(self, t_ut, t_up, d_ut, d_up):
        """Alg. 1 step 3: tangential components, rotated (RD5)."""
        for kind, tgt in (("TH", t_ut), ("PH", t_up)):
            pt, pp, M = self.vector[kind]
            tgt[:, pt[0], pt[1]] = M[:, 0][None, :] * self.apply(pt, d_ut) + M[:, 1][None, :] * self.apply(pp, d_up)

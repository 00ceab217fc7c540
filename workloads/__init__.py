"""Seeded synthetic inputs for the Yin-Yang AC direction-splitting step.

This module is shared by the oracle (``oracle/``), the CUDA path's tests and
``bench.py``.  It holds NONE of the method's arithmetic: no operator, no
sweep, no interpolation, no Schwarz logic.  It only

* names the BASELINE.json configurations C1-C5,
* places the MAC nodes of one chart (so closed forms can be sampled there),
* evaluates the two closed-form solutions the paper tests against
  (manufactured solution eq:Exact; Landau jet, L566-570)
  and the forcing that makes eq:Exact a solution (reading RD32),
* draws the seeded noise of C3 and the random operands of C4.

Every workload is returned as a plain dict of numpy float64 arrays, per patch
(0 = Yin, 1 = Yang), in the staggered shapes of include/yy.h:

    ur (Nr+1, Nth, Nph)   ut (Nr, Nth+1, Nph)   up (Nr, Nth, Nph+1)
    p, T (Nr, Nth, Nph)

Time-dependent wall data and sources are given as a list of
``(timefn, arrays)`` terms, value(t) = sum_m g_m(t) * arrays_m with
g in {1, cos t, sin t, cos^2 t} (SURVEY.md §8(b) "Units").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# time basis functions (must match YY_TF_* in include/yy.h)
TF_ONE, TF_COS, TF_SIN, TF_COS2 = 0, 1, 2, 3


def timefn(tf: int, t: float) -> float:
    """g_m(t) of the wall/source time basis (SURVEY.md §8(b) Units)."""
    if tf == TF_ONE:
        return 1.0
    if tf == TF_COS:
        return math.cos(t)
    if tf == TF_SIN:
        return math.sin(t)
    if tf == TF_COS2:
        return math.cos(t) ** 2
    raise ValueError(f"unknown time function {tf}")


@dataclass
class Config:
    """One workload: shell, grid per patch, physics, time stepping."""
    name: str
    nr: int
    nth: int
    nph: int
    R1: float = 1.0
    R2: float = 2.0
    Pr: float = 1.0
    Ra: float = 0.0
    dt: float = 1e-3
    steps: int = 1
    tol: float = 1e-10
    problem: str = "manufactured"      # manufactured | landau | convection
    # artificial-compressibility chi (eq:ac1).  The paper asks chi = O(1); on the
    # R2/R1 = 2 shell the fixed point of the step is stable only for chi >= beta =
    # R2^2 / (R1^2 sin^2 theta_1) (DESIGN.md RD-E4: Fourier model, oracle, C2 drift
    # on the GPU), beta = 8.3 (C5) ... 16 (C1): every BASELINE workload takes 16.
    chi: float = 16.0
    extra: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        """Cells per patch (SURVEY.md §8 notation)."""
        return self.nr * self.nth * self.nph


# BASELINE.json configs (SURVEY.md §8(d) "Synthetic inputs per BJ config").
def config(name: str, G: int = 1) -> Config:
    if name == "C1":
        return Config("C1", 16, 16, 48, Ra=100.0, dt=1e-3, steps=10, problem="manufactured")
    if name == "C2":
        return Config("C2", 48, 64, 192, Ra=0.0, dt=5e-4, steps=200, problem="landau")
    if name == "C3":
        return Config("C3", 96, 128, 384, Ra=1e4, dt=1e-4, steps=100, problem="convection")
    if name == "C5":
        # weak scaling: patch Nr = 64*G; G=1 holds both patches
        return Config("C5", 64 * G, 192, 576, Ra=1e5, dt=1e-4, steps=50, problem="manufactured")
    raise ValueError(name)


def small(name: str, nr: int, nth: int, nph: int, **kw) -> Config:
    """A reduced-size copy of a config (parity tests at oracle-friendly sizes)."""
    c = config(name)
    c.nr, c.nth, c.nph = nr, nth, nph
    for k, v in kw.items():
        setattr(c, k, v)
    return c


# ---------------------------------------------------------------------------
# node placement (reading RD1/RD2 of SURVEY.md: counts cover the extended patch)
# ---------------------------------------------------------------------------
KINDS = {"C": "ccc", "R": "fcc", "TH": "cfc", "PH": "ccf"}
FIELD_KIND = {"T": "C", "p": "C", "ur": "R", "ut": "TH", "up": "PH"}


def axes(cfg: Config):
    """(x0, h, n) per axis r, theta, phi: O1 of SURVEY.md §8(c)."""
    dr = (cfg.R2 - cfg.R1) / cfg.nr
    dth = math.pi / (2 * (cfg.nth - 4))
    delta = 2 * dth
    dph = (1.5 * math.pi + 2 * delta) / cfg.nph
    return ((cfg.R1, dr, cfg.nr), (math.pi / 4 - delta, dth, cfg.nth),
            (-0.75 * math.pi - delta, dph, cfg.nph))


def node_axes(cfg: Config, kind: str):
    """1-D node coordinates (r, theta, phi) of a staggering kind."""
    out = []
    for (x0, h, n), s in zip(axes(cfg), KINDS[kind]):
        if s == "f":
            out.append(x0 + h * np.arange(n + 1))
        else:
            out.append(x0 + h * (np.arange(n) + 0.5))
    return out


def chart_xyz(patch: int, r, th, ph):
    """Chart -> Cartesian: Yin patch 0, Yang patch 1."""
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    if patch == 0:
        return r * st * cp, r * st * sp, r * ct
    return -r * st * cp, r * ct, r * st * sp


def chart_basis(patch: int, th, ph):
    """Cartesian components of (e_r, e_theta, e_phi) of a chart at (th, ph)."""
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    z = np.zeros_like(st * sp)
    er = (st * cp, st * sp, ct + z)
    et = (ct * cp, ct * sp, -st + z)
    ep = (-sp + z, cp + z, z)
    if patch == 1:  # Yang = R . Yin with R(a,b,c) = (-a, c, b)
        er, et, ep = [(-v[0], v[2], v[1]) for v in (er, et, ep)]
    return er, et, ep


def node_grid(cfg: Config, patch: int, kind: str):
    """3-D broadcast arrays (r, th, ph, x, y, z, basis) at the nodes of a kind."""
    r1, t1, p1 = node_axes(cfg, kind)
    r = r1[:, None, None]
    th = t1[None, :, None]
    ph = p1[None, None, :]
    x, y, z = chart_xyz(patch, r, th, ph)
    shape = (len(r1), len(t1), len(p1))
    x, y, z = (np.broadcast_to(v, shape) for v in (x, y, z))
    basis = chart_basis(patch, th, ph)
    return r, th, ph, x, y, z, basis


def project(vec, basis_vec):
    return vec[0] * basis_vec[0] + vec[1] * basis_vec[1] + vec[2] * basis_vec[2]


# ---------------------------------------------------------------------------
# closed forms
# ---------------------------------------------------------------------------
def manufactured_U(x, y, z):
    """Spatial shape of u in eq:Exact: u = cos t * U."""
    return (2 * x * x * y * z, -x * y * y * z, -x * y * z * z)


def manufactured_P(x, y, z):
    return x * y * z


def manufactured_Theta(x, y, z):
    return 2 * x * x * y * z


def manufactured_forcing_terms(x, y, z, Pr, Ra):
    """f = u_t + (u.grad)u + grad p - Pr Lap u - Pr Ra T e_r and
    s = T_t + u.grad T - Lap T for eq:Exact (reading RD32, buoyancy RD20).

    Returned as {timefn: (fx, fy, fz, s)} with g in {sin t, cos^2 t, cos t}.
    Derivation: (U.grad)U = (4x^3y^2z^2, x^2y^3z^2, x^2y^2z^3),
    Lap U = (4yz, -2xz, -2xy), grad P = (yz, xz, xy), U.grad Theta = 4x^3y^2z^2,
    Lap Theta = 4yz.
    """
    U = manufactured_U(x, y, z)
    Th = manufactured_Theta(x, y, z)
    r = np.sqrt(x * x + y * y + z * z)
    adv = (4 * x**3 * y**2 * z**2, x**2 * y**3 * z**2, x**2 * y**2 * z**3)
    lapU = (4 * y * z, -2 * x * z, -2 * x * y)
    gradP = (y * z, x * z, x * y)
    erv = (x / r, y / r, z / r)
    f_sin = tuple(-U[c] for c in range(3))
    f_cos2 = adv
    f_cos = tuple(gradP[c] - Pr * lapU[c] - Pr * Ra * Th * erv[c] for c in range(3))
    s_sin = -Th
    s_cos2 = 4 * x**3 * y**2 * z**2
    s_cos = -4 * y * z
    return {TF_SIN: (*f_sin, s_sin), TF_COS2: (*f_cos2, s_cos2), TF_COS: (*f_cos, s_cos)}


LANDAU_A_F1 = 50.2880185645353   # a for jet force F = 1, rho = nu = 1


def landau_force(a: float, nu: float = 1.0, rho: float = 1.0) -> float:
    """Jet momentum flux F(a)."""
    return 16 * math.pi * rho * nu * nu * a * (
        1 + 4 / (3 * (a * a - 1)) - (a / 2) * math.log((a + 1) / (a - 1)))


def landau_a_for_force(F: float, nu: float = 1.0, rho: float = 1.0) -> float:
    """Invert F(a) by bisection (F decreasing in a on (1, inf))."""
    lo, hi = 1.0 + 1e-12, 1e8
    for _ in range(400):
        mid = math.sqrt(lo * hi)
        if landau_force(mid, nu, rho) > F:
            lo = mid
        else:
            hi = mid
    return math.sqrt(lo * hi)


def landau_uvp(x, y, z, axis, a: float, nu: float):
    """Landau jet in Cartesian form:
    u = u_R e_R - (2nu/r)(cos(Th) e_R - e)/(a - cos(Th)),
    u_R = (2nu/r)[(a^2-1)/(a-cos(Th))^2 - 1],
    p = 4 nu^2 (a cos(Th) - 1)/(r^2 (a - cos(Th))^2)   (rho = 1)."""
    r = np.sqrt(x * x + y * y + z * z)
    er = (x / r, y / r, z / r)
    c = (er[0] * axis[0] + er[1] * axis[1] + er[2] * axis[2])
    d = a - c
    uR = (2 * nu / r) * ((a * a - 1) / (d * d) - 1)
    u = tuple(uR * er[i] - (2 * nu / r) * (c * er[i] - axis[i]) / d for i in range(3))
    p = 4 * nu * nu * (a * c - 1) / (r * r * d * d)
    return u, p


def landau_axis(seed: int = 1905):
    v = np.random.Generator(np.random.PCG64(seed)).standard_normal(3)
    return tuple(v / np.linalg.norm(v))


# ---------------------------------------------------------------------------
# workload assembly
# ---------------------------------------------------------------------------
def _solved_mask_C(cfg: Config):
    m = np.zeros((cfg.nr, cfg.nth, cfg.nph), dtype=bool)
    m[:, 1:-1, 1:-1] = True
    return m


def _sample_vector(cfg, patch, fn):
    """Sample a Cartesian vector field fn(x,y,z) -> (vx,vy,vz) into (ur, ut, up)."""
    out = {}
    for name, kind, bi in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
        r, th, ph, x, y, z, basis = node_grid(cfg, patch, kind)
        v = fn(x, y, z)
        out[name] = np.ascontiguousarray(project(v, basis[bi]), dtype=np.float64)
    return out


def _sample_scalar(cfg, patch, fn, kind="C"):
    r, th, ph, x, y, z, basis = node_grid(cfg, patch, kind)
    return np.array(np.broadcast_to(fn(x, y, z), (len(r), th.shape[1], ph.shape[2])),
                    dtype=np.float64, order="C", copy=True)


def _sample_walls_vector(cfg, patch, fn):
    """Wall data of (ur, ut, up) at r = R1 and R2: arrays (2, n_th, n_ph)."""
    out = {}
    for name, kind, bi in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
        _, t1, p1 = node_axes(cfg, kind)
        th = t1[None, :, None]
        ph = p1[None, None, :]
        rw = np.array([cfg.R1, cfg.R2])[:, None, None]
        x, y, z = chart_xyz(patch, rw, th, ph)
        shape = (2, len(t1), len(p1))
        x, y, z = (np.broadcast_to(v, shape) for v in (x, y, z))
        basis = chart_basis(patch, th, ph)
        out[name] = np.ascontiguousarray(project(fn(x, y, z), basis[bi]), dtype=np.float64)
    return out


def _sample_walls_scalar(cfg, patch, fn):
    _, t1, p1 = node_axes(cfg, "C")
    th = t1[None, :, None]
    ph = p1[None, None, :]
    rw = np.array([cfg.R1, cfg.R2])[:, None, None]
    x, y, z = chart_xyz(patch, rw, th, ph)
    shape = (2, len(t1), len(p1))
    return np.array(np.broadcast_to(fn(*(np.broadcast_to(v, shape) for v in (x, y, z))), shape),
                    dtype=np.float64, order="C", copy=True)


def make_workload(cfg: Config):
    """Build the initial state, wall data and sources of a config.

    Returns {"cfg", "patches": [per-patch dict]} where each per-patch dict has
      "n":   {"ur","ut","up","p1","p2","T"}  level t^n   (t = 0)
      "nm1": {"ur","ut","up","T"}           level t^{n-1} (t = -dt)
      "walls":   [(timefn, {"T","ur","ut","up"} each (2, ., .))]
      "sources": [(timefn, {"T","ur","ut","up"} full 3-D)]
    and u1 = u2 at both levels (system 0 of yy_set_fields)."""
    patches = []
    for patch in range(2):
        if cfg.problem == "manufactured":
            patches.append(_manufactured(cfg, patch))
        elif cfg.problem == "landau":
            patches.append(_landau(cfg, patch))
        elif cfg.problem == "convection":
            patches.append(_convection(cfg, patch))
        elif cfg.problem == "heat":
            patches.append(_heat(cfg, patch))
        elif cfg.problem == "zero":
            patches.append(_zero(cfg, patch))
        else:
            raise ValueError(cfg.problem)
    return {"cfg": cfg, "patches": patches}


def _manufactured(cfg, patch):
    """eq:Exact at t=0 and t=-dt, walls cos t * exact, forcing (RD32, RD27).

    cfg.extra["amp"] (default 1) scales u, p and T of eq:Exact; the forcing is
    recomputed for the scaled fields (the advective terms scale with amp^2)."""
    A = cfg.extra.get("amp", 1.0)

    def lev(t):
        c = A * math.cos(t)
        v = _sample_vector(cfg, patch, lambda x, y, z: tuple(c * w for w in manufactured_U(x, y, z)))
        v["T"] = _sample_scalar(cfg, patch, lambda x, y, z: c * manufactured_Theta(x, y, z))
        return v
    n = lev(0.0)
    p = A * _sample_scalar(cfg, patch, manufactured_P)
    n["p1"] = p.copy()
    n["p2"] = p.copy()
    nm1 = lev(-cfg.dt)
    w = _sample_walls_vector(cfg, patch, lambda x, y, z: tuple(A * v for v in manufactured_U(x, y, z)))
    w["T"] = A * _sample_walls_scalar(cfg, patch, manufactured_Theta)
    walls = [(TF_COS, w)]
    sources = []
    scale = {TF_SIN: A, TF_COS2: A * A, TF_COS: A}
    for tf in (TF_SIN, TF_COS2, TF_COS):
        comp = {}
        for name, kind, bi in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
            r, th, ph, x, y, z, basis = node_grid(cfg, patch, kind)
            f = manufactured_forcing_terms(x, y, z, cfg.Pr, cfg.Ra)[tf]
            comp[name] = np.ascontiguousarray(scale[tf] * project(f[:3], basis[bi]))
        r, th, ph, x, y, z, basis = node_grid(cfg, patch, "C")
        comp["T"] = np.ascontiguousarray(scale[tf] * manufactured_forcing_terms(x, y, z, cfg.Pr, cfg.Ra)[tf][3])
        sources.append((tf, comp))
    return {"n": n, "nm1": nm1, "walls": walls, "sources": sources}


def _landau(cfg, patch):
    """C2: Landau jet as both levels and wall data (basis ONE), T = 0, Ra = 0."""
    axis = tuple(cfg.extra.get("axis", landau_axis()))
    a = cfg.extra.get("a", LANDAU_A_F1)
    nu = cfg.Pr
    n = _sample_vector(cfg, patch, lambda x, y, z: landau_uvp(x, y, z, axis, a, nu)[0])
    n["T"] = np.zeros((cfg.nr, cfg.nth, cfg.nph))
    p = _sample_scalar(cfg, patch, lambda x, y, z: landau_uvp(x, y, z, axis, a, nu)[1])
    n["p1"] = p.copy()
    n["p2"] = p.copy()
    nm1 = {k: n[k].copy() for k in ("ur", "ut", "up", "T")}
    w = _sample_walls_vector(cfg, patch, lambda x, y, z: landau_uvp(x, y, z, axis, a, nu)[0])
    w["T"] = np.zeros((2, cfg.nth, cfg.nph))
    return {"n": n, "nm1": nm1, "walls": [(TF_ONE, w)], "sources": []}


def _convection(cfg, patch):
    """C3: T0 = 2/r - 1 (conductive, R1=1,R2=2) + N(0,1e-3) on solved nodes
    (PCG64(1905+patch)), u0 = 0 both levels, hydrostatic p (RD27)."""
    R1, R2 = cfg.R1, cfg.R2
    r, th, ph, x, y, z, basis = node_grid(cfg, patch, "C")
    shape = (cfg.nr, cfg.nth, cfg.nph)
    cond = np.broadcast_to((R1 * R2 / r - R1) / (R2 - R1), shape)
    T0 = np.array(cond, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(1905 + patch))
    noise = rng.normal(0.0, cfg.extra.get("noise", 1e-3), size=shape)
    m = _solved_mask_C(cfg)
    T0[m] += noise[m]
    # hydrostatic: dp/dr = Pr Ra T_cond  ->  p = Pr Ra (R1R2 ln r - R1 r)/(R2-R1) + c
    pc = cfg.Pr * cfg.Ra * (R1 * R2 * np.log(r) - R1 * r + R1) / (R2 - R1)
    p = np.ascontiguousarray(np.broadcast_to(pc, shape), dtype=np.float64)
    n = {"ur": np.zeros((cfg.nr + 1, cfg.nth, cfg.nph)), "ut": np.zeros((cfg.nr, cfg.nth + 1, cfg.nph)),
         "up": np.zeros((cfg.nr, cfg.nth, cfg.nph + 1)), "T": T0, "p1": p.copy(), "p2": p.copy()}
    nm1 = {k: n[k].copy() for k in ("ur", "ut", "up", "T")}
    wT = np.zeros((2, cfg.nth, cfg.nph))
    wT[0] = 1.0
    w = {"T": wT, "ur": np.zeros((2, cfg.nth, cfg.nph)), "ut": np.zeros((2, cfg.nth + 1, cfg.nph)),
         "up": np.zeros((2, cfg.nth, cfg.nph + 1))}
    return {"n": n, "nm1": nm1, "walls": [(TF_ONE, w)], "sources": []}


def _heat(cfg, patch):
    """Heat-only manufactured case (u = 0, p = 0, Ra = 0): T = cos t * Theta
    with s = T_t - Lap T = -sin t Theta - cos t 4yz (Lap Theta = 4yz)."""
    def lev(t):
        c = math.cos(t)
        return _sample_scalar(cfg, patch, lambda x, y, z: c * manufactured_Theta(x, y, z))
    zr = _zero(cfg, patch)
    zr["n"]["T"] = lev(0.0)
    zr["nm1"]["T"] = lev(-cfg.dt)
    w = {"T": _sample_walls_scalar(cfg, patch, manufactured_Theta)}
    zr["walls"] = [(TF_COS, w)]
    r, th, ph, x, y, z, basis = node_grid(cfg, patch, "C")
    zr["sources"] = [(TF_SIN, {"T": np.ascontiguousarray(-manufactured_Theta(x, y, z))}),
                     (TF_COS, {"T": np.ascontiguousarray(-4 * y * z + 0 * x)})]
    return zr


def _zero(cfg, patch):
    n = {"ur": np.zeros((cfg.nr + 1, cfg.nth, cfg.nph)), "ut": np.zeros((cfg.nr, cfg.nth + 1, cfg.nph)),
         "up": np.zeros((cfg.nr, cfg.nth, cfg.nph + 1)), "T": np.zeros((cfg.nr, cfg.nth, cfg.nph)),
         "p1": np.zeros((cfg.nr, cfg.nth, cfg.nph)), "p2": np.zeros((cfg.nr, cfg.nth, cfg.nph))}
    nm1 = {k: n[k].copy() for k in ("ur", "ut", "up", "T")}
    return {"n": n, "nm1": nm1, "walls": [], "sources": []}


def random_state(cfg: Config, seed: int, amp: float = 1.0):
    """Seeded random smooth-ish state for parity tests of a generic step:
    a manufactured workload plus uniform noise of amplitude amp*1e-3 on all
    level arrays (so every stencil coefficient and fringe value matters)."""
    wl = make_workload(cfg)
    rng = np.random.Generator(np.random.PCG64(seed))
    for pd in wl["patches"]:
        for lev in ("n", "nm1"):
            for k, v in pd[lev].items():
                v += amp * 1e-3 * rng.uniform(-1, 1, size=v.shape)
    return wl


def c4_inputs(nr=256, nth=384, nph=1152):
    """C4 kernel-only operands: a*_d ~ U[-1,1) (PCG64(1905)),
    RHS ~ U[-1,1) (PCG64(1906)), one patch."""
    g1 = np.random.Generator(np.random.PCG64(1905))
    g2 = np.random.Generator(np.random.PCG64(1906))
    a = {"ur": g1.uniform(-1, 1, (nr + 1, nth, nph)), "ut": g1.uniform(-1, 1, (nr, nth + 1, nph)),
         "up": g1.uniform(-1, 1, (nr, nth, nph + 1))}
    rhs = g2.uniform(-1, 1, (nr, nth, nph))
    return a, rhs

"""Pins of the oracle's MAC operators (oracle/ops.py and the explicit terms of
oracle/scheme.py) against the mathematics: every discrete operator applied to
a smooth closed-form field must reproduce the analytic spherical operator at
second order, and exactness cases must hold exactly.

The analytic references are computed in CARTESIAN form and projected on the
chart basis (workloads.chart_basis), so a wrong metric term, sign, index or a
transposed operand in the spherical discretisation fails (SURVEY §8(c) pins:
'MAC operators', RD10-RD17)."""
import math

import numpy as np
import pytest

import workloads as W
from oracle import ops
from oracle.grid import Grid
from oracle.scheme import Oracle


def _oracle(n, Pr=1.0, Ra=0.0, dt=1e-3):
    return Oracle(*n, 1.0, 2.0, Pr, Ra, dt)


def _set_state(o, cfg, patch, u1, u2, T, p1, p2, walls):
    """levels n and n-1 equal (delta psi = 0, psi^* = psi^n)."""
    s = o.state[patch]
    for lev in ("n", "nm1"):
        for q in ("ur", "ut", "up"):
            s[lev][q + "1"][...] = u1[q]
            s[lev][q + "2"][...] = u2[q]
        s[lev]["T"][...] = T
    s["n"]["p1"][...] = p1
    s["n"]["p2"][...] = p2
    s["walls"] = [(W.TF_ONE, walls)]
    s["sources"] = []


def _interior(o, kind):
    """solved nodes minus the first/last r node of r-centred kinds (the wall
    ghost is a first-order closure of the second derivative there, RD22)."""
    m = o.g.solved_mask(kind).copy()
    if kind != "R":
        m[0] = False
        m[-1] = False
    return m


def _cart_vec(cfg, patch, fn, kind, comp):
    r, th, ph, x, y, z, basis = W.node_grid(cfg, patch, kind)
    return W.project(fn(x, y, z), basis[comp])


def _run_case(n, setup, check):
    o = _oracle(n)
    cfg = W.Config("x", *n)
    setup(o, cfg)
    astar, G = o.static(0, 0.0)
    return check(o, cfg, astar, G)


def _order(errs):
    return math.log2(errs[0] / errs[1])


GRIDS = [(8, 20, 52), (16, 36, 100)]
ZEROV = None


def _zeros(cfg):
    g = Grid(cfg.nr, cfg.nth, cfg.nph)
    return {"ur": np.zeros(g.shape("R")), "ut": np.zeros(g.shape("TH")), "up": np.zeros(g.shape("PH"))}


def test_constants_exact():
    # Delta of a constant is 0 exactly in flux form; grad of a constant p is 0
    o = _oracle((6, 14, 36))
    g = o.g
    astar = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    for q, kind in (("T", "C"), ("ut", "TH"), ("up", "PH")):
        X = np.full(g.shape(kind), 3.7)
        for axis in range(3):
            w = ops.coeffs(g, o.prm, q, axis, True, astar)
            if q != "T":   # velocity rows carry metric reaction terms; use the pure Laplacian rows
                continue
            Y = ops.apply_dir(g, q, X, axis, w, (np.full(X.shape[1:], 3.7),) * 2)
            assert np.max(np.abs(Y[g.solved_mask(kind)])) < 1e-9
    c = np.full(g.shape("C"), 2.5)
    for gr in (ops.grad1, ops.grad2, ops.grad3):
        v = gr(g, c)
        assert np.nanmax(np.abs(v)) == 0.0


def test_div_of_radial_inverse_square_exact():
    # div(u_r = 1/r^2) = 0 to machine precision
    g = Grid(6, 14, 36)
    ur = np.broadcast_to(1.0 / g.bcast("R", 0) ** 2, g.shape("R")).copy()
    d = ops.div(g, ur, np.zeros(g.shape("TH")), np.zeros(g.shape("PH")))
    assert np.max(np.abs(d)) < 1e-14


def test_laplacian_of_r2_is_6():
    # Delta(r^2) = 6, flux form: exact up to O(dr^2/r^2) at every node
    o = _oracle((8, 14, 36))
    g = o.g
    astar = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    X = np.broadcast_to(g.bcast("C", 0) ** 2, g.shape("C")).copy()
    wall = (np.full(g.shape("C")[1:], 1.0), np.full(g.shape("C")[1:], 4.0))
    Y = sum(ops.apply_dir(g, "T", X, a, ops.coeffs(g, o.prm, "T", a, False, astar), wall) for a in range(3))
    m = _interior(o, "C")
    assert np.max(np.abs(Y[m] - 6.0)) < 0.6 * g.dr ** 2


def _viscous(n):
    """nu * (vector Laplacian) of the manufactured U (div-free) through the
    oracle's implicit rows + explicit couplings; a* = 0, c_chi = 0."""
    o = _oracle(n)
    o.prm.cchi = 0.0
    cfg = W.Config("x", *n)
    U = W._sample_vector(cfg, 0, W.manufactured_U)
    Th = W._sample_scalar(cfg, 0, W.manufactured_Theta)
    walls = W._sample_walls_vector(cfg, 0, W.manufactured_U)
    walls["T"] = W._sample_walls_scalar(cfg, 0, W.manufactured_Theta)
    z = np.zeros(o.g.shape("C"))
    _set_state(o, cfg, 0, U, _zeros(cfg), Th, z, z, walls)
    astar, G = o.static(0, 0.0)
    tau = o.prm.dt
    cur = {"T": Th, "p1": z, "ur1": U["ur"], "ut1": U["ut"], "up1": U["up"]}
    lapU = lambda x, y, zz: (4 * y * zz, -2 * x * zz, -2 * x * y)
    errs = {}
    for q, kind, comp in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
        val = G[q + "1"] / tau
        if q != "ur":
            val = val + o.edyn(0, q, 1, cur, astar)
        ref = _cart_vec(cfg, 0, lapU, kind, comp)
        m = _interior(o, kind)
        errs[q] = np.max(np.abs(val - ref)[m])
    m = _interior(o, "C")
    errs["T"] = np.max(np.abs(G["T"] / tau - W._sample_scalar(cfg, 0, lambda x, y, zz: 4 * y * zz))[m])
    return errs


def test_vector_laplacian_second_order():
    e = [_viscous(n) for n in GRIDS]
    for q in ("ur", "ut", "up", "T"):
        assert e[1][q] < 0.1 * max(1.0, 1.0), (q, e)
        assert _order([e[0][q], e[1][q]]) > 1.7, (q, e)


def _advection(n):
    """-(U.grad)U and -U.grad(Theta) through the oracle's advective rows and
    explicit nonlinear terms (RD14-RD17), nu = kappa = 0, c_chi = 0, a* = U."""
    o = _oracle(n)
    o.prm.cchi = 0.0
    o.prm.nu = 0.0
    o.prm.kappa = 0.0
    cfg = W.Config("x", *n)
    U = W._sample_vector(cfg, 0, W.manufactured_U)
    Th = W._sample_scalar(cfg, 0, W.manufactured_Theta)
    walls = W._sample_walls_vector(cfg, 0, W.manufactured_U)
    walls["T"] = W._sample_walls_scalar(cfg, 0, W.manufactured_Theta)
    z = np.zeros(o.g.shape("C"))
    _set_state(o, cfg, 0, U, U, Th, z, z, walls)
    astar, G = o.static(0, 0.0)
    tau = o.prm.dt
    adv = lambda x, y, zz: (-4 * x**3 * y**2 * zz**2, -x**2 * y**3 * zz**2, -x**2 * y**2 * zz**3)
    errs = {}
    for q, kind, comp in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
        ref = _cart_vec(cfg, 0, adv, kind, comp)
        m = _interior(o, kind)
        errs[q] = np.max(np.abs(G[q + "1"] / tau - ref)[m]) / np.max(np.abs(ref[m]))
    ref = W._sample_scalar(cfg, 0, lambda x, y, zz: -4 * x**3 * y**2 * zz**2)
    m = _interior(o, "C")
    errs["T"] = np.max(np.abs(G["T"] / tau - ref)[m]) / np.max(np.abs(ref[m]))
    return errs


def test_advection_second_order():
    e = [_advection(n) for n in GRIDS]
    for q in ("ur", "ut", "up", "T"):
        assert e[1][q] < 0.02, (q, e)
        assert _order([e[0][q], e[1][q]]) > 1.7, (q, e)


def _graddiv_and_pressure(n):
    """c_chi grad(div u) for the gradient field u = grad(x^2 y + z^3) through
    D_ii (implicit rows) + D_ij (explicit, Gauss-Seidel split P:L368-383), and
    -grad p for p = xyz; nu = 0, a* = 0."""
    o = _oracle(n)
    o.prm.nu = 0.0
    o.prm.kappa = 0.0
    o.prm.cchi = 1.0
    cfg = W.Config("x", *n)
    u = W._sample_vector(cfg, 0, lambda x, y, zz: (2 * x * y, x * x, 3 * zz * zz))
    walls = W._sample_walls_vector(cfg, 0, lambda x, y, zz: (2 * x * y, x * x, 3 * zz * zz))
    walls["T"] = np.zeros((2, cfg.nth, cfg.nph))
    P = W._sample_scalar(cfg, 0, W.manufactured_P)
    z = np.zeros(o.g.shape("C"))
    _set_state(o, cfg, 0, u, _zeros(cfg), z, P, P, walls)
    astar, G = o.static(0, 0.0)
    tau = o.prm.dt
    cur = {"T": z, "p1": P, "ur1": u["ur"], "ut1": u["ut"], "up1": u["up"]}
    ref_fn = lambda x, y, zz: (0 * x - y * zz, 2.0 + 0 * x - x * zz, 6.0 + 0 * x - x * y)
    errs = {}
    for q, kind, comp in (("ur", "R", 0), ("ut", "TH", 1), ("up", "PH", 2)):
        val = G[q + "1"] / tau
        if q != "ur":
            val = val + o.edyn(0, q, 1, cur, astar)
        ref = _cart_vec(cfg, 0, ref_fn, kind, comp)
        m = o.g.solved_mask(kind)
        errs[q] = np.max(np.abs(val - ref)[m])
    return errs


def test_graddiv_and_pressure_gradient_second_order():
    e = [_graddiv_and_pressure(n) for n in GRIDS]
    for q in ("ur", "ut", "up"):
        assert e[1][q] < 0.05, (q, e)
        assert _order([e[0][q], e[1][q]]) > 1.7, (q, e)


def test_buoyancy_sign():
    # +Pr Ra T e_r (RD20): hot fluid is pushed outwards
    o = _oracle((4, 12, 28), Ra=10.0)
    z = {k: np.zeros(o.g.shape(k)) for k in ("C", "R", "TH", "PH")}
    cur = {"T": np.ones(o.g.shape("C")), "ur1": z["R"]}
    o.state[0]["n"]["T"][...] = 1.0
    E = o.edyn(0, "ur", 1, cur, [z["R"], z["TH"], z["PH"]])
    assert np.allclose(E[1:-1], 10.0)


def test_hat_operators_commute():
    # Delta_rr, Delta^_thth, Delta^_phph with zero Dirichlet data commute exactly
    # (P:L212 'it is easy to check that ... commute')
    o = _oracle((7, 14, 30))
    g = o.g
    astar = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    rng = np.random.default_rng(5)
    m = g.solved_mask("C")
    f = np.where(m, rng.standard_normal(g.shape("C")), 0.0)
    zero = (np.zeros(g.shape("C")[1:]),) * 2

    def A(axis, X):
        Y = ops.apply_dir(g, "T", np.where(m, X, 0.0), axis, ops.coeffs(g, o.prm, "T", axis, True, astar), zero)
        return np.where(m, Y, 0.0)

    for a, b in ((0, 1), (0, 2), (1, 2)):
        d = A(a, A(b, f)) - A(b, A(a, f))
        assert np.max(np.abs(d)) < 1e-12 * np.max(np.abs(A(a, A(b, f))))


def test_hat_negative_and_dominant():
    # (-Delta^_d f, f)_omega >= 0 (eq:HeatStab2) and hat dominates full (eq:HeatStab1)
    o = _oracle((6, 14, 30))
    g = o.g
    astar = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    rng = np.random.default_rng(6)
    m = g.solved_mask("C")
    w = g.weights_omega("C")
    zero = (np.zeros(g.shape("C")[1:]),) * 2
    for _ in range(5):
        f = np.where(m, rng.standard_normal(g.shape("C")), 0.0)
        for axis in (1, 2):
            Lh = ops.apply_dir(g, "T", f, axis, ops.coeffs(g, o.prm, "T", axis, True, astar), zero)
            Lf = ops.apply_dir(g, "T", f, axis, ops.coeffs(g, o.prm, "T", axis, False, astar), zero)
            ih = -np.sum((w * Lh * f)[m])
            iF = -np.sum((w * Lf * f)[m])
            assert ih >= 0 and ih >= iF - 1e-10 * abs(iF)

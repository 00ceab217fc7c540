"""Pins of oracle/grid.py: chart maps, rotation of
tangential components (RD5), Lagrange stencils (RD4, RD42) and the fringe
exchange — against closed forms, worked examples and
exactness properties, never against the oracle itself."""
import math

import numpy as np
import pytest

import workloads as W
from oracle.grid import (Exchange, Grid, cart_to_yang, cart_to_yin, lagrange4, other_chart,
                         rotation, yang_basis, yang_to_cart, yin_basis, yin_to_cart)


def test_worked_examples():
    # S:L65-66
    assert np.allclose(yin_to_cart(1.0, math.pi / 2, 0.0), (1, 0, 0), atol=1e-16)
    assert np.allclose(yang_to_cart(1.0, math.pi / 2, math.pi / 2), (0, 0, 1), atol=1e-16)
    # Yin (2, pi/2, pi/4) -> Yang (2, pi/4, pi)
    r, t, p = cart_to_yang(*yin_to_cart(2.0, math.pi / 2, math.pi / 4))
    assert abs(r - 2) < 1e-15 and abs(t - math.pi / 4) < 1e-15 and abs(abs(p) - math.pi) < 1e-15


def test_round_trip_and_radius():
    rng = np.random.default_rng(1)
    th = rng.uniform(math.pi / 4, 3 * math.pi / 4, 10000)
    ph = rng.uniform(-0.75 * math.pi, 0.75 * math.pi, 10000)
    r = rng.uniform(1, 2, 10000)
    x, y, z = yin_to_cart(r, th, ph)
    assert np.max(np.abs(np.sqrt(x * x + y * y + z * z) - r)) < 1e-14
    tt, pp = other_chart(th, ph)
    t2, p2 = other_chart(tt, pp)           # involution
    assert np.max(np.abs(t2 - th)) < 1e-12 and np.max(np.abs(p2 - ph)) < 1e-12
    # the Yang coordinates really describe the same point
    xr, yr, zr = yang_to_cart(r, tt, pp)
    assert max(np.max(np.abs(xr - x)), np.max(np.abs(yr - y)), np.max(np.abs(zr - z))) < 1e-14


def test_coverage():
    # every direction is inside at least one chart box, delta = 0
    rng = np.random.default_rng(2)
    v = rng.standard_normal((3, 200000))
    v /= np.linalg.norm(v, axis=0)
    _, t1, p1 = cart_to_yin(*v)
    _, t2, p2 = cart_to_yang(*v)
    inside = lambda t, p: (t >= math.pi / 4) & (t <= 3 * math.pi / 4) & (np.abs(p) <= 0.75 * math.pi)
    assert np.all(inside(t1, p1) | inside(t2, p2))


def test_rotation_orthogonal_and_symmetric():
    rng = np.random.default_rng(3)
    for _ in range(200):
        th = rng.uniform(math.pi / 4 - 0.1, 3 * math.pi / 4 + 0.1)
        ph = rng.uniform(-0.75 * math.pi - 0.1, 0.75 * math.pi + 0.1)
        M = rotation(th, ph)
        assert np.allclose(M @ M.T, np.eye(2), atol=1e-14)
        assert abs(np.linalg.det(M) - 1) < 1e-14
        # Yang target with Yin donor, computed directly from the two bases
        tt, pp = other_chart(th, ph)
        ea, eb = yang_basis(th, ph)
        da, db = yin_basis(tt, pp)
        dot = lambda a, b: a[0] * b[0] + a[1] * b[1] + a[2] * b[2]
        M2 = np.array([[dot(ea, da), dot(ea, db)], [dot(eb, da), dot(eb, db)]])
        assert np.allclose(M, M2, atol=1e-14)


def test_lagrange_exact_on_cubics():
    rng = np.random.default_rng(4)
    for _ in range(100):
        s = rng.uniform(3, 20)
        base, w = lagrange4(s)
        assert abs(sum(w) - 1) < 1e-14
        assert base + 1 <= s <= base + 2
        c = rng.standard_normal(4)
        f = lambda x: c[0] + c[1] * x + c[2] * x * x + c[3] * x ** 3
        assert abs(sum(wi * f(base + a) for a, wi in enumerate(w)) - f(s)) < 1e-10 * (1 + abs(f(s)))
    base, w = lagrange4(7.0)     # target exactly on a node (RD42 tie rule)
    assert base == 5 and np.allclose(w, [0, 0, 1, 0], atol=0)


def test_grid_spacings_rd2():
    g = Grid(16, 16, 48)
    assert abs(g.dth - 0.1308997) < 1e-6 and abs(g.dph - 0.1090831) < 1e-6
    g = Grid(96, 128, 384)
    assert abs(g.dth - 0.012668) < 1e-6 and abs(g.dph - 0.012404) < 1e-6


@pytest.mark.parametrize("shape", [(4, 12, 28), (16, 16, 48), (48, 64, 192), (96, 128, 384)])
def test_stencils_stay_in_donor_interior(shape):
    Exchange(Grid(*shape))      # raises if any stencil touches the donor fringe


def test_exchange_cubic_exact_and_rigid_vector():
    g = Grid(3, 16, 44)
    ex = Exchange(g)
    # scalar: a field that is a cubic polynomial of the donor's own (th, ph) is
    # reproduced exactly at every fringe node (Lagrange exactness)
    th = g.coord("C", 1)[None, :, None]
    ph = g.coord("C", 2)[None, None, :]
    f = lambda t, p: 1 + 2 * t - t * t * p + 0.5 * p ** 3 + t ** 3
    donor = np.broadcast_to(f(th, ph), g.shape("C")).copy()
    tgt = np.zeros(g.shape("C"))
    ex.fill_scalar("C", tgt, donor)
    j, k = ex.scalar["C"][0], ex.scalar["C"][1]
    tt, pp = other_chart(g.coord("C", 1)[j], g.coord("C", 2)[k])
    assert np.max(np.abs(tgt[0, j, k] - f(tt, pp))) < 1e-11
    # vector: a rigid Cartesian field sampled in both charts is exchanged with
    # interpolation error only, errors shrink ~h^4
    errs = []
    for n in ((3, 16, 44), (3, 28, 80)):
        cfg = W.Config("x", *n)
        gg = Grid(*n)
        e = Exchange(gg)
        V = lambda x, y, z: (0.3 + 0 * x, -0.7 + 0 * x, 0.2 + 0 * x)
        s = [W._sample_vector(cfg, p, V) for p in range(2)]
        t_ut, t_up = np.zeros(gg.shape("TH")), np.zeros(gg.shape("PH"))
        e.fill_vector(t_ut, t_up, s[1]["ut"], s[1]["up"])
        m = ~gg.solved_mask("TH")
        m2 = ~gg.solved_mask("PH")
        errs.append(max(np.max(np.abs(t_ut - s[0]["ut"])[m]), np.max(np.abs(t_up - s[0]["up"])[m2])))
    assert errs[0] < 1e-3 and errs[1] < errs[0] / 8


def _box_volume(R1, R2, ta, tb, pa, pb):
    """int_{R1}^{R2} int_{ta}^{tb} int_{pa}^{pb} r^2 sin(th) dph dth dr (closed form)."""
    return (R2 ** 3 - R1 ** 3) / 3.0 * (math.cos(ta) - math.cos(tb)) * (pb - pa)


def test_weights_omega_midpoint_rule():
    # RD24 / P:L559-560 ("standard mid-point approximation to the L2 norm"): the
    # omega weights of one patch's cell centres are the midpoint rule for
    # int r^2 sin(th) dr dth dph over the patch box.  The midpoint sums have closed
    # forms (sum_i r_i^2 dr = (R2^3-R1^3)/3 - (R2-R1) dr^2/12 exactly; sum_j
    # sin(th_j) dth = (cos a - cos b) (dth/2)/sin(dth/2) exactly), so the weights
    # are pinned to rounding — a dropped r^2 or sin(th), a wrong cell width or a
    # half-cell node offset fails — and the sum converges to the box integral.
    # Over the full shell r in [1,2], th in [0,pi], ph in [0,2pi) the integral is
    # ||1||^2_omega = 28 pi / 3.
    assert abs(_box_volume(1.0, 2.0, 0.0, math.pi, 0.0, 2 * math.pi) - 28 * math.pi / 3) < 1e-13
    for n in (1, 2, 4):
        for R1, R2 in ((1.0, 2.0), (0.5, 3.0)):
            g = Grid(6 * n, 12 * n, 28 * n, R1, R2)
            S = float(np.sum(g.weights_omega("C")))
            ta, pa = g.x0[1], g.x0[2]
            tb, pb = ta + g.nth * g.dth, pa + g.nph * g.dph
            mid_r = (R2 ** 3 - R1 ** 3) / 3.0 - (R2 - R1) * g.dr ** 2 / 12.0
            mid_t = (math.cos(ta) - math.cos(tb)) * (0.5 * g.dth) / math.sin(0.5 * g.dth)
            assert abs(S - mid_r * mid_t * (pb - pa)) < 1e-13 * S
            exact = _box_volume(R1, R2, ta, tb, pa, pb)
            assert abs(S - exact) / exact < (g.dr / (R2 - R1)) ** 2 + g.dth ** 2
    # the other node kinds: nonnegative, and they integrate the same box at O(h)
    g = Grid(24, 48, 112, 1.0, 2.0)
    exact = _box_volume(1.0, 2.0, g.x0[1], g.x0[1] + g.nth * g.dth, g.x0[2], g.x0[2] + g.nph * g.dph)
    for kind in ("R", "TH", "PH"):
        w = g.weights_omega(kind)
        assert np.all(w >= 0)
        assert abs(float(np.sum(w)) - exact) / exact < 0.1

"""One time step of the second-order AC direction-splitting scheme on the
Yin-Yang shell, additive Schwarz with splitting-error reduction.

Follows SURVEY.md §8(c) O1-O12 (the readings RD1-RD42 of the garbled paper are
listed in DESIGN.md):

  O2  a* = u2^{*,n+1/2} = 1.5 u2^n - 0.5 u2^{n-1}
  O3  G_q = tau [L_full,q psi_q^* - 1/2 L_split,q (psi_q^n - psi_q^{n-1}) + E_static,q]
                                                             (eq:HeatDouglas P:L237-242, RD10)
  O4  psi^(0) = psi^n
  O5  each iteration k: fringe <- Lagrange interpolation of the other patch's
      psi^(k-1) (Alg.1 steps 1,3,7), walls at t_{n+1}
  O6  T:  R = G - (I - tau/2 L_split)(T~ - T^n);  (I-tau/2 A_r)(I-tau/2 A_th)(I-tau/2 A_ph) D = R
      T^(k) = T~ + D   (eq:er with the sign of RD9; staging P:L461-472)
  O7  system 1 u_r -> u_th -> u_ph (Gauss-Seidel), R adds tau E_dyn
  O8  p1^(k) = p1^n - (1/chi) div(1/2 (u1^(k) + u1^n))          (eq:nst_Mass1 P:L457)
  O9  system 2 with the extra -1/2 grad(p1^(k) - p1^n);
      p2^(k) = p2^n + (p1^(k) - p1^n) - (1/chi) div(1/2 (u2^(k) + u2^n))   (eq:ac2, RD18)
  O10 rho_k = max over 9 quantities x 2 patches of the omega-weighted l2 norm of
      psi^(k) - psi~^(k-1) on solved nodes; stop when rho_k < tol   (RD24)
  O11 rotate levels, t += tau.
"""
from __future__ import annotations

import copy
import math
import time

import numpy as np

from . import fluxfix, ops
from .grid import Exchange, Grid
from .ops import FACTOR_ORDER, QKIND, Params, to_kind
from .tridiag import thomas

VEC = ("ur", "ut", "up")
TF_ONE, TF_COS, TF_SIN, TF_COS2 = 0, 1, 2, 3


def g_of(tf: int, t: float) -> float:
    return {TF_ONE: 1.0, TF_COS: math.cos(t), TF_SIN: math.sin(t), TF_COS2: math.cos(t) ** 2}[tf]


class Oracle:
    """Both patches of one shell, stepped with plain numpy."""

    def __init__(self, nr, nth, nph, R1, R2, Pr, Ra, dt, chi=1.0, max_iters=100, fixed_iters=0,
                 factor_order=None, schwarz="additive", flux_fix_eps=None, advection="split"):
        self.g = Grid(nr, nth, nph, R1, R2)
        self.prm = Params(Pr, Ra, dt, chi)
        self.ex = Exchange(self.g)
        self.max_iters = max_iters
        self.fixed_iters = fixed_iters
        if schwarz not in ("additive", "multiplicative", "none"):
            raise ValueError(schwarz)
        # additive (RD26): both patches take the other's iterate k-1.  multiplicative
        # (Algorithm 1 as printed): Yin first with Yang's iterate k-1,
        # then Yang with Yin's fresh iterate k.  none: no exchange —
        # each patch is a single domain whose fringe keeps the Dirichlet values it
        # holds (Theorem 1's setting: one simply shaped domain).
        self.schwarz = schwarz
        # Algorithm 1 step 4 (optional in the paper): None = off
        self.flux_fix_eps = flux_fix_eps
        self.order = dict(FACTOR_ORDER) if factor_order is None else factor_order
        # where the linearised advection goes: "split" = inside the
        # direction-wise factors (the paper's scheme, eq:Convect_Douglas and
        # eq:r_comp..phi_comp); "imex" = the IMEX alternative: the
        # split operators are the a* = 0 rows (diffusion, metric, grad-div), the
        # transport terms (advection and the a*-reaction terms of RD14 / P:L444)
        # stay only in the explicit L_full psi^* of G (AB2-extrapolated)
        if advection not in ("split", "imex"):
            raise ValueError(advection)
        self.imex = advection == "imex"
        self.t = 0.0
        g = self.g
        z = lambda k: np.zeros(g.shape(k))
        self.state = []
        for _ in range(2):
            s = {"n": {"T": z("C"), "p1": z("C"), "p2": z("C")}, "nm1": {"T": z("C")}}
            for sysn in (1, 2):
                for q in VEC:
                    s["n"][f"{q}{sysn}"] = z(QKIND[q])
                    s["nm1"][f"{q}{sysn}"] = z(QKIND[q])
            s["walls"] = []
            s["sources"] = []
            self.state.append(s)
        self.stats = []   # (iterations, rho) per step
        self._cc = {}

    # ---- set / get (mirror include/yy.h semantics) -------------------------------
    def set_fields(self, patch, level, system, f):
        lev = self.state[patch]["n" if level == 0 else "nm1"]
        systems = (1, 2) if system == 0 else (system,)
        for q in VEC:
            if f.get(q) is not None:
                for s in systems:
                    lev[f"{q}{s}"][...] = f[q]
        if f.get("T") is not None:
            lev["T"][...] = f["T"]
        if level == 0 and f.get("p") is not None:
            for s in systems:
                lev[f"p{s}"][...] = f["p"]

    def get_fields(self, patch, level, system):
        lev = self.state[patch]["n" if level == 0 else "nm1"]
        out = {q: lev[f"{q}{system}"].copy() for q in VEC}
        out["T"] = lev["T"].copy()
        if level == 0:
            out["p"] = lev[f"p{system}"].copy()
        return out

    def set_wall_terms(self, patch, terms):
        self.state[patch]["walls"] = [(tf, {k: np.array(v, dtype=np.float64) for k, v in d.items()})
                                      for tf, d in terms]

    def set_source_terms(self, patch, terms):
        self.state[patch]["sources"] = [(tf, {k: np.array(v, dtype=np.float64) for k, v in d.items()})
                                        for tf, d in terms]

    def load_workload(self, wl):
        for patch, pd in enumerate(wl["patches"]):
            n = pd["n"]
            self.set_fields(patch, 0, 1, {"ur": n["ur"], "ut": n["ut"], "up": n["up"], "T": n["T"], "p": n["p1"]})
            self.set_fields(patch, 0, 2, {"ur": n["ur"], "ut": n["ut"], "up": n["up"], "p": n["p2"]})
            self.set_fields(patch, 1, 0, pd["nm1"])
            self.set_wall_terms(patch, pd["walls"])
            self.set_source_terms(patch, pd["sources"])

    # ---- wall data and sources at time t -----------------------------------------
    def wall(self, patch, name, t):
        g = self.g
        shp = (2,) + g.shape(QKIND[name])[1:]
        w = np.zeros(shp)
        for tf, d in self.state[patch]["walls"]:
            if name in d:
                w = w + g_of(tf, t) * d[name]
        return w

    def source(self, patch, name, t):
        w = np.zeros(self.g.shape(QKIND[name]))
        for tf, d in self.state[patch]["sources"]:
            if name in d:
                w = w + g_of(tf, t) * d[name]
        return w

    # ---- operator helpers -------------------------------------------------------
    def W(self, q, axis, hat, astar):
        """Directional weights, cached per step (a* is fixed for the whole step)."""
        key = (id(astar), q, axis, hat)
        if key not in self._cc:
            if hat and self.imex:
                a0 = [np.zeros(self.g.shape(k)) for k in ("R", "TH", "PH")]
                self._cc[key] = ops.coeffs(self.g, self.prm, q, axis, hat, a0)
            else:
                self._cc[key] = ops.coeffs(self.g, self.prm, q, axis, hat, astar)
        return self._cc[key]

    def L(self, q, X, W, hat, astar):
        """sum over the three directions of L_{q,d} X (full or split), wall ghost W."""
        out = 0.0
        for axis in range(3):
            out = out + ops.apply_dir(self.g, q, X, axis, self.W(q, axis, hat, astar), W)
        return out

    def solved(self, kind):
        g = self.g
        nr, nt, npp = g.shape(kind)
        i0, i1 = (1, nr - 1) if kind == "R" else (0, nr)
        return (slice(i0, i1), slice(1, nt - 1), slice(1, npp - 1))

    def sweep(self, q, R, axis, w):
        """Solve (I - tau/2 A_{q,axis}) Y = R on the solved block, homogeneous
        Dirichlet increments at fringe / u_r walls, antisymmetric ghost at the
        walls of r-centred fields (RD23)."""
        tau = self.prm.dt
        kind = QKIND[q]
        blk = self.solved(kind)
        am, a0, ap = (x[blk] for x in w)
        lo = -0.5 * tau * am
        di = 1.0 - 0.5 * tau * a0
        up = -0.5 * tau * ap
        if axis == 0 and kind in ops.CENTRED_R:
            di[0] = 1.0 - 0.5 * tau * (a0[0] - am[0])
            di[-1] = 1.0 - 0.5 * tau * (a0[-1] - ap[-1])
        mv = lambda x: np.moveaxis(x, axis, 0)
        Y = thomas(mv(lo), mv(di), mv(up), mv(R[blk]))
        out = np.zeros(self.g.shape(kind))
        out[blk] = np.moveaxis(Y, 0, axis)
        return out

    def wnorm2(self, kind, D):
        blk = self.solved(kind)
        return float(np.sum(self.g.weights_omega(kind)[blk] * D[blk] ** 2))

    # ---- static RHS (O2, O3) -----------------------------------------------------
    def static(self, patch, t):
        g, prm, s = self.g, self.prm, self.state[patch]
        tau = prm.dt
        n, m = s["n"], s["nm1"]
        astar = [1.5 * n[f"{q}2"] - 0.5 * m[f"{q}2"] for q in VEC]
        th = {}
        for name in ("T", "ut", "up"):
            wn, wm = self.wall(patch, name, t), self.wall(patch, name, t - tau)
            th[name] = (1.5 * wn - 0.5 * wm, wn - wm)
        th["ur"] = (None, None)
        src = {name: self.source(patch, name, t + 0.5 * tau) for name in ("T", "ur", "ut", "up")}
        G = {}
        # temperature (eq:Convect_Douglas with RD6-RD8)
        Ts = 1.5 * n["T"] - 0.5 * m["T"]
        dT = n["T"] - m["T"]
        G["T"] = tau * (self.L("T", Ts, th["T"][0], False, astar)
                        - 0.5 * self.L("T", dT, th["T"][1], True, astar) + src["T"])
        rf = g.bcast("R", 0)
        rc = g.bcast("TH", 0)
        tf = g.bcast("TH", 1)
        for sysn in (1, 2):
            us = {q: 1.5 * n[f"{q}{sysn}"] - 0.5 * m[f"{q}{sysn}"] for q in VEC}
            du = {q: n[f"{q}{sysn}"] - m[f"{q}{sysn}"] for q in VEC}
            p = n[f"p{sysn}"]
            # u_r (eq:r_comp; RD10, RD11, RD17)
            at_R = ops.abar(g, astar, "R", 1)
            ap_R = ops.abar(g, astar, "R", 2)
            E = (-ops.grad1(g, p)
                 + prm.cchi * ops.grad1(g, ops.div2(g, us["ut"]) + ops.div3(g, us["up"]))
                 + (at_R ** 2 + ap_R ** 2) / rf + src["ur"])
            G[f"ur{sysn}"] = tau * (self.L("ur", us["ur"], None, False, astar)
                                    - 0.5 * self.L("ur", du["ur"], None, True, astar) + E)
            # u_th (eq:theta_comp; RD13, RD14)
            ap_TH = ops.abar(g, astar, "TH", 2)
            E = (-ops.grad2(g, p) + prm.cchi * ops.grad2(g, ops.div3(g, us["up"]))
                 + ap_TH ** 2 * (np.cos(tf) / np.sin(tf)) / rc + src["ut"])
            G[f"ut{sysn}"] = tau * (self.L("ut", us["ut"], th["ut"][0], False, astar)
                                    - 0.5 * self.L("ut", du["ut"], th["ut"][1], True, astar) + E)
            # u_ph (eq:phi_comp)
            E = -ops.grad3(g, p) + src["up"]
            G[f"up{sysn}"] = tau * (self.L("up", us["up"], th["up"][0], False, astar)
                                    - 0.5 * self.L("up", du["up"], th["up"][1], True, astar) + E)
        return astar, G

    # ---- dynamic explicit terms (Gauss-Seidel) -----------------------
    def edyn(self, patch, q, sysn, cur, astar):
        g, prm, n = self.g, self.prm, self.state[patch]["n"]
        if q == "ur":
            # buoyancy +Pr Ra T^{n+1/2,(k)} e_r (RD20, RD21)
            E = prm.Pr * prm.Ra * to_kind(0.5 * (cur["T"] + n["T"]), "C", "R")
        else:
            ubr = 0.5 * (cur[f"ur{sysn}"] + n[f"ur{sysn}"])
            d1 = ops.div1(g, ubr)
            if q == "ut":
                r = g.bcast("TH", 0)
                th = g.bcast("TH", 1)
                dthur = np.full(g.shape("TH"), np.nan)     # (1/1) d_th u_r at (r_c, th_f)
                dd = (ubr[:, 1:] - ubr[:, :-1]) / g.dth       # at (r_f, th_f interior)
                dthur[:, 1:-1] = 0.5 * (dd[:-1] + dd[1:])
                E = (prm.cchi * ops.grad2(g, d1)
                     + prm.nu * (2.0 / r ** 2) * dthur
                     + prm.nu * (2.0 * np.cos(th) / (np.sin(th) * r)) * to_kind(d1, "C", "TH"))
            else:
                ubt = 0.5 * (cur[f"ut{sysn}"] + n[f"ut{sysn}"])
                r = g.bcast("PH", 0)
                th = g.bcast("PH", 1)
                dphur = np.full(g.shape("PH"), np.nan)
                dd = (ubr[:, :, 1:] - ubr[:, :, :-1]) / g.dph
                dphur[:, :, 1:-1] = 0.5 * (dd[:-1] + dd[1:])
                dphut = np.full(g.shape("PH"), np.nan)
                dd = (ubt[:, :, 1:] - ubt[:, :, :-1]) / g.dph
                dphut[:, :, 1:-1] = 0.5 * (dd[:, :-1] + dd[:, 1:])
                E = (prm.cchi * ops.grad3(g, d1 + ops.div2(g, ubt))
                     + prm.nu * (2.0 / (r ** 2 * np.sin(th))) * dphur
                     + prm.nu * (2.0 * np.cos(th) / (r ** 2 * np.sin(th) ** 2)) * dphut)
        if sysn == 2:
            dp1 = cur["p1"] - n["p1"]
            grad = {"ur": ops.grad1, "ut": ops.grad2, "up": ops.grad3}[q]
            E = E - 0.5 * grad(g, dp1)
        return E

    # ---- the step ------------------------------------------------------------------
    def step(self, nsteps=1, tol=1e-10):
        status = 0
        for _ in range(nsteps):
            k, rho = self._one_step(tol)
            self.stats.append((k, rho))
            if not self.fixed_iters and k >= self.max_iters and rho >= tol:
                status = 4
        return status

    def _one_step(self, tol):
        g, prm = self.g, self.prm
        tau = prm.dt
        t = self.t
        self._cc = {}
        # wall-clock of the static part and of every iteration (instrumentation
        # for bench.py's CPU baseline; no effect on the arithmetic)
        t0 = time.perf_counter()
        stat = [self.static(p, t) for p in range(2)]
        self.timing = {"static": time.perf_counter() - t0, "iters": []}
        t_it = time.perf_counter()
        cur = [copy.deepcopy(self.state[p]["n"]) for p in range(2)]
        wnew = [{name: self.wall(p, name, t + tau) for name in ("T", "ur", "ut", "up")} for p in range(2)]
        wdiff = [{name: wnew[p][name] - self.wall(p, name, t) for name in ("T", "ut", "up")} for p in range(2)]
        kmax = self.fixed_iters if self.fixed_iters else self.max_iters
        rows_r = np.arange(1, g.nr)
        rho = math.inf
        k = 0
        while k < kmax:
            k += 1
            if self.schwarz == "multiplicative":
                rho = 0.0
                for p in range(2):
                    self._fill_fringe(p, cur, wnew)
                    self._flux_fix(p, cur, tol)
                    rho = max(rho, self._iterate_patch(p, cur[p], stat[p], wdiff[p]))
                if not self.fixed_iters and rho < tol:
                    break
                continue
            if self.schwarz == "none":
                for p in range(2):
                    for s_ in (1, 2):
                        cur[p][f"ur{s_}"][0] = wnew[p]["ur"][0]
                        cur[p][f"ur{s_}"][-1] = wnew[p]["ur"][1]
                rho = 0.0
                for p in range(2):
                    rho = max(rho, self._iterate_patch(p, cur[p], stat[p], wdiff[p]))
                if not self.fixed_iters and rho < tol:
                    break
                continue
            # O5 (a): fringe of all 9 quantities from the other patch's iterate k-1
            fr = []
            for p in range(2):
                d = cur[1 - p]
                vals = {}
                for name in ("T", "p1", "p2"):
                    tgt = d[name].copy()
                    self.ex.fill_scalar("C", tgt, d[name])
                    vals[name] = tgt
                for s in (1, 2):
                    tgt = d[f"ur{s}"].copy()
                    self.ex.fill_scalar("R", tgt, d[f"ur{s}"])
                    vals[f"ur{s}"] = tgt
                    tt, tp = d[f"ut{s}"].copy(), d[f"up{s}"].copy()
                    self.ex.fill_vector(tt, tp, d[f"ut{s}"], d[f"up{s}"])
                    vals[f"ut{s}"], vals[f"up{s}"] = tt, tp
                fr.append(vals)
            for p in range(2):
                for name, v in fr[p].items():
                    kind = QKIND[name.rstrip("12")]
                    mask = ~self.g.solved_mask(kind)
                    if kind == "R":
                        mask[0] = False
                        mask[-1] = False
                    cur[p][name][mask] = v[mask]
                # O5 (b): u_r wall faces at t_{n+1}
                for s in (1, 2):
                    cur[p][f"ur{s}"][0] = wnew[p]["ur"][0]
                    cur[p][f"ur{s}"][-1] = wnew[p]["ur"][1]
            for p in range(2):
                self._flux_fix(p, cur, tol)
            rho = 0.0
            for p in range(2):
                rho = max(rho, self._iterate_patch(p, cur[p], stat[p], wdiff[p]))
            now = time.perf_counter()
            self.timing["iters"].append(now - t_it)
            t_it = now
            if not self.fixed_iters and rho < tol:
                break
        for p in range(2):
            s = self.state[p]
            s["nm1"] = {kk: s["n"][kk] for kk in s["nm1"]}
            s["n"] = cur[p]
        self.t = t + tau
        return k, rho

    def _fill_fringe(self, p, cur, wnew):
        """O5 for patch p alone: its fringe of all 9 quantities from the other
        patch's current iterate, and its u_r wall faces at t_{n+1} (multiplicative
        Schwarz, Algorithm 1 steps 1/3/7 in patch order)."""
        d = cur[1 - p]
        for name in ("T", "p1", "p2"):
            tgt = d[name].copy()
            self.ex.fill_scalar("C", tgt, d[name])
            self._set_fringe(p, cur, name, tgt)
        for s in (1, 2):
            tgt = d[f"ur{s}"].copy()
            self.ex.fill_scalar("R", tgt, d[f"ur{s}"])
            self._set_fringe(p, cur, f"ur{s}", tgt)
            tt, tp = d[f"ut{s}"].copy(), d[f"up{s}"].copy()
            self.ex.fill_vector(tt, tp, d[f"ut{s}"], d[f"up{s}"])
            self._set_fringe(p, cur, f"ut{s}", tt)
            self._set_fringe(p, cur, f"up{s}", tp)
        for s in (1, 2):
            cur[p][f"ur{s}"][0] = wnew[p]["ur"][0]
            cur[p][f"ur{s}"][-1] = wnew[p]["ur"][1]

    def _flux_fix(self, p, cur, tol):
        """Algorithm 1 step 4 on both systems' interpolated velocities of patch p."""
        if self.flux_fix_eps is None:
            return
        for s in (1, 2):
            fluxfix.flux_fix(self.g, cur[p][f"ur{s}"], cur[p][f"ut{s}"], cur[p][f"up{s}"], tol, self.flux_fix_eps)

    def _set_fringe(self, p, cur, name, v):
        kind = QKIND[name.rstrip("12")]
        mask = ~self.g.solved_mask(kind)
        if kind == "R":
            mask[0] = False
            mask[-1] = False
        cur[p][name][mask] = v[mask]

    def _solve(self, p, q, name, R, astar, cur):
        for axis in self.order[q]:
            R = self.sweep(q, R, axis, self.W(q, axis, True, astar))
        kind = QKIND[q]
        blk = self.solved(kind)
        new = cur[name].copy()
        new[blk] = cur[name][blk] + R[blk]
        return new, self.wnorm2(kind, R)

    def _iterate_patch(self, p, cur, stat, wdiff):
        prm = self.prm
        tau = prm.dt
        astar, G = stat
        n = self.state[p]["n"]
        worst = 0.0
        # T (O6)
        X = cur["T"] - n["T"]
        R = G["T"] - (X - 0.5 * tau * self.L("T", X, wdiff["T"], True, astar))
        cur["T"], nn = self._solve(p, "T", "T", R, astar, cur)
        worst = max(worst, nn)
        for sysn in (1, 2):
            for q in VEC:
                name = f"{q}{sysn}"
                X = cur[name] - n[name]
                W = None if q == "ur" else wdiff[q]
                R = (G[name] + tau * self.edyn(p, q, sysn, cur, astar)
                     - (X - 0.5 * tau * self.L(q, X, W, True, astar)))
                cur[name], nn = self._solve(p, q, name, R, astar, cur)
                worst = max(worst, nn)
            # pressure (O8 / O9)
            ub = [0.5 * (cur[f"{q}{sysn}"] + n[f"{q}{sysn}"]) for q in VEC]
            dv = ops.div(self.g, *ub)
            blk = self.solved("C")
            newp = cur[f"p{sysn}"].copy()
            if sysn == 1:
                newp[blk] = n["p1"][blk] - dv[blk] / prm.chi
            else:
                newp[blk] = (n["p2"][blk] + (cur["p1"][blk] - n["p1"][blk]) - dv[blk] / prm.chi)
            worst = max(worst, self.wnorm2("C", newp - cur[f"p{sysn}"]))
            cur[f"p{sysn}"] = newp
        return math.sqrt(worst)

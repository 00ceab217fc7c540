"""The discrete energy of Theorem 1 (eq:Stability) for the
heat-only Douglas scheme eq:HeatDouglas on ONE patch with
homogeneous Dirichlet data (the theorem's single simply shaped domain).

Test infrastructure only (see oracle/__init__.py): never imported by the
product path.

With a = dT^{n+1} = T^{n+1} - T^n, b = dT^n, the proof of Theorem 1 multiplies
eq:StabProof2 by a.  Rearranged from eq:HeatDouglas the second term is
-1/2 (Lh - L)(T^{n+1} - 2T^n + T^{n-1}) (the printed [L - Lh] has the opposite
sign; reading RD-E6), Lh - L <= 0 by eq:HeatStab1, so with the weight norm
||v||^2_D := -((Lh - L) v, v)_omega >= 0 (the omega_1 / omega_2 terms, with the
positive weight of RD34) the identity reads

  ||a||^2_omega / tau + E(T^{n+1}, a) - E(T^n, b) + 1/4 ||a - b||^2_D + diss = 0,
  E(T, d) = 1/2 (-L T, T)_omega + 1/4 ||d||^2_D,

diss >= 0 the eq:StabProof5-8 terms.  Hence the left side of eq:Stability,

  S_N = tau sum_{n=1}^{N-1} ||dT^{n+1} / tau||^2_omega + E(T^N, dT^N),

is non-increasing in N.  The discrete operators are the oracle's own rows
(ops.coeffs, full L and hat Lh), the inner product the midpoint rule of RD24 over
the solved cell centres, so the identity holds to rounding when the discrete L,
Lh are omega-symmetric (flux forms, RD30) and the boundary data are zero.
"""
from __future__ import annotations

import numpy as np

from . import ops


def stability_terms(o, patch: int):
    """(1/2 (-L T^n, T^n)_w, 1/4 ||dT^n||^2_D, ||dT^n||^2_w) of one patch of an
    Oracle with u = 0 (the T rows are then pure diffusion)."""
    g = o.g
    s = o.state[patch]
    Tn, Tm = s["n"]["T"], s["nm1"]["T"]
    astar = [np.zeros(g.shape(k)) for k in ("R", "TH", "PH")]
    zero = (np.zeros(g.shape("C")[1:]), np.zeros(g.shape("C")[1:]))
    blk = o.solved("C")
    w = g.weights_omega("C")[blk]
    d = Tn - Tm
    LT = 0.0
    for axis in range(3):
        LT = LT + ops.apply_dir(g, "T", Tn, axis, ops.coeffs(g, o.prm, "T", axis, False, astar), zero)
    DL = 0.0
    for axis in (1, 2):                     # the hat operators differ from the full ones in theta, phi
        Lh = ops.apply_dir(g, "T", d, axis, ops.coeffs(g, o.prm, "T", axis, True, astar), zero)
        Lf = ops.apply_dir(g, "T", d, axis, ops.coeffs(g, o.prm, "T", axis, False, astar), zero)
        DL = DL + (Lh - Lf)
    e_grad = 0.5 * float(np.sum(w * (-LT[blk]) * Tn[blk]))
    e_hat = 0.25 * float(np.sum(w * (-DL[blk]) * d[blk]))
    e_dt = float(np.sum(w * d[blk] ** 2))
    return e_grad, e_hat, e_dt

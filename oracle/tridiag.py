"""Tridiagonal line solvers (§4).

'the system in each direction can be solved directly by the Thomas algorithm'
(P:L480).  `thomas` is the textbook forward elimination / back substitution,
vectorised over independent lines only (each line is processed in its own
order i = 0..n-1, n-1..0).  `partitioned` is the domain-decomposition Schur
complement solve of P:L477-480 (the cited fld.2583 scheme, restated): every
segment is reduced to its two end unknowns, the interface system is solved,
and the segment interiors are recovered.
"""
from __future__ import annotations

import numpy as np

PIVOT_MIN = 1e-14


class SolverError(RuntimeError):
    pass


def thomas(a, b, c, d):
    """Solve a_i x_{i-1} + b_i x_i + c_i x_{i+1} = d_i, i = 0..n-1 (a_0, c_{n-1}
    unused) for every line; arrays have the line index first: shape (n, ...)."""
    a, b, c, d = (np.asarray(v, dtype=np.float64) for v in (a, b, c, d))
    n = d.shape[0]
    cp = np.empty_like(d)
    dp = np.empty_like(d)
    piv = b[0].copy()
    if np.any(np.abs(piv) < PIVOT_MIN):
        raise SolverError("pivot breakdown")
    cp[0] = c[0] / piv
    dp[0] = d[0] / piv
    for i in range(1, n):
        piv = b[i] - a[i] * cp[i - 1]
        if np.any(np.abs(piv) < PIVOT_MIN):
            raise SolverError("pivot breakdown")
        cp[i] = c[i] / piv
        dp[i] = (d[i] - a[i] * dp[i - 1]) / piv
    x = np.empty_like(d)
    x[n - 1] = dp[n - 1]
    for i in range(n - 2, -1, -1):
        x[i] = dp[i] - cp[i] * x[i + 1]
    return x


def partitioned(a, b, c, d, P: int):
    """Schur-complement solve of one batch of lines split into P contiguous
    segments.  Per segment s with rows [l, r]:
      local solve  A_s y = d_s,  A_s v = -a_l e_0,  A_s w = -c_r e_last
      (so x_s = y + v x_{l-1} + w x_{r+1}),
    interface unknowns x_{l-1}, x_{r+1} are the segment end values of the
    neighbours, giving a tridiagonal-by-blocks system on the 2P end unknowns,
    solved here densely per line; then x_s is recovered."""
    a, b, c, d = (np.asarray(v, dtype=np.float64) for v in (a, b, c, d))
    n = d.shape[0]
    if P < 1 or P > n:
        raise ValueError("bad partition")
    bounds = np.linspace(0, n, P + 1).round().astype(int)
    segs = [(bounds[s], bounds[s + 1] - 1) for s in range(P)]
    rest = d.shape[1:]
    ys, vs, ws = [], [], []
    for (l, r) in segs:
        m = r - l + 1
        aa, bb, cc = a[l:r + 1].copy(), b[l:r + 1], c[l:r + 1].copy()
        aa[0] = 0.0
        cc[-1] = 0.0
        y = thomas(aa, bb, cc, d[l:r + 1])
        e0 = np.zeros((m,) + rest)
        e0[0] = -a[l] if l > 0 else 0.0
        el = np.zeros((m,) + rest)
        el[-1] = -c[r] if r < n - 1 else 0.0
        ys.append(y)
        vs.append(thomas(aa, bb, cc, e0))
        ws.append(thomas(aa, bb, cc, el))
    # interface unknowns: first and last value of every segment, z = (f_0, g_0, f_1, g_1, ...)
    # f_s = y_s[0] + v_s[0] g_{s-1} + w_s[0] f_{s+1};  g_s = y_s[-1] + v_s[-1] g_{s-1} + w_s[-1] f_{s+1}
    N = 2 * P
    flat = int(np.prod(rest)) if rest else 1
    Y0 = np.stack([y[0].reshape(flat) for y in ys])
    Y1 = np.stack([y[-1].reshape(flat) for y in ys])
    V0 = np.stack([v[0].reshape(flat) for v in vs])
    V1 = np.stack([v[-1].reshape(flat) for v in vs])
    W0 = np.stack([w[0].reshape(flat) for w in ws])
    W1 = np.stack([w[-1].reshape(flat) for w in ws])
    Z = np.empty((N, flat))
    for L in range(flat):
        M = np.eye(N)
        rhs = np.zeros(N)
        for s in range(P):
            rhs[2 * s] = Y0[s, L]
            rhs[2 * s + 1] = Y1[s, L]
            if s > 0:
                M[2 * s, 2 * (s - 1) + 1] -= V0[s, L]
                M[2 * s + 1, 2 * (s - 1) + 1] -= V1[s, L]
            if s < P - 1:
                M[2 * s, 2 * (s + 1)] -= W0[s, L]
                M[2 * s + 1, 2 * (s + 1)] -= W1[s, L]
        Z[:, L] = np.linalg.solve(M, rhs)
    x = np.empty_like(d)
    for s, (l, r) in enumerate(segs):
        gl = Z[2 * (s - 1) + 1].reshape(rest) if s > 0 else 0.0
        fr = Z[2 * (s + 1)].reshape(rest) if s < P - 1 else 0.0
        x[l:r + 1] = ys[s] + vs[s] * gl + ws[s] * fr
    return x

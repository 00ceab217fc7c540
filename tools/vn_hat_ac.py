#!/usr/bin/env python
"""Von Neumann model of the fixed point of one AC direction-splitting step
(DESIGN.md RD-E4).  2-D periodic Stokes + artificial compressibility:

  (u1 - u)/tau = -nu(alpha k^2 + l^2) u^* - 1/2 nu (beta k^2 + l^2)(u1 - 2u + um)
                 + c_chi grad div u^{n+1/2} - grad p^n,      c_chi = 1/(2 chi)
  chi (p1 - p) + div u^{n+1/2} = 0

i.e. CN with the implicit hat operator (coefficient beta >= alpha in x, the
"over-implicit" Delta^ of P:L208) and the AB2-lagged explicit (full - hat)
part of eq:HeatDouglas, plus the CN-AC pressure coupling.
Prints max |amplification| over wavenumbers: > 1 means unstable.

    python tools/vn_hat_ac.py [chi ...]
"""
import sys

import numpy as np


def amplification(tau, chi, nu, k, l, alpha, beta):
    c = 1 / (2 * chi)
    A = np.zeros((3, 3), complex)
    B = np.zeros((3, 5), complex)   # state (u, v, p, um, vm)
    for row in (0, 1):
        F = alpha * k * k + l * l
        H = beta * k * k + l * l
        A[row, row] += 1 / tau + 0.5 * nu * H
        B[row, row] += 1 / tau - 1.5 * nu * F + nu * H
        B[row, row + 3] += 0.5 * nu * F - 0.5 * nu * H
    G = np.array([[k * k, k * l], [k * l, l * l]])
    for i in range(2):
        for j in range(2):
            A[i, j] += 0.5 * c * G[i, j]
            B[i, j] -= 0.5 * c * G[i, j]
    B[0, 2] -= 1j * k
    B[1, 2] -= 1j * l
    A[2, 2] = 1
    A[2, 0] = 1j * k / (2 * chi)
    A[2, 1] = 1j * l / (2 * chi)
    B[2, 2] = 1
    B[2, 0] = -1j * k / (2 * chi)
    B[2, 1] = -1j * l / (2 * chi)
    X = np.linalg.solve(A, B)
    M = np.zeros((5, 5), complex)
    M[:3] = X
    M[3, 0] = 1
    M[4, 1] = 1
    return max(abs(np.linalg.eigvals(M)))


def max_growth(tau, chi, beta, nu=1.0):
    ks = np.geomspace(0.3, 3000, 90)
    return max(amplification(tau, chi, nu, k, l, 1.0, beta) for k in ks for l in (0.0, 0.3 * k, k, 3 * k))


if __name__ == "__main__":
    chis = [float(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16]
    for beta in (1.0, 2.0, 3.0, 4.0, 8.4, 16.0):
        print("beta %5.1f  " % beta + "  ".join("chi=%g: %.4f" % (c, max_growth(1e-3, c, beta)) for c in chis))

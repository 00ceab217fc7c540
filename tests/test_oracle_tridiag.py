"""Pins of oracle/tridiag.py (Thomas; partitioned Schur solve, L477-480)
against things other than itself: worked examples and a dense
LU solve (numpy.linalg.solve, LAPACK gesv with partial pivoting)."""
import numpy as np
import pytest

from oracle.tridiag import SolverError, partitioned, thomas


def test_worked_example():
    # diag (2,2,2), off (-1,-1), b = (1,0,1) -> x = (1,1,1)
    a = np.array([0.0, -1, -1])
    b = np.array([2.0, 2, 2])
    c = np.array([-1.0, -1, 0])
    x = thomas(a, b, c, np.array([1.0, 0, 1]))
    assert np.max(np.abs(x - 1.0)) <= 4e-16


def test_identity_exact():
    rng = np.random.default_rng(0)
    d = rng.standard_normal((7, 5))
    x = thomas(np.zeros_like(d), np.ones_like(d), np.zeros_like(d), d)
    assert np.array_equal(x, d)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 17, 64])
def test_vs_dense_lu(n):
    rng = np.random.default_rng(n)
    L = 11
    a = rng.uniform(-1, 1, (n, L))
    c = rng.uniform(-1, 1, (n, L))
    b = 2.5 + rng.uniform(0, 1, (n, L))
    d = rng.uniform(-1, 1, (n, L))
    x = thomas(a, b, c, d)
    for line in range(L):
        M = np.diag(b[:, line])
        for i in range(1, n):
            M[i, i - 1] = a[i, line]
            M[i - 1, i] = c[i - 1, line]
        ref = np.linalg.solve(M, d[:, line])
        assert np.max(np.abs(x[:, line] - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


def test_pivot_breakdown_raises():
    with pytest.raises(SolverError):
        thomas(np.zeros(2), np.zeros(2), np.zeros(2), np.ones(2))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_partitioned_equals_thomas(P):
    rng = np.random.default_rng(100 + P)
    n, L = 101, 6
    a = rng.uniform(-1, 1, (n, L))
    c = rng.uniform(-1, 1, (n, L))
    b = 2.5 + rng.uniform(0, 1, (n, L))
    d = rng.uniform(-1, 1, (n, L))
    x = partitioned(a, b, c, d, P)
    ref = thomas(a, b, c, d)
    assert np.max(np.abs(x - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_partitioned_degenerate_and_worked():
    # S:L257 (2 segments on the 3x3 example) and S:L259 (segments = n)
    a = np.array([0.0, -1, -1])
    b = np.array([2.0, 2, 2])
    c = np.array([-1.0, -1, 0])
    d = np.array([1.0, 0, 1])
    assert np.allclose(partitioned(a, b, c, d, 2), 1.0, atol=1e-15)
    assert np.allclose(partitioned(a, b, c, d, 3), 1.0, atol=1e-15)

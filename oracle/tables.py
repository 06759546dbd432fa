"""1D tables for the numpy oracles (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

- Gauss rule on [0,1] with m points: tensor Gauss quadrature.
  Library primitive numpy.polynomial.legendre.leggauss on [-1,1], mapped.
- Orthonormal shifted Legendre basis theta_j(x) = sqrt(2j+1) P_j(2x-1)
  (reading C-2; "L2-orthogonal Legendre polynomials"),
  evaluated with numpy's Legendre series class.
"""
import numpy as np
from numpy.polynomial import legendre as npleg


def gauss01(m):
    """m-point Gauss-Legendre points (ascending) and weights on [0,1]."""
    t, w = npleg.leggauss(m)
    return 0.5 * (t + 1.0), 0.5 * w


def theta(n, x):
    """Values and derivatives of theta_0..theta_{n-1} at points x.

    Returns (th, dth), each of shape (len(x), n)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    th = np.empty((x.size, n))
    dth = np.empty((x.size, n))
    for j in range(n):
        c = np.zeros(j + 1)
        c[j] = np.sqrt(2.0 * j + 1.0)
        th[:, j] = npleg.legval(2.0 * x - 1.0, c)
        dth[:, j] = 2.0 * npleg.legval(2.0 * x - 1.0, npleg.legder(c))
    return th, dth

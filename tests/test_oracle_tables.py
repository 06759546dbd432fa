"""Pins of the oracle's 1D tables (C O-1 tables and numpy tables.py) against
closed forms (SPEC.md worked examples), quadrature exactness and a library
routine. PAPER.md:404-416 (tensor Gauss rule), :373 (orthonormal Legendre)."""
import math

import numpy as np
import pytest

from conftest import golden, num
from oracle import o1, tables


def test_gauss_closed_forms():
    g = golden("tables_1d.json")
    xi, w, *_ = o1.tables(0)
    assert np.allclose(xi, g["gauss_m1"]["x"], atol=1e-15) and np.allclose(w, g["gauss_m1"]["w"], atol=1e-15)
    xi, w, *_ = o1.tables(1)
    assert np.allclose(xi, [num(v) for v in g["gauss_m2"]["x"]], atol=1e-15)
    assert np.allclose(w, g["gauss_m2"]["w"], atol=1e-15)
    x2, w2 = tables.gauss01(2)
    assert np.allclose(x2, [num(v) for v in g["gauss_m2"]["x"]], atol=1e-15)


@pytest.mark.parametrize("m", range(1, 12))
def test_gauss_exactness_and_library(m):
    xi, w, *_ = o1.tables(m - 1)
    assert np.all(np.diff(xi) > 0) and np.all(w > 0)
    for p in range(2 * m):
        assert abs(np.dot(w, xi ** p) - 1.0 / (p + 1)) < 1e-14
    # not exact for 2m (the rule is not over-integrating)
    assert abs(np.dot(w, xi ** (2 * m)) - 1.0 / (2 * m + 1)) > 1e-15
    t, wl = np.polynomial.legendre.leggauss(m)
    assert np.allclose(xi, 0.5 * (t + 1), atol=2e-16 * 8) and np.allclose(w, 0.5 * wl, atol=1e-15)
    assert np.allclose(xi + xi[::-1], 1.0, atol=1e-15)


def test_theta_closed_forms():
    g = golden("tables_1d.json")
    xi, w, th, dth, t0, t1, d0, d1 = o1.tables(1)
    assert np.allclose(t0, [num(v) for v in g["theta_k1_at0"]], atol=1e-15)
    assert np.allclose(t1, [num(v) for v in g["theta_k1_at1"]], atol=1e-15)
    assert np.allclose(dth[:, 1], num(g["dtheta1"]), atol=1e-14)
    assert np.allclose(th[:, 0], 1.0)
    v, _ = tables.theta(2, [0.5])
    assert abs(v[0, 1]) < 1e-16


@pytest.mark.parametrize("k", [1, 3, 7, 10])
def test_theta_orthonormal_endpoints_fd(k):
    n = k + 1
    xi, w, th, dth, t0, t1, d0, d1 = o1.tables(k)
    G = th.T @ np.diag(w) @ th
    assert np.abs(G - np.eye(n)).max() < 1e-13
    j = np.arange(n)
    s = np.sqrt(2 * j + 1.0)
    assert np.allclose(t1, s, atol=1e-13) and np.allclose(t0, (-1.0) ** j * s, atol=1e-13)
    assert np.allclose(d1, s * j * (j + 1), rtol=1e-13, atol=1e-12)
    assert np.allclose(d0, (-1.0) ** (j + 1) * s * j * (j + 1), rtol=1e-13, atol=1e-12)
    # derivative by central finite differences of the numpy tables (independent evaluator)
    x = np.array([0.13, 0.5, 0.77])
    hfd = 1e-5
    vp, _ = tables.theta(n, x + hfd)
    vm, _ = tables.theta(n, x - hfd)
    _, dv = tables.theta(n, x)
    assert np.allclose((vp - vm) / (2 * hfd), dv, atol=1e-6 * max(1.0, np.abs(dv).max()))
    # the C oracle and numpy tables agree
    vn, dn = tables.theta(n, xi)
    assert np.allclose(vn, th, atol=1e-13) and np.allclose(dn, dth, atol=1e-11)

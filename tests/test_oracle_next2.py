"""NEXT-2 / NEXT-3 oracle pins: a velocity field b(x) evaluated at every quadrature point
(the Taylor-Green field, eq:2 PAPER.md:1093-1100) and over-integration with m = k+3 Gauss
points per direction (q = 2p+4).

- O-1 (naive C) == O-2 (assembled from the weak form) with the Taylor-Green field on the
  paper's periodic box (-pi, pi)^3 and with a linear field on a Dirichlet box, m = k+1, k+3;
- over-integration changes nothing where the integrands are polynomials of degree <= 2k+1:
  constant coefficients give the same operator for m = k+1 and m = k+3;
- conservation: on a periodic box with c = 0, a_h(u, 1) = 0 term by term for ANY b(x), so
  the constant-mode components of A z sum to zero (the discrete mass of the transport step);
- consistency with a variable velocity: for the linear divergence-free field b = (x2, x3, x1)
  and u* in Q_k every integrand is a polynomial the rule integrates exactly, so A z* = F with
  f = b.grad u* + c u* - div(D grad u*) (a dropped or misplaced b(x) breaks it).
"""
import numpy as np
import pytest

from oracle import o1, o2_assembled as o2, rhs
from paper_1711_10885_b200 import inputs


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


TG_BOX = ((-np.pi,) * 3, (np.pi,) * 3)


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("extra", [0, 2])
def test_o1_equals_o2_taylor_green_periodic(k, extra):
    nc = (3, 2, 2)
    z = inputs.uniform(12 * (k + 1) ** 3, 3)
    args = (nc, TG_BOX[0], TG_BOX[1], k, np.diag([1.0, 2.0, 0.5]), (0, 0, 0), 0.3, 20.0)
    y1, _ = o1.apply(*args, z, m=k + 1 + extra, bkind=1, periodic=(1, 1, 1))
    A = o2.assemble(*args, m=k + 1 + extra, bfield=o2.taylor_green, periodic=(1, 1, 1))
    assert rel(y1, A @ z) < 1e-13


@pytest.mark.parametrize("k", [1, 3])
def test_o1_equals_o2_linear_field_dirichlet(k):
    nc, lo, hi = (3, 2, 2), (-0.3, 0.1, 0.2), (1.2, 1.1, 0.7)
    z = inputs.uniform(12 * (k + 1) ** 3, 4)
    args = (nc, lo, hi, k, np.diag([1.0, 2.0, 0.5]), (0, 0, 0), 0.3, 20.0)
    for mask in (1, 2, 4, 7):
        y1, _ = o1.apply(*args, z, mask=mask, m=k + 3, bkind=2, bamp=(0.7, -1.1, 0.4))
        A = o2.assemble(*args, mask=mask, m=k + 3,
                        bfield=lambda x: o2.linear_field(x) * np.array([0.7, -1.1, 0.4])[:, None])
        assert rel(y1, A @ z) < 1e-13


@pytest.mark.parametrize("k", [1, 2, 4])
def test_over_integration_exact_for_constant_coefficients(k):
    nc, lo, hi = (3, 2, 2), (0, 0, 0), (1.5, 1.0, 0.5)
    z = inputs.uniform(12 * (k + 1) ** 3, 5)
    args = (nc, lo, hi, k, np.diag([1.0, 2.0, 0.5]), (1.0, -0.5, 0.25), 0.3, 30.0)
    ya, _ = o1.apply(*args, z)
    yb, _ = o1.apply(*args, z, m=k + 3)
    assert rel(yb, ya) < 1e-13
    # and a field that is NOT polynomial does see the quadrature order (the pin has teeth)
    yc, _ = o1.apply(*args, z, bkind=1)
    yd, _ = o1.apply(*args, z, m=k + 3, bkind=1)
    assert rel(yd, yc) > 1e-9


@pytest.mark.parametrize("k,extra", [(1, 2), (3, 2), (2, 0)])
def test_conservation_any_velocity_periodic(k, extra):
    nc = (3, 3, 2)
    n3 = (k + 1) ** 3
    z = inputs.uniform(18 * n3, 6)
    y, _ = o1.apply(nc, TG_BOX[0], TG_BOX[1], k, 5e-6 * np.eye(3), (0, 0, 0), 0.0, 3.0 * k * (k + 2),
                    z, m=k + 1 + extra, bkind=1, periodic=(1, 1, 1))
    assert abs(y.reshape(18, n3)[:, 0].sum()) < 1e-14 * np.abs(y).sum()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_consistency_linear_velocity(k):
    nc, lo, hi = (3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5)
    D = np.diag([1.0, 2.0, 0.5])
    args = (nc, lo, hi, k, D, (0, 0, 0), 0.4, 3.0 * k * (k + 2) / 0.25)
    amp = np.array([0.8, -0.6, 1.2])
    bf = lambda x: o2.linear_field(x) * amp[:, None]
    zs, F = rhs.consistency_data(*args, seed=k, bfield=bf)
    for extra in (0, 2):
        y, _ = o1.apply(*args, zs, m=k + 1 + extra, bkind=2, bamp=tuple(amp))
        assert rel(y, F) < 1e-13
    # control: the same data with the field dropped (constant b = 0) is not consistent
    y0, _ = o1.apply(*args, zs)
    assert rel(y0, F) > 1e-6


# ---- the Taylor-Green field itself (eq:2), pinned independently of the
# operator: hand values at points where every factor is 0 or +-1, div b = 0 by central
# differences (the field of a transport step must be divergence free, PAPER.md:334-341 relies
# on it), and 2 pi periodicity on the paper's box (-pi, pi)^3.
TG_HAND = [  # x -> b, each factor of each component 0 or +-1 (a sign slip on any factor shows)
    ((0.0, -np.pi / 2, -np.pi / 2), (1.0, 0.0, 0.0)),     # cos 0 sin(pi/2) sin(pi/2)
    ((np.pi / 2, 0.0, -np.pi / 2), (0.0, 0.5, 0.0)),      # 1/2 sin(pi/2) cos 0 sin(pi/2)
    ((np.pi / 2, -np.pi / 2, 0.0), (0.0, 0.0, 0.5)),      # 1/2 sin(pi/2) sin(pi/2) cos 0
    ((np.pi, np.pi / 2, np.pi / 2), (-1.0, 0.0, 0.0)),    # cos pi sin(-pi/2) sin(-pi/2)
    ((-np.pi / 2, 0.0, np.pi / 2), (0.0, 0.5, 0.0)),      # 1/2 sin(-pi/2) cos 0 sin(-pi/2)
]


def _tg_fields():
    return {"O-1 (C)": lambda x: o1.velocity(1, x),
            "O-2 (numpy)": lambda x: o2.taylor_green(np.asarray(x).T).T}


@pytest.mark.parametrize("which", ["O-1 (C)", "O-2 (numpy)"])
def test_taylor_green_hand_values(which):
    f = _tg_fields()[which]
    for x, b in TG_HAND:
        got = f(np.array([x]))[0]
        assert np.allclose(got, b, rtol=0, atol=1e-15), (which, x, got, b)


@pytest.mark.parametrize("which", ["O-1 (C)", "O-2 (numpy)"])
def test_taylor_green_divergence_free_and_periodic(which):
    f = _tg_fields()[which]
    rng = np.random.default_rng(11)
    x = rng.uniform(-np.pi, np.pi, (64, 3))
    h = 1e-5
    div = np.zeros(x.shape[0])
    for q in range(3):
        e = np.zeros(3)
        e[q] = h
        div += (f(x + e)[:, q] - f(x - e)[:, q]) / (2 * h)
    assert np.abs(div).max() < 1e-9
    # not trivially zero: each partial derivative is O(1) somewhere
    dq = (f(x + [h, 0, 0])[:, 0] - f(x - [h, 0, 0])[:, 0]) / (2 * h)
    assert np.abs(dq).max() > 0.3
    for q in range(3):
        e = np.zeros(3)
        e[q] = 2 * np.pi
        assert np.abs(f(x + e) - f(x)).max() < 1e-14


def test_o1_linear_field_and_amplitudes():
    x = np.array([[0.5, -2.0, 3.0]])
    assert np.array_equal(o1.velocity(2, x), [[-2.0, 3.0, 0.5]])          # b = (x2, x3, x1)
    assert np.array_equal(o1.velocity(2, x, (2.0, 0.5, -1.0)), [[-4.0, 1.5, -0.5]])

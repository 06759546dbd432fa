"""NEXT-1 oracle pins: periodic boundaries and a per-cell diffusion
tensor with live WSIPG weights and harmonic penalty (the paper's Problem A,
PAPER.md:940-948; weights :274-281; <a,b> :293; gamma :328-333).

Pins chosen so a plausible mistake fails one of them:
- hand-derived two-cell entries (tests/golden/two_cell_wsipg.json): harmonic gamma,
  which side's weight multiplies which side's flux, the off-diagonal D term, upwind side;
- O-1 (naive C) == O-2 (assembled from the weak form) with per-cell SPD tensors and
  every periodic combination; O-3 (Kronecker closed form) == O-1 for periodic diagonal D;
- translation invariance on a periodic box (a wrong wrap orientation breaks it);
- constant u on a fully periodic box: A 1 = c Delta_T 1 (div b = 0, no jumps);
- consistency with discontinuous D: a continuous piecewise-linear u* whose normal flux
  is continuous across the jumps of D is reproduced (A z* = F);
- SIPG symmetry (b = 0) with per-cell D and periodic faces.
"""
import numpy as np
import pytest

from oracle import o1, o2_assembled as o2, o3_kron as o3, rhs
from paper_1711_10885_b200 import inputs

from conftest import golden, num


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def spd_field(ncell, seed, iso=0.5):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(ncell, 3, 3))
    return np.einsum("eij,ekj->eik", M, M) + iso * np.eye(3)[None]


MESH = ((3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5))


def _entry(case):
    d1, d2, e, bx, s = case["d1"], case["d2"], case["e"], case["bx"], case["sigma"]
    Dc = np.zeros((2, 3, 3))
    Dc[0] = np.eye(3) * d1
    Dc[1] = np.eye(3) * d2
    Dc[1, 0, 1] = Dc[1, 1, 0] = e
    unit = np.zeros(16)
    unit[case["j"]] = 1.0
    y, _ = o1.apply((2, 1, 1), (0, 0, 0), (2, 1, 1), 1, np.eye(3), (bx, 0.0, 0.0), 0.0, s, unit, Dcell=Dc)
    return y[case["i"]]


@pytest.mark.parametrize("idx", range(5))
def test_two_cell_hand_entries(idx):
    case = golden("two_cell_wsipg.json")["cases"][idx]
    assert abs(_entry(case) - num(case["value"])) < 1e-13 * max(1.0, abs(num(case["value"])))


def test_two_cell_entries_o2_agrees():
    for case in golden("two_cell_wsipg.json")["cases"]:
        d1, d2, e = case["d1"], case["d2"], case["e"]
        Dc = np.stack([np.eye(3) * d1, np.eye(3) * d2])
        Dc[1, 0, 1] = Dc[1, 1, 0] = e
        A = o2.assemble((2, 1, 1), (0, 0, 0), (2, 1, 1), 1, np.eye(3), (case["bx"], 0, 0), 0.0, case["sigma"],
                        Dcell=Dc)
        assert abs(A[case["i"], case["j"]] - num(case["value"])) < 1e-13 * max(1.0, abs(num(case["value"])))


@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)])
@pytest.mark.parametrize("k", [1, 2])
def test_o1_equals_o2_percell_D(periodic, k):
    nc, lo, hi = MESH
    ncell = 12
    Dc = spd_field(ncell, 5 + k)
    z = inputs.uniform(ncell * (k + 1) ** 3, 21 + k)
    b, c, sigma = (0.8, -0.4, 0.3), 0.6, 3.0 * k * (k + 2) / 0.25
    for mask in (1, 2, 4, 7):
        y1, _ = o1.apply(nc, lo, hi, k, np.eye(3), b, c, sigma, z, mask=mask, periodic=periodic, Dcell=Dc)
        A = o2.assemble(nc, lo, hi, k, np.eye(3), b, c, sigma, mask=mask, periodic=periodic, Dcell=Dc)
        if mask == 4 and all(periodic):
            assert not np.any(y1) and not np.any(A)
            continue
        assert rel(y1, A @ z) < 1e-13


def test_o1_equals_o2_one_cell_periodic():
    # a periodic direction with a single cell: the cell is its own neighbour
    Dc = spd_field(2, 3)
    z = inputs.uniform(2 * 27, 4)
    args = ((1, 2, 1), (0, 0, 0), (0.5, 1.0, 0.5), 2, np.eye(3), (0.3, 0.2, -0.6), 0.4, 40.0)
    y1, _ = o1.apply(*args, z, periodic=(1, 1, 1), Dcell=Dc)
    A = o2.assemble(*args, periodic=(1, 1, 1), Dcell=Dc)
    assert rel(y1, A @ z) < 1e-13


@pytest.mark.parametrize("periodic", [(1, 0, 0), (0, 1, 1), (1, 1, 1)])
def test_o3_periodic_equals_o1(periodic):
    nc, lo, hi = (4, 3, 2), (0, 0, 0), (1.0, 1.5, 0.5)
    k = 3
    D = np.diag([1.0, 2.0, 0.5])
    z = inputs.uniform(24 * 64, 8)
    args = (nc, lo, hi, k, D, (1.0, -0.5, 0.25), 0.3, 30.0)
    y1, _ = o1.apply(*args, z, periodic=periodic)
    y3 = o3.apply(*args, z, periodic=periodic)
    assert rel(y1, y3) < 1e-13


def _shift(v, nc, n3, q):
    a = np.asarray(v).reshape(nc[2], nc[1], nc[0], -1)
    return np.roll(a, 1, axis=2 - q).reshape(-1)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_translation_invariance_periodic(q):
    nc, lo, hi = (4, 3, 3), (0, 0, 0), (1.0, 0.75, 0.75)
    k = 2
    n3 = 27
    ncell = 36
    Dc = spd_field(ncell, 9)
    z = inputs.uniform(ncell * n3, 10)
    args = (nc, lo, hi, k, np.eye(3), (0.9, -0.3, 0.5), 0.2, 96.0)
    per = (1, 1, 1)
    y, _ = o1.apply(*args, z, periodic=per, Dcell=Dc)
    ys, _ = o1.apply(*args, _shift(z, nc, n3, q), periodic=per, Dcell=_shift(Dc.reshape(ncell, 9), nc, 9, q))
    assert rel(ys, _shift(y, nc, n3, q)) < 1e-14


def test_translation_breaks_without_periodic():
    # control: the same check on a Dirichlet box must fail (the pin has teeth)
    nc, lo, hi = (4, 3, 3), (0, 0, 0), (1.0, 0.75, 0.75)
    z = inputs.uniform(36 * 27, 10)
    args = (nc, lo, hi, 2, np.eye(3), (0.9, -0.3, 0.5), 0.2, 96.0)
    y, _ = o1.apply(*args, z)
    ys, _ = o1.apply(*args, _shift(z, nc, 27, 0))
    assert rel(ys, _shift(y, nc, 27, 0)) > 1e-3


@pytest.mark.parametrize("k", [1, 3])
def test_constant_state_periodic_is_mass(k):
    nc, lo, hi = MESH
    ncell, n3 = 12, (k + 1) ** 3
    z = np.zeros((ncell, n3))
    z[:, 0] = 1.7                       # u = 1.7 everywhere (theta_0 = 1)
    c = 0.45
    y, _ = o1.apply(nc, lo, hi, k, np.eye(3), (0.8, -0.4, 0.3), c, 50.0, z.ravel(), periodic=(1, 1, 1),
                    Dcell=spd_field(ncell, 2))
    dT = 0.5 * 0.5 * 0.25
    assert rel(y, c * dT * z.ravel()) < 1e-13


@pytest.mark.parametrize("k", [1, 2, 4])
def test_consistency_discontinuous_D(k):
    # D jumps across every x-face (random SPD tensor per x-layer); u* piecewise linear in x
    # with slope F / D_xx per layer: continuous u* and continuous normal flux.
    nc, lo, hi = (4, 2, 2), (0.0, 0.0, 0.0), (1.0, 0.5, 0.5)
    ncell = 16
    layers = spd_field(4, 31 + k)
    Dc = np.stack([layers[e % 4] for e in range(ncell)])
    field = rhs.KinkedField(lo[0], 0.25, layers[:, 0, 0], flux=1.3, u0=-0.4)
    b, c, sigma = (0.7, -0.2, 0.5), 0.9, 3.0 * k * (k + 2) / 0.25
    args = (nc, lo, hi, k, np.eye(3), b, c, sigma)
    zs, F = rhs.consistency_data(*args, Dcell=Dc, field=field)
    y, _ = o1.apply(*args, zs, Dcell=Dc)
    assert rel(y, F) < 1e-13
    # the same u* with a tensor that is continuous (layer 0 everywhere) is NOT reproduced
    # by the discontinuous-D operator: the check sees D per side
    Dbad = np.stack([layers[0]] * ncell)
    ybad, _ = o1.apply(*args, zs, Dcell=Dbad)
    assert rel(ybad, F) > 1e-6


def test_symmetry_percell_D_periodic():
    nc, lo, hi = MESH
    A = o2.assemble(nc, lo, hi, 2, np.eye(3), (0, 0, 0), 0.5, 60.0, periodic=(1, 0, 1), Dcell=spd_field(12, 4))
    assert np.abs(A - A.T).max() < 1e-13 * np.abs(A).max()
    z = inputs.uniform(A.shape[0], 1)
    w = inputs.uniform(A.shape[0], 2)
    args = (nc, lo, hi, 2, np.eye(3), (0, 0, 0), 0.5, 60.0)
    Az, _ = o1.apply(*args, z, periodic=(1, 0, 1), Dcell=spd_field(12, 4))
    Aw, _ = o1.apply(*args, w, periodic=(1, 0, 1), Dcell=spd_field(12, 4))
    assert abs(w @ Az - z @ Aw) < 1e-12 * abs(w @ Az)


def test_uniform_field_equals_constant_D():
    nc, lo, hi = MESH
    D = np.array([[1.0, 0.2, -0.1], [0.2, 2.0, 0.3], [-0.1, 0.3, 0.5]])
    z = inputs.uniform(12 * 27, 6)
    args = (nc, lo, hi, 2, D, (1.0, 0.5, 0.25), 1.0, 40.0)
    ya, _ = o1.apply(*args, z, periodic=(0, 1, 0))
    yb, _ = o1.apply(*args, z, periodic=(0, 1, 0), Dcell=np.tile(D, (12, 1, 1)))
    assert np.array_equal(ya, yb)


# ------------------------------------------------------------------ NEXT-2: explicit SSP stages
@pytest.mark.parametrize("k", [1, 3])
def test_ssp_pure_reaction_closed_form(k):
    """D = 0, b = 0: A = c Delta_T I, so M^-1 A = c and forward Euler gives z (1 - c dt), Heun
    z (1 - c dt + (c dt)^2 / 2) -- the textbook stability polynomials of the two methods."""
    nc, lo, hi = (3, 2, 2), (0, 0, 0), (1.5, 1.0, 0.5)
    n3 = (k + 1) ** 3
    z = inputs.uniform(12 * n3, 3)
    args = (nc, lo, hi, k, np.zeros(9), (0, 0, 0), 0.7, 10.0)
    dt = 0.3
    e1 = o1.ssp_stage(*args, z, dt)
    assert rel(e1, z * (1 - 0.7 * dt)) < 1e-14
    h2 = o1.ssp_stage(*args, e1, dt, w=z, a=0.5, bcoef=0.5)
    assert rel(h2, z * (1 - 0.7 * dt + (0.7 * dt) ** 2 / 2)) < 1e-14


@pytest.mark.parametrize("k", [1, 2])
def test_ssp_conserves_mass_periodic(k):
    """Periodic box, c = 0, f = 0: a_h(u, 1) = 0 term by term (grad 1 = 0, [[1]] = 0), so every
    stage conserves the integral of u = Delta_T sum_e z_(e, 0)."""
    nc, lo, hi = MESH
    n3 = (k + 1) ** 3
    z = inputs.uniform(12 * n3, 5)
    args = (nc, lo, hi, k, np.eye(3), (0.8, -0.4, 0.3), 0.0, 30.0)
    Dc = spd_field(12, 8)
    mass = lambda v: v.reshape(12, n3)[:, 0].sum()
    e1 = o1.ssp_stage(*args, z, 1e-3, periodic=(1, 1, 1), Dcell=Dc)
    h2 = o1.ssp_stage(*args, e1, 1e-3, w=z, a=0.5, bcoef=0.5, periodic=(1, 1, 1), Dcell=Dc)
    assert abs(mass(e1) - mass(z)) < 1e-13 * np.abs(z).sum()
    assert abs(mass(h2) - mass(z)) < 1e-13 * np.abs(z).sum()
    # control: with Dirichlet faces the boundary fluxes change the mass
    d1 = o1.ssp_stage(*args, z, 1e-3, Dcell=Dc)
    assert abs(mass(d1) - mass(z)) > 1e-8

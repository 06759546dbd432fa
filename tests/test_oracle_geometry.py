"""Pins of the multilinear-geometry oracle (oracle/o2_geometry.py; NEXT-3, Problem C's
"multilinear geometries"), each fixed by something other than the
oracle itself:

- the regular vertex grid is the axis-aligned mesh: equals O-2 of o2_assembled.py (pinned by the
  hand-derived cells, the Kronecker closed form and the anchors), for m = k+1 and k+3, periodic;
- an affine vertex grid lo + J (xhat - lo) equals the affine O-2 (cof(J) = det J J^-T there,
  cyclic cross products of the tangents here);
- polynomial consistency on PERTURBED meshes: a physical linear u* is Q_1 on every mapped cell, the
  integrands are polynomial, and SIPG reproduces it: A z* = F to rounding, while the same data on
  the unperturbed operator fail (the pin sees the geometry);
- symmetry for b = 0 on a perturbed mesh; total mass: D = 0, b = 0, c = 1 and the constant state
  give sum_T (A 1)_{T,0} = |Omega| (the box volume: the box sides stay planar);
- conservation: on a periodic perturbed mesh with c = 0 the constant-mode components of A z sum to
  zero for any z (a_h(u, 1) = 0 term by term: the face fluxes cancel between the two sides).
"""
import numpy as np
import pytest

from oracle import o2_assembled as o2, o2_geometry as o2g
from paper_1711_10885_b200 import inputs


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


NC, LO, HI = (3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5)
DFULL = np.array([[1.0, 0.2, 0.1], [0.2, 2.0, -0.3], [0.1, -0.3, 0.5]])
B = (1.0, -0.5, 0.25)


@pytest.mark.parametrize("k,extra", [(1, 0), (2, 0), (2, 2), (3, 0)])
@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 1)])
def test_regular_grid_equals_axis_aligned_o2(k, extra, periodic):
    X = inputs.vertex_grid(NC, LO, HI, 0.0, 0, periodic)
    for mask in (1, 2, 4, 7):
        Ag = o2g.assemble(NC, X, k, DFULL, B, 0.3, 20.0, m=k + 1 + extra, periodic=periodic, mask=mask)
        Aa = o2.assemble(NC, LO, HI, k, DFULL, B, 0.3, 20.0, m=k + 1 + extra, periodic=periodic, mask=mask)
        assert rel(Ag, Aa) < 1e-13, mask


@pytest.mark.parametrize("k", [1, 2])
def test_affine_grid_equals_affine_o2(k):
    J = np.array([[1.0, 0.3, 0.0], [-0.2, 0.9, 0.1], [0.1, 0.0, 1.2]])
    X0 = inputs.vertex_grid(NC, LO, HI, 0.0, 0)
    lo = np.asarray(LO)
    X = lo + np.einsum("rs,zyxs->zyxr", J, X0 - lo)
    Ag = o2g.assemble(NC, X, k, DFULL, B, 0.3, 20.0)
    Aa = o2.assemble(NC, LO, HI, k, DFULL, B, 0.3, 20.0, J=J)
    assert rel(Ag, Aa) < 1e-13


@pytest.mark.parametrize("k,m", [(1, 3), (2, 3), (3, 4), (4, 5), (3, 8)])
@pytest.mark.parametrize("Dkind", ["diag", "full"])
def test_linear_consistency_on_perturbed_mesh(k, m, Dkind):
    D = np.diag([1.0, 2.0, 0.5]) if Dkind == "diag" else DFULL
    X = inputs.vertex_grid(NC, LO, HI, 0.22, 4)
    assert np.abs(X - inputs.vertex_grid(NC, LO, HI, 0.0, 4)).max() > 0.02     # really perturbed
    sigma = 3.0 * k * (k + 2) / 0.25
    A = o2g.assemble(NC, X, k, D, B, 0.7, sigma, m=m)
    z, F = o2g.consistency_data(NC, X, k, D, B, 0.7, sigma, m=m, seed=k)
    assert rel(A @ z, F) < 1e-12
    # the geometry matters: the unperturbed operator does not reproduce the perturbed mesh's data
    A0 = o2g.assemble(NC, inputs.vertex_grid(NC, LO, HI, 0.0, 4), k, D, B, 0.7, sigma, m=m)
    assert rel(A0 @ z, F) > 1e-4


def test_symmetry_and_total_mass_perturbed():
    X = inputs.vertex_grid(NC, LO, HI, 0.2, 9)
    k = 2
    A = o2g.assemble(NC, X, k, DFULL, (0, 0, 0), 0.4, 30.0, m=4)
    assert rel(A, A.T) < 1e-13
    M = o2g.assemble(NC, X, k, np.zeros((3, 3)), (0, 0, 0), 1.0, 30.0, m=3)
    n3 = (k + 1) ** 3
    one = np.zeros(M.shape[0])
    one[::n3] = 1.0                                   # u = 1: theta_0 = 1 on every cell
    vol = np.prod(np.subtract(HI, LO))
    assert abs((M @ one)[::n3].sum() - vol) < 1e-14 * vol
    # ... and each cell's own entry is its volume, int det J dxi, with the trilinear map's
    # det J of degree <= 2 per direction integrated exactly by m = 2
    M2 = o2g.assemble(NC, X, k, np.zeros((3, 3)), (0, 0, 0), 1.0, 30.0, m=2)
    assert rel((M2 @ one)[::n3], (M @ one)[::n3]) < 1e-14


@pytest.mark.parametrize("k", [1, 3])
def test_conservation_periodic_perturbed(k):
    per = (1, 1, 1)
    X = inputs.vertex_grid(NC, LO, HI, 0.2, 5, per)
    A = o2g.assemble(NC, X, k, DFULL, B, 0.0, 25.0, m=k + 2, periodic=per)
    n3 = (k + 1) ** 3
    z = inputs.uniform(A.shape[0], 2)
    y = A @ z
    assert abs(y[::n3].sum()) < 1e-12 * np.abs(y).max()
    # the periodic perturbation is real (not the regular grid)
    assert np.abs(X - inputs.vertex_grid(NC, LO, HI, 0.0, 5, per)).max() > 0.02

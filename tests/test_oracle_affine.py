"""NEXT-3 affine geometry oracle pins (Problem B's "affine geometries"): O-2 on the
physical mesh x = lo + J (xhat - lo), every integral in physical terms.

- J = I reproduces the axis-aligned operator exactly;
- rigid rotation: the operator of (R D R^T, R b) on the rotated mesh equals the operator of
  (D, b) on the axis-aligned mesh (a wrong normal, face measure or gradient transform breaks it);
- consistency: a polynomial u* of total degree <= min(k, 2) in PHYSICAL coordinates lies in the
  mapped Q_k, so A z* = F with l_h assembled in physical terms, for a sheared J (and not for the
  same data on the unmapped mesh);
- SIPG symmetry for b = 0 on a sheared mesh.
"""
import numpy as np
import pytest

from oracle import o2_assembled as o2, rhs
from paper_1711_10885_b200 import inputs

MESH = ((3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5))
SHEAR = np.array([[1.0, 0.3, 0.0], [0.0, 0.9, -0.2], [0.1, 0.0, 1.2]])
DFULL = np.array([[1.0, 0.2, 0.0], [0.2, 2.0, 0.1], [0.0, 0.1, 0.5]])


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_identity_map_is_axis_aligned():
    nc, lo, hi = MESH
    A = o2.assemble(nc, lo, hi, 2, DFULL, (1, -0.5, 0.25), 0.3, 20.0)
    B = o2.assemble(nc, lo, hi, 2, DFULL, (1, -0.5, 0.25), 0.3, 20.0, J=np.eye(3))
    assert np.array_equal(A, B)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_rotation_invariance(axis):
    nc, lo, hi = MESH
    th = 0.4
    c, s = np.cos(th), np.sin(th)
    i, j = [(1, 2), (0, 2), (0, 1)][axis]
    R = np.eye(3)
    R[i, i], R[i, j], R[j, i], R[j, j] = c, -s, s, c
    b = np.array([0.7, -0.4, 0.3])
    A1 = o2.assemble(nc, lo, hi, 2, DFULL, b, 0.6, 30.0)
    A2 = o2.assemble(nc, lo, hi, 2, R @ DFULL @ R.T, R @ b, 0.6, 30.0, J=R)
    assert rel(A2, A1) < 1e-13


@pytest.mark.parametrize("k", [1, 2, 3])
def test_consistency_sheared_mesh(k):
    nc, lo, hi = MESH
    sig = 3.0 * k * (k + 2) / 0.25
    args = (nc, lo, hi, k, DFULL, (0.7, -0.4, 0.3), 0.6, sig)
    zs, F = rhs.consistency_data_affine(*args, SHEAR, seed=k)
    A = o2.assemble(*args, J=SHEAR)
    assert rel(A @ zs, F) < 1e-13
    A0 = o2.assemble(*args)
    assert rel(A0 @ zs, F) > 1e-3


def test_symmetry_sheared_mesh():
    nc, lo, hi = MESH
    A = o2.assemble(nc, lo, hi, 2, DFULL, (0, 0, 0), 0.4, 40.0, J=SHEAR, periodic=(1, 0, 0))
    assert np.abs(A - A.T).max() < 1e-13 * np.abs(A).max()

"""ctypes front end of O-1 (oracle/o1_naive.c). TEST INFRASTRUCTURE ONLY.

O-1 evaluates y = A z by plain quadrature loops with no sum factorization
(the "plain, slow" oracle BASELINE.json's north_star asks for). See the C
file's header for the formulas and PAPER.md citations.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "o1_naive.c")
_LIB = os.path.join(_HERE, "libo1_naive.so")

VOLUME, INTERIOR, BOUNDARY, ALL = 1, 2, 4, 7


class _Problem(ctypes.Structure):
    _fields_ = [("nc", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("k", ctypes.c_int), ("D", ctypes.c_double * 9), ("b", ctypes.c_double * 3),
                ("c", ctypes.c_double), ("sigma", ctypes.c_double), ("periodic", ctypes.c_int * 3),
                ("Dcell", ctypes.c_void_p), ("m", ctypes.c_int), ("bkind", ctypes.c_int),
                ("bamp", ctypes.c_double * 3)]


def build(force=False):
    """Compile the C oracle with gcc (-O3, OpenMP, portable x86-64 code)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + ".tmp%d" % os.getpid()
    subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.o1_apply.restype = ctypes.c_int
        _lib.o1_apply.argtypes = [ctypes.POINTER(_Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint,
                                  ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        _lib.o1_tables.restype = ctypes.c_int
        _lib.o1_tables.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 8
        _lib.o1_velocity_at.restype = ctypes.c_int
        _lib.o1_velocity_at.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64]
    return _lib


def velocity(bkind, x, bamp=(1.0, 1.0, 1.0)):
    """The velocity field O-1 evaluates at its quadrature points (bkind as in apply) at points
    x of shape (npts, 3); returns b of shape (npts, 3)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, 3))
    b = np.zeros_like(x)
    amp = np.ascontiguousarray(bamp, dtype=np.float64)
    if lib().o1_velocity_at(int(bkind), amp.ctypes.data, x.ctypes.data, b.ctypes.data, x.shape[0]) != 0:
        raise ValueError("o1_velocity_at: bad kind %d" % bkind)
    return b


def _problem(ncells, lo, hi, k, D, b, c, sigma, periodic=(0, 0, 0), Dcell=None, m=0, bkind=0, bamp=(1.0, 1.0, 1.0)):
    P = _Problem()
    P.m = int(m)
    P.bkind = int(bkind)
    for q in range(3):
        P.bamp[q] = float(bamp[q])
    for q in range(3):
        P.periodic[q] = 1 if periodic[q] else 0
    P.Dcell = None if Dcell is None else Dcell.ctypes.data
    for q in range(3):
        P.nc[q] = int(ncells[q])
        P.lo[q] = float(lo[q])
        P.hi[q] = float(hi[q])
        P.b[q] = float(b[q])
    Dm = np.asarray(D, dtype=np.float64).reshape(3, 3)
    for i in range(9):
        P.D[i] = float(Dm.flat[i])
    P.k = int(k)
    P.c = float(c)
    P.sigma = float(sigma)
    return P


def tables(k):
    """The oracle's own 1D tables: (xi, w, theta[i,j], dtheta[i,j], th0, th1, dth0, dth1)."""
    n = k + 1
    arrs = [np.zeros(n), np.zeros(n), np.zeros((n, n)), np.zeros((n, n))] + [np.zeros(n) for _ in range(4)]
    rc = lib().o1_tables(k, *[a.ctypes.data for a in arrs])
    if rc != 0:
        raise ValueError("o1_tables: bad degree %d" % k)
    return arrs


def apply(ncells, lo, hi, k, D, b, c, sigma, z, mask=ALL, cells=None, nthreads=0, periodic=(0, 0, 0), Dcell=None,
          m=0, bkind=0, bamp=(1.0, 1.0, 1.0)):
    """y = A z (mask selects volume / interior-face / boundary-face terms).

    cells=None: full vector. cells=int64 array: returns the compact blocks of
    those cells only, shape (len(cells), n^3) (sampled mode). Returns (y, threads).
    periodic[q]: glue the two sides normal to q (NEXT-1). Dcell: per-cell diffusion
    tensors, array [ncells_total, 3, 3] in global cell order (NEXT-1; D is then ignored).
    m: Gauss points per direction (0: k+1; NEXT-3 over-integration). bkind: 0 constant b,
    1 Taylor-Green field, 2 linear test field (x2, x3, x1); times bamp."""
    n3 = (k + 1) ** 3
    ncell_total = int(ncells[0]) * int(ncells[1]) * int(ncells[2])
    z = np.ascontiguousarray(z, dtype=np.float64)
    if z.size != ncell_total * n3:
        raise ValueError("z has %d entries, expected %d" % (z.size, ncell_total * n3))
    if Dcell is not None:
        Dcell = np.ascontiguousarray(Dcell, dtype=np.float64).reshape(-1, 9)
        if Dcell.shape[0] != ncell_total:
            raise ValueError("Dcell has %d tensors, expected %d" % (Dcell.shape[0], ncell_total))
    P = _problem(ncells, lo, hi, k, D, b, c, sigma, periodic, Dcell, m, bkind, bamp)
    if cells is None:
        y = np.zeros(ncell_total * n3)
        used = lib().o1_apply(ctypes.byref(P), z.ctypes.data, y.ctypes.data, mask, None, 0, 0, nthreads)
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        if cells.size and (cells.min() < 0 or cells.max() >= ncell_total):
            raise ValueError("cell index out of range")
        y = np.zeros((cells.size, n3))
        used = lib().o1_apply(ctypes.byref(P), z.ctypes.data, y.ctypes.data, mask, cells.ctypes.data,
                              cells.size, 1, nthreads)
    if used < 0:
        raise ValueError("o1_apply failed (%d)" % used)
    return y, used


def ssp_stage(ncells, lo, hi, k, D, b, c, sigma, z, dt, f=None, w=None, a=0.0, bcoef=1.0, periodic=(0, 0, 0),
              Dcell=None, **kw):
    """One explicit SSP Runge-Kutta stage in Shu-Osher form, written out from PAPER.md:366-373:
    M z^(k+1) = M z^(k) + dt (f - A z^(k)) with M = (phi_j, phi_i) = Delta_T I for the orthonormal
    Legendre basis on cuboid cells, generalised to out = a w + b (z + dt M^-1 (f - A z)).
    A z by O-1 (naive quadrature)."""
    n3 = (k + 1) ** 3
    h = [(hi[q] - lo[q]) / ncells[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    Az, _ = apply(ncells, lo, hi, k, D, b, c, sigma, z, periodic=periodic, Dcell=Dcell, **kw)
    r = (np.zeros_like(Az) if f is None else np.asarray(f, dtype=np.float64)) - Az
    znew = np.asarray(z, dtype=np.float64) + (dt / dT) * r
    out = bcoef * znew
    if a != 0.0:
        out = out + a * np.asarray(w, dtype=np.float64)
    assert out.size == np.asarray(z).size and out.size % n3 == 0
    return out

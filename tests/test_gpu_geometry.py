"""Multilinear-geometry kernel (dg_geo.cuh, dg_set_geometry; NEXT-3: Problem C's "multilinear
geometries") against the geometry oracle O-2 (oracle/o2_geometry.py,
pinned in tests/test_oracle_geometry.py), at 1e-12 of max|y| (reading C-14):
every compiled quadrature (q = 2p, 2p + 4, 3p + 4), per term mask, full constant D, Dirichlet and
periodic boxes of perturbed hexahedra; the regular grid against the axis-aligned kernels; linear
consistency through dg_residual; conservation; a partitioned run (in-process fabric) against the
single-rank one; rejection of inverted meshes."""
import threading

import numpy as np
import pytest

from oracle import o2_geometry as o2g
from paper_1711_10885_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DFULL = (1.0, 0.2, 0.1, 0.2, 2.0, -0.3, 0.1, -0.3, 0.5)
B = (1.0, -0.5, 0.25)


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def padded(ncells, lo, hi, amp, seed, periodic, cell_lo=(0, 0, 0), cell_cnt=None):
    """The padded vertex grid of a rank's box (include/dg.h: local vertices -1 .. nloc + 1)."""
    cnt = ncells if cell_cnt is None else cell_cnt
    box = (tuple(cell_lo[q] - 1 for q in range(3)), tuple(cell_lo[q] + cnt[q] + 2 for q in range(3)))
    return inputs.vertex_grid(ncells, lo, hi, amp, seed, periodic, box=box)


def m_choices(k):
    return sorted({k + 1, k + 3, -(-(3 * k + 5) // 2)} - {m for m in (k + 3, -(-(3 * k + 5) // 2)) if m > 16})


def gpu_apply(ncells, lo, hi, k, D, b, c, sigma, z, m, amp, seed, periodic=(0, 0, 0), mask=7, f=None):
    from paper_1711_10885_b200 import dg
    op = dg.Operator(ncells, lo, hi, k, D, b, c, sigma, bc=dg.bc_from_periodic(periodic))
    op.set_geometry(padded(ncells, lo, hi, amp, seed, periodic), m)
    zt = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    y = torch.full_like(zt, float("nan"))
    if f is not None:
        op.residual(zt, torch.from_numpy(np.ascontiguousarray(f)).cuda(), y)
    else:
        op.apply(zt, y, terms=mask)
    torch.cuda.synchronize()
    op.close()
    return y.cpu().numpy()


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 1)])
def test_geometry_vs_o2_every_quadrature(k, periodic):
    nc, lo, hi = (3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5)
    sigma = 3.0 * k * (k + 2) / 0.25
    z = inputs.uniform(12 * (k + 1) ** 3, 11 + k)
    X = inputs.vertex_grid(nc, lo, hi, 0.2, k, periodic)
    for m in m_choices(k):
        A = o2g.assemble(nc, X, k, DFULL, B, 0.3, sigma, m=m, periodic=periodic)
        y = gpu_apply(nc, lo, hi, k, DFULL, B, 0.3, sigma, z, m, 0.2, k, periodic)
        assert rel(y, A @ z) < 1e-12, m


@pytest.mark.parametrize("mask", [1, 2, 4])
def test_geometry_term_masks(mask):
    k, nc, lo, hi = 3, (3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5)
    X = inputs.vertex_grid(nc, lo, hi, 0.22, 3)
    z = inputs.uniform(12 * 64, 5)
    A = o2g.assemble(nc, X, k, DFULL, B, 0.3, 40.0, m=6, mask=mask)
    y = gpu_apply(nc, lo, hi, k, DFULL, B, 0.3, 40.0, z, 6, 0.22, 3, mask=mask)
    assert rel(y, A @ z) < 1e-12


@pytest.mark.parametrize("k,m", [(6, 7), (6, 12), (7, 8), (7, 10), (7, 13), (8, 15), (9, 16), (10, 11), (10, 13)])
def test_geometry_high_degree_vs_o2(k, m):
    """Two cells: an interior and two Dirichlet x-faces, self-periodic y and z (wrap onto itself)."""
    nc, lo, hi = (2, 1, 1), (0.0, 0.0, 0.0), (1.0, 0.5, 0.5)
    per = (0, 1, 1)
    sigma = 3.0 * k * (k + 2) / 0.5
    z = inputs.uniform(2 * (k + 1) ** 3, 21)
    X = inputs.vertex_grid(nc, lo, hi, 0.2, 8, per)
    A = o2g.assemble(nc, X, k, DFULL, B, 0.3, sigma, m=m, periodic=per)
    y = gpu_apply(nc, lo, hi, k, DFULL, B, 0.3, sigma, z, m, 0.2, 8, per)
    assert rel(y, A @ z) < 1e-12


@pytest.mark.parametrize("k", [2, 7])
def test_regular_grid_equals_axis_aligned_kernels(k):
    """The identity geometry on the Q1 path reproduces the axis-aligned operator (fast kernel for a
    diagonal D, general kernel for a full D)."""
    from paper_1711_10885_b200 import dg
    for D in ((1.0, 0, 0, 0, 2.0, 0, 0, 0, 0.5), DFULL):
        cfg = configs.small(k, ncells=(4, 3, 2), hi=(2.0, 1.5, 1.0), D=D)
        op = dg.from_config(cfg)
        z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
        op.fill_uniform_local(z, 3)
        y0, y1 = torch.empty_like(z), torch.empty_like(z)
        op.apply(z, y0)
        op.set_geometry(padded(cfg.ncells, cfg.lo, cfg.hi, 0.0, 0, (0, 0, 0)))
        op.apply(z, y1)
        op.set_geometry(None)
        y2 = torch.empty_like(z)
        op.apply(z, y2)
        torch.cuda.synchronize()
        op.close()
        assert rel(y1.cpu().numpy(), y0.cpu().numpy()) < 1e-13
        assert torch.equal(y0, y2)


@pytest.mark.parametrize("k,m", [(2, 3), (3, 4), (5, 6), (7, 8)])
def test_geometry_linear_consistency_residual(k, m):
    """dg_residual(z*, F) = F - A z* ~ 0 for a physical linear field on a perturbed mesh (the oracle's
    z*, F: rhs written on the physical mesh, oracle/o2_geometry.consistency_data)."""
    nc, lo, hi = (3, 3, 2), (0.0, 0.0, 0.0), (1.5, 1.5, 1.0)
    X = inputs.vertex_grid(nc, lo, hi, 0.2, 2)
    sigma = 3.0 * k * (k + 2) / 0.5
    D = np.array(DFULL).reshape(3, 3)
    z, F = o2g.consistency_data(nc, X, k, D, B, 0.7, sigma, m=m, seed=k)
    r = gpu_apply(nc, lo, hi, k, DFULL, B, 0.7, sigma, z, m, 0.2, 2, f=F)
    assert np.abs(r).max() < 1e-12 * np.abs(F).max()


@pytest.mark.parametrize("k", [1, 4, 7])
def test_geometry_conservation_periodic(k):
    """a_h(u, 1) = 0 with c = 0 on a periodic box: the constant-mode components of y sum to zero."""
    nc, lo, hi = (4, 3, 3), (0.0, 0.0, 0.0), (2.0, 1.5, 1.5)
    per = (1, 1, 1)
    n3 = (k + 1) ** 3
    z = inputs.uniform(36 * n3, 4)
    y = gpu_apply(nc, lo, hi, k, DFULL, B, 0.0, 3.0 * k * (k + 2) / 0.5, z, k + 1, 0.2, 6, per)
    assert abs(y[::n3].sum()) < 1e-12 * np.abs(y).max() * np.sqrt(36)


def test_geometry_rejects_inverted_and_unsupported():
    from paper_1711_10885_b200 import dg
    nc, lo, hi = (2, 2, 2), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    op = dg.Operator(nc, lo, hi, 2, DFULL, B, 0.3, 20.0)
    X = padded(nc, lo, hi, 0.1, 1, (0, 0, 0))
    X[2, 2, 2] += (0.9, 0.9, 0.9)             # the middle vertex crosses its neighbours: inverted cells
    with pytest.raises(dg.DGError) as ei:
        op.set_geometry(X, 3)
    assert ei.value.code == dg.DG_EINVAL
    with pytest.raises(dg.DGError) as ei:
        op.set_geometry(padded(nc, lo, hi, 0.1, 1, (0, 0, 0)), 4)      # m = k+2: not compiled
    assert ei.value.code == dg.DG_EUNSUPPORTED
    op.set_geometry(padded(nc, lo, hi, 0.1, 1, (0, 0, 0)), 3)
    with pytest.raises(dg.DGError):
        op.set_velocity(1)
    z = torch.zeros(op.ndofs, dtype=torch.float64, device="cuda")
    with pytest.raises(dg.DGError):
        op.ssp_stage(z, torch.empty_like(z), 1e-3)
    op.close()


@pytest.mark.parametrize("parts,periodic", [((2, 1, 1), (1, 0, 0)), ((2, 2, 1), (0, 0, 0)), ((1, 2, 2), (0, 1, 1))])
def test_geometry_partitioned_fabric_equals_single(parts, periodic):
    """Ranks as threads (in-process fabric): the face traces cross the partition, each rank's padded
    vertex grid holds the neighbour rank's vertices; bit for bit the single-rank result."""
    from paper_1711_10885_b200 import dg
    k, m = 3, 4
    nc, lo, hi = (4, 4, 4), (0.0, 0.0, 0.0), (2.0, 2.0, 2.0)
    world = parts[0] * parts[1] * parts[2]
    fid = dg.fabric_id()
    ops = [dg.Operator(nc, lo, hi, k, DFULL, B, 0.3, 60.0, rank=r, nranks=world, parts=parts, nccl_id=fid,
                       bc=dg.bc_from_periodic(periodic)) for r in range(world)]
    out, errors = [None] * world, []

    def work(r):
        try:
            op = ops[r]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                op.set_geometry(padded(nc, lo, hi, 0.2, 3, periodic, op.cell_lo, op.cell_cnt), m, stream=st)
                z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
                op.fill_uniform_local(z, 9, stream=st)
                y = torch.empty_like(z)
                op.apply(z, y, stream=st)
                st.synchronize()
                out[r] = y.cpu().numpy()
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    n3 = (k + 1) ** 3
    yg = np.full(np.prod(nc) * n3, np.nan)
    for op, y in zip(ops, out):
        lo_, cnt = op.cell_lo, op.cell_cnt
        gz, gy, gx = np.meshgrid(np.arange(lo_[2], lo_[2] + cnt[2]), np.arange(lo_[1], lo_[1] + cnt[1]),
                                 np.arange(lo_[0], lo_[0] + cnt[0]), indexing="ij")
        yg.reshape(-1, n3)[(gx + nc[0] * (gy + nc[1] * gz)).reshape(-1)] = y.reshape(-1, n3)
        op.close()
    z = inputs.uniform(len(yg), 9)
    ys = gpu_apply(nc, lo, hi, k, DFULL, B, 0.3, 60.0, z, m, 0.2, 3, periodic)
    assert np.array_equal(yg, ys)
    X = inputs.vertex_grid(nc, lo, hi, 0.2, 3, periodic)
    A = o2g.assemble(nc, X, k, DFULL, B, 0.3, 60.0, m=m, periodic=periodic)
    assert rel(yg, A @ z) < 1e-12

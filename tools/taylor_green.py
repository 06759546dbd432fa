"""The paper's instationary Taylor-Green transport run at small scale (NEXT-2).

    python tools/taylor_green.py [--k 3] [--cells 24] [--steps 200] [--cfl 0.1] [--out FILE]

-div(D grad u) + div(b u) = 0 on the periodic box (-pi, pi)^3 with D = 5e-6 I, c = f = 0, the
Taylor-Green field b(x) of eq:2 at every quadrature point, q = 2p + 4 (m = k + 3 Gauss points),
SIPG in space and Heun (SSP-RK2, Shu-Osher form) in time, every stage one fused dg_ssp_stage
(kernel + M^-1 update in the store). u_0 = exp(-2 |x - x_0|^2), x_0 = (1/2, 0, 0), L2-projected
cell by cell (the Gaussian is a product of 1D factors, so the projection is a product of 1D
integrals, computed here with a 24-point Gauss rule per cell and direction).

Reports: DOF-stages/s of the time loop (CUDA events), the conserved mass sum_e Delta_T z_(e,0)
(drift relative to the start), the L2 norm (it may only decrease: upwind + SIPG dissipation) and
min/max of the cell means.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import dg  # noqa: E402


def project_gaussian(N, k, lo, h, x0, alpha=2.0, nq=24):
    """z[e, jz, jy, jx] of u0 = prod_d exp(-alpha (x_d - x0_d)^2) in the orthonormal Legendre basis."""
    t, w = np.polynomial.legendre.leggauss(nq)
    xi, wq = 0.5 * (t + 1.0), 0.5 * w
    n = k + 1
    # theta_j(xi) = sqrt(2j+1) P_j(2 xi - 1)
    th = np.stack([np.sqrt(2 * j + 1) * np.polynomial.legendre.legval(2 * xi - 1, [0] * j + [1]) for j in range(n)], 1)
    facs = []
    for d in range(3):
        X = lo[d] + (np.arange(N)[:, None] + xi[None, :]) * h      # [cell, point]
        g = np.exp(-alpha * (X - x0[d]) ** 2)
        facs.append(np.einsum("cp,p,pj->cj", g, wq, th))             # (1/h) int g theta_j dx = sum w g theta
    z = np.einsum("zc,yb,xa->zyxcba", facs[2], facs[1], facs[0])     # [iz, iy, ix, jz, jy, jx]
    return np.ascontiguousarray(z).reshape(-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--cells", type=int, default=24)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--cfl", type=float, default=0.1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    k, N = a.k, a.cells
    lo, hi = (-math.pi,) * 3, (math.pi,) * 3
    h = 2 * math.pi / N
    d = 5e-6
    sigma = 3.0 * k * (k + 2) / h
    op = dg.Operator((N, N, N), lo, hi, k, (d, 0, 0, 0, d, 0, 0, 0, d), (0, 0, 0), 0.0, sigma,
                     bc=dg.bc_from_periodic((1, 1, 1)))
    op.set_velocity(1)
    op.set_quadrature(k + 3)
    u = torch.from_numpy(project_gaussian(N, k, lo, h, (0.5, 0.0, 0.0))).cuda()
    n3 = (k + 1) ** 3
    dT = h ** 3
    dt = a.cfl * h / (2 * k + 1)          # |b| <= 1 for the Taylor-Green field

    def stats(v):
        means = v.view(-1, n3)[:, 0]
        return {"mass": float(means.sum()) * dT, "l2": float(torch.linalg.vector_norm(v)) * math.sqrt(dT),
                "min_mean": float(means.min()), "max_mean": float(means.max())}

    s0 = stats(u)
    tmp, nxt = torch.empty_like(u), torch.empty_like(u)
    op.heun_step(u, dt, tmp, nxt)          # warm-up (not counted)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        op.heun_step(u, dt, tmp, nxt)
        u, nxt = nxt, u
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) * 1e-3
    s1 = stats(u)
    info = op.kernel_info()
    op.close()
    out = {"run": "Taylor-Green transport (PAPER.md:1089-1106), small scale", "k": k, "cells": [N, N, N],
           "ndofs": N ** 3 * n3, "m": k + 3, "dt": dt, "steps": a.steps + 1, "t_end": dt * (a.steps + 1),
           "stage_gdofs": 2 * a.steps * N ** 3 * n3 / secs / 1e9, "ms_per_step": secs / a.steps * 1e3,
           "start": s0, "end": s1, "mass_drift_rel": abs(s1["mass"] - s0["mass"]) / abs(s0["mass"]),
           "l2_nonincreasing": s1["l2"] <= s0["l2"] * (1 + 1e-12), "kernel": info}
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

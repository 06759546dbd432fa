"""Kernel-variant and determinism checks on the GPU.

* The k = 7 FP64 tensor-core kernel (dg_mma8.cuh, opt-in DG_CELL_KERNEL=mma) against the
  oracle O-1 per term mask, on meshes with every boundary type (run in a subprocess: the
  kernel choice is read once per process).
* k = 1, 2: the register-resident kernels (dg_reg.cuh, the default for n <= 3) and the pencil kernels (DG_CELL_KERNEL=pencil) against O-1, per mask, constant and
  per-cell tensors, Dirichlet and periodic (subprocess per kernel choice).
* Determinism: repeated applies are bit-identical (no atomics, no races: each cell is
  computed by one CTA and written once). compute-sanitizer is closed on this pool, so this
  plus NaN-initialised outputs in every parity test stand in for racecheck/initcheck.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1711_10885_b200 import configs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from oracle import o1
from paper_1711_10885_b200 import configs, dg, inputs
out = []
cases = [configs.small(7, ncells=(3, 2, 2)), configs.small(7, ncells=(5, 3, 2), b=(-1.0, 0.5, -0.25), c=0.3),
         configs.small(7, ncells=(1, 1, 1)), configs.small(7, ncells=(4, 1, 3), D=(0,) * 9)]
for cfg in cases:
    z = inputs.uniform(cfg.ndofs, 11)
    op = dg.from_config(cfg)
    zt = torch.from_numpy(z).cuda()
    for mask in (1, 2, 4, 7):
        y = torch.full_like(zt, float('nan'))
        op.apply(zt, y, terms=mask)
        torch.cuda.synchronize()
        yref, _ = o1.apply(*cfg.args(), z, mask=mask)
        den = max(np.abs(yref).max(), 1e-300)
        out.append([cfg.name, mask, float(np.abs(y.cpu().numpy() - yref).max() / den), float(np.abs(yref).max())])
    op.close()
print(json.dumps({"kernel": %r, "rows": out}))
"""


@pytest.mark.parametrize("kernel", ["mma", "simt"])
def test_k7_kernel_variants_vs_o1(kernel):
    env = dict(os.environ, DG_CELL_KERNEL=kernel, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, kernel)], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, mask, err, scale in res["rows"]:
        if scale == 0.0:
            assert err == 0.0
        else:
            assert err < 1e-12, (name, mask, err)


SCRIPT_LOWK = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from oracle import o1
from paper_1711_10885_b200 import configs, dg, inputs
out = []
rng = np.random.default_rng(3)
for k in (1, 2):
    for cfg, per, tensors in ((configs.small(k, ncells=(5, 3, 4)), (0, 0, 0), False),
                              (configs.small(k, ncells=(4, 3, 2), b=(-1.0, 0.5, -0.25)), (1, 0, 1), False),
                              (configs.small(k, ncells=(3, 4, 2), b=(0.3, -0.2, 0.1)), (1, 1, 1), True),
                              (configs.small(k, ncells=(4, 2, 3)), (0, 1, 0), True)):
        ncell = cfg.ncells[0] * cfg.ncells[1] * cfg.ncells[2]
        op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, k, cfg.D, cfg.b, cfg.c, cfg.sigma, bc=dg.bc_from_periodic(per))
        Dc = None
        if tensors:
            M = rng.normal(size=(ncell, 3, 3))
            Dc = np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)[None]
            op.set_diffusion(torch.from_numpy(Dc.reshape(-1).copy()).cuda())
        z = inputs.uniform(cfg.ndofs, 5 + k)
        zt = torch.from_numpy(z).cuda()
        info = op.kernel_info()
        for mask in (1, 2, 4, 7):
            y = torch.full_like(zt, float("nan"))
            op.apply(zt, y, terms=mask)
            torch.cuda.synchronize()
            yref, _ = o1.apply(*cfg.args(), z, mask=mask, periodic=per, Dcell=Dc)
            den = max(np.abs(yref).max(), 1e-300)
            out.append([k, str(per), tensors, mask, float(np.abs(y.cpu().numpy() - yref).max() / den),
                        float(np.abs(yref).max()), info["cells_per_cta"] == info["threads_per_cta"]])
        op.close()
print(json.dumps({"rows": out}))
"""


@pytest.mark.parametrize("kernel", ["reg", "pencil"])
def test_low_degree_kernels_vs_o1(kernel):
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("DG_CELL_KERNEL", None)
    if kernel == "pencil":
        env["DG_CELL_KERNEL"] = "pencil"
    r = subprocess.run([sys.executable, "-c", SCRIPT_LOWK % ROOT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(res["rows"]) == 2 * 4 * 4
    for k, per, tensors, mask, err, scale, one_thread_per_cell in res["rows"]:
        # the register kernels run one thread per cell (the pencil kernels several): shows which kernel ran
        assert one_thread_per_cell == (kernel == "reg"), (k, per, tensors)
        if scale == 0.0:
            assert err == 0.0
        else:
            assert err < 1e-12, (k, per, tensors, mask, err)


def test_repeat_applies_bit_identical():
    from paper_1711_10885_b200 import dg
    for cfg in (configs.small(7, ncells=(16, 8, 8), hi=(1, 1, 1)), configs.small(3, ncells=(20, 9, 7))):
        op = dg.from_config(cfg)
        z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
        op.fill_uniform_local(z, 5)
        ys = []
        for _ in range(3):
            y = torch.full_like(z, float("nan"))
            op.apply(z, y)
            torch.cuda.synchronize()
            ys.append(y.cpu().numpy())
        op.close()
        assert np.all(np.isfinite(ys[0]))
        assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])


@pytest.mark.parametrize("ncells,periodic,general", [((6, 5, 37), (0, 0, 0), False), ((4, 4, 3), (1, 1, 0), False),
                                                    ((5, 3, 20), (0, 0, 1), False), ((4, 3, 19), (1, 0, 0), True)])
def test_apply_host_pipeline_equals_device_apply(ncells, periodic, general):
    """dg_apply_host (z-slab pipeline: H2D / kernel / D2H overlapped; plain path for z-periodic)
    gives bit for bit the device dg_apply result."""
    from paper_1711_10885_b200 import configs, dg, inputs
    cfg = configs.small(3, ncells=ncells, hi=(1.0, 1.0, 2.0))
    op = dg.from_config(cfg, bc=dg.bc_from_periodic(periodic))
    if general:
        op.set_tensor_field(6)
    zh = inputs.uniform(cfg.ndofs, 4)
    yh = np.full(cfg.ndofs, np.nan)
    op.apply_host(zh, yh)
    z = torch.from_numpy(zh).cuda()
    y = torch.empty_like(z)
    op.apply(z, y)
    torch.cuda.synchronize()
    op.close()
    assert np.array_equal(yh, y.cpu().numpy())

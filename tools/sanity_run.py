"""Small end-to-end runs of every kernel path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): C1 (k=2), a k=7 mesh with ragged edges, masks, the residual
epilogue and a 2x1x1 loopback partition. Prints one line per case."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import configs, dg  # noqa: E402

cases = [configs.c1(), configs.small(7, ncells=(3, 2, 2)), configs.small(10, ncells=(2, 2, 1)),
         configs.small(1, ncells=(5, 3, 2))]
for cfg in cases:
    op = dg.from_config(cfg)
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.empty_like(z)
    for terms in (7, 1, 2, 4):
        op.apply(z, y, terms=terms)
    f = torch.ones_like(z)
    r = torch.empty_like(z)
    op.residual(z, f, r)
    torch.cuda.synchronize()
    print(cfg.name, "ok", float(y.abs().max()), flush=True)
    op.close()
# loopback partition 2x1x1 (k = 7)
cfg = configs.small(7, ncells=(4, 2, 2))
ops = [dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, rank=r, nranks=2,
                   parts=(2, 1, 1)) for r in range(2)]
zs = []
for op in ops:
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    op.halo_pack(z)
    zs.append(z)
torch.cuda.synchronize()
for r, op in enumerate(ops):
    y = torch.empty_like(zs[r])
    op.apply(zs[r], y, terms=dg.ALL | dg.HALO_EXTERNAL)
torch.cuda.synchronize()
print("loopback ok", flush=True)

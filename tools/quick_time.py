"""Quick device timing of dg_apply for one config (development aid; bench.py is the contract)."""
import os
import sys
import time

import torch

if os.environ.get("PYTHONPATH"):
    sys.path.insert(0, os.environ["PYTHONPATH"].split(":")[0])   # tools/ab_time.py: the tree under test first
else:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1711_10885_b200 import configs, dg

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = configs.by_name(name)
op = dg.from_config(cfg)
if cfg.dfield_seed >= 0:
    op.set_tensor_field(cfg.dfield_seed)
print(cfg.name, "ndofs", cfg.ndofs, op.kernel_info(), flush=True)
z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
y = torch.empty_like(z)
op.fill_uniform_local(z, cfg.seed)
for _ in range(3):
    op.apply(z, y)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    op.apply(z, y)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
ts.sort()
t = ts[len(ts) // 2]
print("median %.3f ms  min %.3f ms  GDOF/s %.2f" % (t * 1e3, ts[0] * 1e3, cfg.ndofs / t / 1e9), flush=True)

"""A/B of dg_apply_host wall time (development aid)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1711_10885_b200 import configs, dg
cfg = configs.c3()
op = dg.from_config(cfg)
z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
op.fill_uniform_local(z, cfg.seed)
zh = z.cpu().pin_memory().numpy()
yh = torch.empty(cfg.ndofs, dtype=torch.float64).pin_memory().numpy()
for _ in range(2):
    op.apply_host(zh, yh)
ts = []
for _ in range(8):
    t0 = time.perf_counter(); op.apply_host(zh, yh); ts.append(time.perf_counter() - t0)
ts.sort()
print("median %.2f ms min %.2f ms -> %.2f GDOF/s" % (ts[4] * 1e3, ts[0] * 1e3, cfg.ndofs / ts[4] / 1e9))

"""Per-term-mask timing of one workload (development aid): full, volume only, faces only."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1711_10885_b200 import configs, dg
cfg = configs.by_name(sys.argv[1])
op = dg.from_config(cfg)
if cfg.dfield_seed >= 0:
    op.set_tensor_field(cfg.dfield_seed)
z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
op.fill_uniform_local(z, cfg.seed)
y = torch.empty_like(z)
for name, m in (("all", 7), ("volume", 1), ("interior", 2), ("faces", 6), ("none", 0)):
    for _ in range(2):
        op.apply(z, y, terms=m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        op.apply(z, y, terms=m)
    e1.record()
    torch.cuda.synchronize()
    print("%-8s %.3f ms" % (name, e0.elapsed_time(e1) / 5))
